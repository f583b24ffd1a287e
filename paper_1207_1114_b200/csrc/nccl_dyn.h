// nccl_dyn.h — NCCL entry points resolved at run time (dlopen), so the library links no NCCL and
// uses the same libnccl.so.2 the host process (torch) already loaded. FASTPFP_NCCL_LIB may name
// the library explicitly (the Python binding points it at torch's bundled NCCL).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace fpfp {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
};

// nullptr (with `err` set) if NCCL cannot be loaded.
const NcclApi* nccl_api(std::string& err);

}  // namespace fpfp
