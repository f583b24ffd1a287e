// gemm_tc.cu — tcgen05 (5th-gen tensor core) 3xTF32 GEMM for sm_100a. (placeholder: filled in
// by the tensor-core milestone)
#include "common.cuh"

namespace fpfp {

bool gemm_tc_supported(const GemmArgs&) { return false; }

cudaError_t launch_gemm_tc(const GemmArgs&, int, cudaStream_t, int) {
  return cudaErrorNotSupported;
}

}  // namespace fpfp
