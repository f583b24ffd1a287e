// nccl_dyn.cu — see nccl_dyn.h.
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

#include "nccl_dyn.h"

namespace fpfp {

namespace {
NcclApi g_api;
bool g_ok = false;
std::string g_err;
std::once_flag g_once;

template <typename F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

void load() {
  const char* cands[3] = {std::getenv("FASTPFP_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* c : cands) {
    if (!c || !*c) continue;
    h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    g_err = std::string("cannot dlopen NCCL (set FASTPFP_NCCL_LIB): ") + (dlerror() ? dlerror() : "");
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclAllGather", g_api.AllGather) &&
            sym(h, "ncclAllReduce", g_api.AllReduce) && sym(h, "ncclGroupStart", g_api.GroupStart) &&
            sym(h, "ncclGroupEnd", g_api.GroupEnd) && sym(h, "ncclGetErrorString", g_api.GetErrorString) &&
            sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
            sym(h, "ncclCommAbort", g_api.CommAbort) && sym(h, "ncclSend", g_api.Send) &&
            sym(h, "ncclRecv", g_api.Recv);
  if (!ok) {
    g_err = "NCCL library lacks a required symbol";
    return;
  }
  g_ok = true;
}
}  // namespace

const NcclApi* nccl_api(std::string& err) {
  std::call_once(g_once, load);
  if (!g_ok) {
    err = g_err;
    return nullptr;
  }
  return &g_api;
}

}  // namespace fpfp
