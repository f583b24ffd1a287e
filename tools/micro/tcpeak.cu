// Microbenchmark: issue rate of tcgen05.mma (cta_group::2) with operands resident in shared memory
// and no global traffic: kind::i8 M=256 N=128 K=32 and kind::tf32 M=256 N=256 K=8, one CTA pair
// per 2 SMs (74 pairs). Prints MAC/clk/SM from clock64 and TOPS from CUDA events. Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1207_1114_b200/csrc \
//        tools/micro/tcpeak.cu -o tools/micro/tcpeak -lcuda
#include <cstdio>
#include "tcgen05.cuh"
using namespace fpfp::tc;

template <int KIND>   // 0 = i8 (N=128), 1 = tf32 (N=256)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  long long t0 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t a = smem_desc(smem_u32(sm)), b = smem_desc(smem_u32(sm + 16384));
    constexpr uint32_t id_i8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
    constexpr uint32_t id_tf = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tbase + (uint32_t)((i % 3) * 128)), "l"(a), "l"(b), "r"(id_i8), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tbase + (uint32_t)((i % 2) * 256)), "l"(a), "l"(b), "r"(id_tf), "r"(1));
    }
    umma_commit<2>(&bar);
  }
  if (threadIdx.x == 0) mbar_wait(&bar, 0);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

template <int KIND>
void run(const char* name, int iters) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  auto kern = k<KIND>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<148, 128, 64 * 1024>>>(iters / 10, cyc);
  cudaEventRecord(e0);
  kern<<<148, 128, 64 * 1024>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const double mac_per_mma = KIND == 0 ? 256.0 * 128 * 32 : 256.0 * 256 * 8;   // per CTA pair
  const double macs = 74.0 * iters * mac_per_mma;
  printf("%s: %s, %d MMAs/pair, %.3f ms, %.1f T(ops)/s dense, %.0f MAC/clk/SM (cycles %lld)\n", name,
         cudaGetErrorString(err), iters, ms, 2 * macs / (ms * 1e-3) / 1e12,
         mac_per_mma * iters / 2.0 / (double)h[0], h[0]);
  cudaFree(cyc);
}

int main() {
  run<0>("kind::i8  M256 N128 K32", 200000);
  run<1>("kind::tf32 M256 N256 K8", 100000);
  run<0>("kind::i8  M256 N128 K32", 200000);
  return 0;
}
