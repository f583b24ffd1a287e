// Microbenchmark: cost of a grid-wide barrier on B200 (cooperative groups vs a hand-rolled
// sense-reversing barrier), and of L2 round trips. Diagnostic only (not part of the library).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void k_custom(int iters, unsigned* bar) {
  // bar[0] = arrival counter, bar[1] = generation
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned gen = ld_acquire(&bar[1]);
      __threadfence();
      const unsigned arrived = atomicAdd(&bar[0], 1u);
      if (arrived == gridDim.x - 1) {
        bar[0] = 0;
        __threadfence();
        atomicAdd(&bar[1], 1u);
      } else {
        while (ld_acquire(&bar[1]) == gen) {}
      }
    }
    __syncthreads();
  }
}

__global__ void k_l2chain(const double* p, int n, double* out) {
  // dependent loads: latency of an L2 round trip
  double s = 0; int idx = 0;
  for (int i = 0; i < n; ++i) { double v = p[idx]; s += v; idx = ((int)v + i * 97) & 4095; }
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

int main() {
  int* sink; unsigned* bar; double* buf; double* out;
  cudaMalloc(&sink, 4); cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  cudaMalloc(&buf, 4096 * 8); cudaMemset(buf, 0, 4096 * 8); cudaMalloc(&out, 4096 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {4, 16, 144, 148, 296}) {
    for (int mode = 0; mode < 2; ++mode) {
      int iters = 2000;
      void* args_cg[] = {&iters, &sink};
      void* args_cu[] = {&iters, &bar};
      // warm
      if (mode == 0) cudaLaunchCooperativeKernel((void*)k_cg, blocks, 256, args_cg, 0, 0);
      else cudaLaunchCooperativeKernel((void*)k_custom, blocks, 256, args_cu, 0, 0);
      cudaEventRecord(a);
      if (mode == 0) cudaLaunchCooperativeKernel((void*)k_cg, blocks, 256, args_cg, 0, 0);
      else cudaLaunchCooperativeKernel((void*)k_custom, blocks, 256, args_cu, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("blocks=%3d %-6s barrier: %.3f us  (%s)\n", blocks, mode ? "custom" : "cg",
             ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaEventRecord(a);
  k_l2chain<<<1, 32>>>(buf, 10000, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("dependent L2 load round trip: %.1f ns\n", ms * 1e6 / 10000);
  return 0;
}
