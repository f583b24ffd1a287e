// Microbenchmark: per-sweep global exchange cost (write partials -> barrier -> read partials) on
// B200 with cg::grid.sync vs a monotonic release/acquire counter barrier. Diagnostic only.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

template <int MODE>  // 0 = cg grid.sync, 1 = monotonic counter barrier
__global__ void k_exchange(int iters, double* part, unsigned* ctr, int per_block, double* out) {
  cg::grid_group g = cg::this_grid();
  const int nb = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int buf = it & 1;
    for (int k = threadIdx.x; k < per_block; k += blockDim.x)
      part[((size_t)buf * nb + blockIdx.x) * per_block + k] = acc + k;
    if (MODE == 0) {
      g.sync();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        red_rel(ctr, 1u);
        const unsigned target = (unsigned)nb * (unsigned)(it + 1);
        while (ld_acq(ctr) < target) {}
      }
      __syncthreads();
    }
    // read the partials of 12 peers (like a tile row + column)
    double s = 0;
    for (int k = threadIdx.x; k < per_block; k += blockDim.x)
#pragma unroll
      for (int q = 0; q < 12; ++q) s += part[((size_t)buf * nb + (blockIdx.x + q * 7) % nb) * per_block + k];
    acc += s * 1e-30;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
  double *part, *out; unsigned* ctr;
  cudaMalloc(&part, 2 * 296 * 256 * 8); cudaMalloc(&out, 4096 * 8); cudaMalloc(&ctr, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int nb : {16, 64, 144}) for (int mode = 0; mode < 2; ++mode) {
    int iters = 3000, per = 168;
    cudaMemset(ctr, 0, 4);
    void* args[] = {&iters, &part, &ctr, &per, &out};
    void* fn = mode ? (void*)k_exchange<1> : (void*)k_exchange<0>;
    cudaLaunchCooperativeKernel(fn, nb, 256, args, 0, 0);
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel(fn, nb, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("blocks=%3d %-8s exchange: %.3f us/iter (%s)\n", nb, mode ? "counter" : "grid.sync",
           ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
