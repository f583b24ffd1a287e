// Microbenchmark: latency / throughput of fp64 ops and double warp shuffles on sm_100a (one CTA of
// 256 threads on one SM), to size the on-chip projection sweep. Diagnostic only.
#include <cstdio>
__global__ void k(int iters, double seed, double* out, long long* cyc) {
  double a = seed + threadIdx.x, b = seed * 0.5, c = 0.0;
  long long t0, t1;
  // 1: dependent DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a + b; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // 2: dependent fmax chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { c = fmax(c, a - (double)i); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // 3: 5-level double shuffle reduction (dependent), 4 interleaved
  double r0 = a, r1 = b, r2 = c, r3 = a * b;
  t0 = clock64();
  for (int i = 0; i < iters / 8; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r0 += __shfl_xor_sync(0xffffffffu, r0, o); r1 += __shfl_xor_sync(0xffffffffu, r1, o);
      r2 += __shfl_xor_sync(0xffffffffu, r2, o); r3 += __shfl_xor_sync(0xffffffffu, r3, o);
    }
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // 4: independent DADD throughput (8 chains)
  double x[8];
  for (int q = 0; q < 8; ++q) x[q] = seed + q;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = x[q] * 1.0000001 + b;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // 5: float shuffle reduction, 4 interleaved
  float f0 = a, f1 = b, f2 = c, f3 = a * b;
  t0 = clock64();
  for (int i = 0; i < iters / 8; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f0 += __shfl_xor_sync(0xffffffffu, f0, o); f1 += __shfl_xor_sync(0xffffffffu, f1, o);
      f2 += __shfl_xor_sync(0xffffffffu, f2, o); f3 += __shfl_xor_sync(0xffffffffu, f3, o);
    }
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  double s = a + c + r0 + r1 + r2 + r3 + f0 + f1 + f2 + f3;
  for (int q = 0; q < 8; ++q) s += x[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
  const int iters = 8192;
  for (int threads : {32, 256, 1024}) {
    k<<<1, threads>>>(iters, 1.0, out, cyc);
    cudaDeviceSynchronize();
    long long h[5]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads %4d: DADD dep %.1f clk | fmax dep %.1f clk | dbl shfl-reduce (4x5 levels) %.1f clk/round | "
           "8 indep DFMA %.2f clk/iter (%.1f DFMA/clk/SM) | flt shfl-reduce %.1f clk/round\n",
           threads, (double)h[0] / iters, (double)h[1] / iters, (double)h[2] / (iters / 8),
           (double)h[3] / iters, 8.0 * threads / ((double)h[3] / iters), (double)h[4] / (iters / 8));
  }
  return 0;
}
