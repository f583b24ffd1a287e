// pipes.cu — per-SM throughput of the instruction forms the batched small-pair kernel leans on:
// FADD (3-register), FADD2 (add.rn.f32x2), FFMA2, FMNMX, I2F (cvt.rn.f32.s32), IADD-magic
// conversion, SHFL; and the fp64 forms of the on-chip projection: DADD, DFMA, max.f64, cvt.rn.f32.f64. Each thread runs 8 independent chains; 1 CTA of 1024 threads per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}

template <int K>
__global__ void bench(float* out, int iters, float s, long long* clk) {
  float v[8]; int iv[8]; unsigned long long p[8]; double dv[8];
  for (int k = 0; k < 8; ++k) { v[k] = threadIdx.x * 0.001f + k; iv[k] = threadIdx.x + k; p[k] = __float_as_uint(v[k]) | ((unsigned long long)__float_as_uint(v[k] + 1) << 32); dv[k] = v[k]; }
  const unsigned long long ps = __float_as_uint(s) | ((unsigned long long)__float_as_uint(s) << 32);
  float sv = s; float sv2 = s * 1.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (K == 0) asm volatile("add.f32 %0, %0, %1;" : "+f"(v[k]) : "f"(sv));
      if (K == 1) p[k] = add2(p[k], ps);
      if (K == 2) p[k] = fma2(p[k], ps, ps);
      if (K == 3) asm volatile("max.f32 %0, %0, %1;" : "+f"(v[k]) : "f"(sv2));
      if (K == 4) { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(iv[k])); iv[k] = __float_as_int(f) ^ it; }
      if (K == 5) { float f = __int_as_float(iv[k] + 0x4B400000) - 12582912.0f; iv[k] = __float_as_int(f) ^ it; }
      if (K == 6) v[k] = __shfl_xor_sync(0xffffffffu, v[k], 1 + (k & 7)) + 0.0f;
      if (K == 7) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[k]) : "f"(sv), "f"(sv2));
      if (K == 8) asm volatile("add.f64 %0, %0, %1;" : "+d"(dv[k]) : "d"((double)sv));
      if (K == 9) { float f; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(dv[k])); dv[k] = (double)0 + __int_as_float(__float_as_int(f) ^ it); }
      if (K == 10) asm volatile("max.f64 %0, %0, %1;" : "+d"(dv[k]) : "d"((double)sv2));
      if (K == 11) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dv[k]) : "d"((double)sv), "d"((double)sv2));
    }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int k = 0; k < 8; ++k) acc += v[k] + __int_as_float(iv[k]) + __uint_as_float((unsigned)p[k]) + (float)dv[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int K>
void run(const char* name, float* out, long long* dclk) {
  const int iters = 4096, threads = 1024, blocks = 148;
  bench<K><<<blocks, threads>>>(out, iters, 1.0001f, dclk);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, dclk, sizeof h, cudaMemcpyDeviceToHost);
  double c = 0; for (int b = 0; b < blocks; ++b) c += h[b]; c /= blocks;
  const double warp_instr = (double)iters * 8 * threads / 32;
  printf("%-10s %.3f warp-instr/clk/SM  (%.1f lane-ops/clk/SM)\n", name, warp_instr / c, warp_instr / c * 32);
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  run<0>("FADD", out, clk); run<1>("FADD2", out, clk); run<2>("FFMA2", out, clk);
  run<3>("FMNMX", out, clk); run<4>("I2F", out, clk); run<5>("magicI2F", out, clk);
  run<6>("SHFL", out, clk); run<7>("FFMA", out, clk);
  run<8>("DADD", out, clk); run<9>("F2F.F32.F64+", out, clk); run<10>("DMAX", out, clk); run<11>("DFMA", out, clk);
  return 0;
}
