// gemm_simt.cu — fp32 FFMA GEMM C = P Q^T (+ epilogue): the scaffold / reference-precision path
// for the products of Algorithm 1 line 3 and K = B B'^T. The tensor-core path
// (gemm_tc.cu, 3xTF32 tcgen05) is the default; this kernel is FASTPFP_OPT_PRECISION = 2 and the
// path used for the small attribute GEMM.
//
// Tile 128 x 128 x 16, 256 threads, 8 x 8 outputs per thread, both operands K-major (row-major
// with K contiguous), staged transposed in shared memory. Zero-filled at the M/N/K edges.
#include <algorithm>

#include "common.cuh"

namespace fpfp {

namespace {

constexpr int BM = 128, BN = 128, BK = 16;

__device__ __forceinline__ void load_tile(const float* __restrict__ src, int64_t ld, int r0,
                                          int rows, int k0, int K, bool vec_ok,
                                          float (*dst)[BM + 4]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int idx = threadIdx.x + 256 * h;
    const int row = idx >> 2, kq = (idx & 3) * 4;
    const int gr = r0 + row, gk = k0 + kq;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (gr < rows) {
      const float* p = src + (int64_t)gr * ld + gk;
      if (vec_ok && gk + 3 < K) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (gk + e < K) v[e] = p[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) dst[kq + e][row] = v[e];
  }
}

__global__ void __launch_bounds__(256) gemm_nt_simt_kernel(GemmArgs g, bool vec_ok) {
  if (g.done && *g.done) return;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < g.K; k0 += BK) {
    load_tile(g.P, g.ldP, m0, g.M, k0, g.K, vec_ok, As);
    load_tile(g.Q, g.ldQ, n0, g.N, k0, g.K, vec_ok, Bs);
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int gr = m0 + ty * 8 + i;
    if (gr >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gc = n0 + tx * 8 + j;
      if (gc >= g.N) continue;
      const float v = acc[i][j];
      const int64_t o = (int64_t)gr * g.ldC + gc;
      if (g.epi == kEpiAxpy) {
        g.C[o] = g.D ? v + g.lam * g.D[(int64_t)gr * g.ldD + gc] : v;
      } else if (g.epi == kEpiPG) {
        const float gd = g.D ? v + g.lam * g.D[(int64_t)gr * g.ldD + gc] : v;
        g.C[o] = g.scale * gd + g.D2[(int64_t)gr * g.ldD2 + gc];
      } else if (g.epi == kEpiSplit) {
        const float hb = tf32_rna(v);
        g.C[o] = hb;
        g.C2[o] = tf32_rna(v - hb);
        if (g.C3) g.C3[o] = v;
      } else {
        g.C[o] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  const bool vec_ok = (g.ldP % 4 == 0) && (g.ldQ % 4 == 0) &&
                      (reinterpret_cast<uintptr_t>(g.P) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(g.Q) % 16 == 0);
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM));
  gemm_nt_simt_kernel<<<grid, 256, 0, s>>>(g, vec_ok);
  return cudaGetLastError();
}

}  // namespace fpfp
