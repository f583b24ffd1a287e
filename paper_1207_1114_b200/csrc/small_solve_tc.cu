// small_solve_tc.cu — Algorithm 1 for many small pairs (n, n' <= 128), one pair per
// CTA, with the two products of line 3 on the int8 tensor cores: the Ozaki digit
// decomposition of gemm_i8.cu (3 signed 7-bit digit planes per operand row, 6 exact int32 digit
// products in 3 TMEM accumulators, fp32-accurate) at M = N = K = 128 per CTA
// (tcgen05.mma.cta_group::1.kind::i8, 24 MMAs per product). BASELINE configs[3] (8192 pairs of 128).
//
// Per pair: the digit planes of A and A' are built once in shared memory (swizzled K-major,
// SWIZZLE_128B: one 128-byte row per matrix row). Per outer iteration:
//   X (global, L2-resident) -> digits -> GEMM1 U = A' X^T (TMEM) -> U digits (row scales over the
//   whole row) -> GEMM2 G = A U^T (TMEM) -> + lambda K -> fp32 staging -> Y registers
//   -> the projection sweeps (same on-chip code as small_solve.cu: Y in registers, fp32 sums)
//   -> blend + rescale on X in global memory.
// Replaces the SIMT FFMA products of small_solve.cu, which are bound by shared-memory bandwidth.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fpfp {

namespace {

using namespace tc;

#ifndef FPFP_SS_THREADS
#define FPFP_SS_THREADS 512
#endif
constexpr int kT = FPFP_SS_THREADS;   // threads (256 or 512)
constexpr int kS = 128;       // max n, n', m
constexpr int kW = kT / 32;   // warps
constexpr int kRW = kS / kW;  // rows of the Y / X register tiles per warp (8 at 512 threads)
constexpr int kEC = kS / (kW / 4);    // epilogue columns per warp (TMEM lane quarter = warp & 3)
constexpr int kLdG = kS + 4;  // fp32 staging row stride
constexpr int kPlane = kS * kS;   // one digit plane: 128 rows x 128 bytes
static_assert(kT == 256 || kT == 512, "256 or 512 threads");

struct __align__(1024) SmemTC {
  int8_t Pd[3][kPlane];       // A' digit planes (GEMM1 M side)
  int8_t Ad[3][kPlane];       // A digit planes (GEMM2 M side)
  int8_t Wd[3][kPlane];       // X digits (GEMM1 N side), then U digits (GEMM2 N side)
  float G[kS][kLdG];          // product staging (row = TMEM lane); during the sweeps it holds
                              // the per-warp column partial sums colp[2][kW][kS] (double buffered)
  float csum[kS];             // combined column sums of the current sweep
  float rsum[2][kW][kRW];     // row sums of each warp's rows (double buffered)
  float dl[2][kW];
  float red[kW];
  int eP[kS], eA[kS], eW[kS]; // row exponents
  float wmax[kW / 4][kS];     // row |max| of U per epilogue column group
  float cscale[kS];           // 2^(e_col - 14) of the N side of the current product
  uint64_t bar;               // MMA completion
  uint32_t tmem_base;
};

static_assert(sizeof(float) * 2 * kW * kS <= sizeof(float) * kS * kLdG, "colp fits in G");
__device__ __forceinline__ float (*colp_of(SmemTC& sm))[kW][kS] {
  return reinterpret_cast<float (*)[kW][kS]>(&sm.G[0][0]);
}

__device__ __forceinline__ float pow2(int e) {
  return (e > -127 && e < 128) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e);
}

// byte offset of (row, col) in a SWIZZLE_128B K-major plane (128-byte rows, 1024-byte atoms)
__device__ __forceinline__ int swz(int row, int col) {
  return row * 128 + ((((col >> 4) ^ (row & 7))) << 4) + (col & 15);
}

__device__ __forceinline__ void digits3(float x, float inv, int& a, int& b, int& c) {
  ozaki_digits3(x, inv, a, b, c);
}
__device__ __forceinline__ int pack4(int d0, int d1, int d2, int d3) {
  return (d0 & 0xFF) | ((d1 & 0xFF) << 8) | ((d2 & 0xFF) << 16) | ((d3 & 0xFF) << 24);
}
// 4 consecutive values -> one packed word (4 digits) per plane
__device__ __forceinline__ void digits4(const float (&v)[4], float inv, int& w1, int& w2, int& w3) {
  int a[4], b[4], c[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) digits3(v[t], inv, a[t], b[t], c[t]);
  w1 = pack4(a[0], a[1], a[2], a[3]);
  w2 = pack4(b[0], b[1], b[2], b[3]);
  w3 = pack4(c[0], c[1], c[2], c[3]);
}

// rows x cols fp32 matrix (row-major, ld = cols, rows/cols <= 128) -> 3 swizzled digit planes +
// row exponents; zero outside. One warp per row (lane l owns columns 4l .. 4l + 3), 4 rows' loads
// in flight per warp (global/L2 latency bounds this step).
__device__ __forceinline__ void split_rows_smem(const float* src, int rows, int cols, int8_t (*d)[kPlane],
                                                int* ex) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = lane * 4;
  for (int r0 = warp * 4; r0 < kS; r0 += (kT / 32) * 4) {
    float v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r = r0 + u;
        v[u][t] = (r < rows && c0 + t < cols) ? __ldg(src + (int64_t)r * cols + c0 + t) : 0.0f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = r0 + u;
      float mx = fmaxf(fmaxf(fabsf(v[u][0]), fabsf(v[u][1])), fmaxf(fabsf(v[u][2]), fabsf(v[u][3])));
      mx = warp_max(mx);
      const int e = frexp_exp(mx);
      if (lane == 0) ex[r] = e;
      int w1, w2, w3;
      digits4(v[u], exp2i(-e), w1, w2, w3);
      const int o = swz(r, c0);
      *reinterpret_cast<int*>(&d[0][o]) = w1;
      *reinterpret_cast<int*>(&d[1][o]) = w2;
      *reinterpret_cast<int*>(&d[2][o]) = w3;
    }
  }
}

// The digit planes of the new X straight from the Y-tile register layout of the blend (warp w owns
// rows 16w .. 16w + 15, lane l columns 4l .. 4l + 3): no reload from global memory; the 4 digits of
// a lane's consecutive columns go to shared memory as one packed word per plane.
__device__ __forceinline__ void split_tile_smem(const float2 (&x)[kRW][2], int8_t (*d)[kPlane], int* ex) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < kRW; ++r) {
    const int row = warp * kRW + r;
    const float v4[4] = {x[r][0].x, x[r][0].y, x[r][1].x, x[r][1].y};
    float mx = fmaxf(fmaxf(fabsf(v4[0]), fabsf(v4[1])), fmaxf(fabsf(v4[2]), fabsf(v4[3])));
    mx = warp_max(mx);
    const int e = frexp_exp(mx);
    if (lane == 0) ex[row] = e;
    int w1, w2, w3;
    digits4(v4, exp2i(-e), w1, w2, w3);
    const int o = swz(row, 4 * lane);
    *reinterpret_cast<int*>(&d[0][o]) = w1;
    *reinterpret_cast<int*>(&d[1][o]) = w2;
    *reinterpret_cast<int*>(&d[2][o]) = w3;
  }
}

__device__ __forceinline__ void mma_i8_1cta(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// C = P Q^T over K = 128 (zero-padded digits): 4 K steps x 6 digit products into the 3 weight-class
// accumulators at TMEM columns 0 / 128 / 256. One thread issues, the commit arrives on `bar`.
__device__ __forceinline__ void issue_product(const int8_t (*P)[kPlane], const int8_t (*Q)[kPlane],
                                              uint32_t tmem, uint64_t* bar) {
  constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kS >> 3) << 17) |
                              ((uint32_t)(kS >> 4) << 24);
  const uint32_t acc2 = tmem, acc3 = tmem + 128, acc4 = tmem + 256;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t off = (uint32_t)k * 32u;
    const uint64_t p1 = smem_desc(smem_u32(P[0]) + off), p2 = smem_desc(smem_u32(P[1]) + off),
                   p3 = smem_desc(smem_u32(P[2]) + off);
    const uint64_t q1 = smem_desc(smem_u32(Q[0]) + off), q2 = smem_desc(smem_u32(Q[1]) + off),
                   q3 = smem_desc(smem_u32(Q[2]) + off);
    const uint32_t acc = k == 0 ? 0u : 1u;
    mma_i8_1cta(acc4, p3, q1, kIdesc, acc);
    mma_i8_1cta(acc4, p2, q2, kIdesc, 1u);
    mma_i8_1cta(acc4, p1, q3, kIdesc, 1u);
    mma_i8_1cta(acc3, p2, q1, kIdesc, acc);
    mma_i8_1cta(acc3, p1, q2, kIdesc, 1u);
    mma_i8_1cta(acc2, p1, q1, kIdesc, acc);
  }
  umma_commit<1>(bar);
}

// This thread's 64 values of row (32 (warp & 3) + lane), columns 64 (warp >> 2) .. + 63, of the
// digit product, (a2 + 2^-7 (a3 + 2^-7 a4)) * rscale * cscale[col] with cscale = 2^(e_col - 14),
// written to dst[0..63] (shared memory, fp32); returns their max |value|.
__device__ __forceinline__ float product_to_smem(uint32_t tmem, float rscale, const float* cscale,
                                                 float* dst) {
  const int warp = threadIdx.x >> 5;
  const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * kEC);
  float mx = 0.0f;
#pragma unroll 1
  for (int h = 0; h < kEC / 16; ++h) {   // 16 columns at a time (48 registers of accumulators)
    uint32_t a2[16], a3[16], a4[16];
    tmem_ld16_nowait(tb + (uint32_t)(h * 16), a2);
    tmem_ld16_nowait(tb + 128u + (uint32_t)(h * 16), a3);
    tmem_ld16_nowait(tb + 256u + (uint32_t)(h * 16), a4);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      float o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int col = (warp >> 2) * kEC + h * 16 + j + t;
        float v = fmaf((float)(int)a4[j + t], 0.0078125f, (float)(int)a3[j + t]);
        v = fmaf(v, 0.0078125f, (float)(int)a2[j + t]);
        o[t] = (v * rscale) * cscale[col];
        mx = fmaxf(mx, fabsf(o[t]));
      }
      *reinterpret_cast<float4*>(dst + h * 16 + j) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  return mx;
}

// All 32 lanes hold partial maxima v[0..15] of 16 rows; on return every lane holds the row maxima
// (transpose butterfly as rows_allreduce16: 32 shuffles instead of 16 x 5).
__device__ __forceinline__ void rows_allmax16(float (&v)[16]) {
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  float a[8], b4[4], b2[2], b1;
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float send = hi ? v[k] : v[8 + k], keep = hi ? v[8 + k] : v[k];
      a[k] = fmaxf(keep, __shfl_xor_sync(F, send, 16));
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float send = hi ? a[k] : a[4 + k], keep = hi ? a[4 + k] : a[k];
      b4[k] = fmaxf(keep, __shfl_xor_sync(F, send, 8));
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float send = hi ? b4[k] : b4[2 + k], keep = hi ? b4[2 + k] : b4[k];
      b2[k] = fmaxf(keep, __shfl_xor_sync(F, send, 4));
    }
  }
  {
    const bool hi = lane & 2;
    const float send = hi ? b2[0] : b2[1], keep = hi ? b2[1] : b2[0];
    b1 = fmaxf(keep, __shfl_xor_sync(F, send, 2));
  }
  b1 = fmaxf(b1, __shfl_xor_sync(F, b1, 1));
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int src = (((r >> 3) & 1) << 4) | (((r >> 2) & 1) << 3) | (((r >> 1) & 1) << 2) | ((r & 1) << 1);
    v[r] = __shfl_sync(F, b1, src);
  }
}

// All 32 lanes hold partial sums v[0..15] of 16 rows; on return every lane holds the full sums
// (the same transpose-butterfly as small_solve.cu).
__device__ __forceinline__ void rows_allreduce16(float (&v)[16]) {
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  float a[8], b4[4], b2[2], b1;
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float send = hi ? v[k] : v[8 + k], keep = hi ? v[8 + k] : v[k];
      a[k] = keep + __shfl_xor_sync(F, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float send = hi ? a[k] : a[4 + k], keep = hi ? a[4 + k] : a[k];
      b4[k] = keep + __shfl_xor_sync(F, send, 8);
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float send = hi ? b4[k] : b4[2 + k], keep = hi ? b4[2 + k] : b4[k];
      b2[k] = keep + __shfl_xor_sync(F, send, 4);
    }
  }
  {
    const bool hi = lane & 2;
    const float send = hi ? b2[0] : b2[1], keep = hi ? b2[1] : b2[0];
    b1 = keep + __shfl_xor_sync(F, send, 2);
  }
  b1 += __shfl_xor_sync(F, b1, 1);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int src = (((r >> 3) & 1) << 4) | (((r >> 2) & 1) << 3) | (((r >> 1) & 1) << 2) | ((r & 1) << 1);
    v[r] = __shfl_sync(F, b1, src);
  }
}

// 8-row versions (16 warps x 8 rows): three halving exchanges leave the lanes whose bits 4..2
// equal a row's index with partials of that row; xor 2 and 1 finish them, then a broadcast
template <bool kMax>
__device__ __forceinline__ void rows_all8(float (&v)[8]) {
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  auto op = [](float a, float b) { return kMax ? fmaxf(a, b) : a + b; };
  float a[4], b2[2], b1;
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float send = hi ? v[k] : v[4 + k], keep = hi ? v[4 + k] : v[k];
      a[k] = op(keep, __shfl_xor_sync(F, send, 16));
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float send = hi ? a[k] : a[2 + k], keep = hi ? a[2 + k] : a[k];
      b2[k] = op(keep, __shfl_xor_sync(F, send, 8));
    }
  }
  {
    const bool hi = lane & 4;
    const float send = hi ? b2[0] : b2[1], keep = hi ? b2[1] : b2[0];
    b1 = op(keep, __shfl_xor_sync(F, send, 4));
  }
  b1 = op(b1, __shfl_xor_sync(F, b1, 2));
  b1 = op(b1, __shfl_xor_sync(F, b1, 1));
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int src = (((r >> 2) & 1) << 4) | (((r >> 1) & 1) << 3) | ((r & 1) << 2);
    v[r] = __shfl_sync(F, b1, src);
  }
}
// element e (0..3) of a lane's 4 consecutive columns held as two float2 pairs
__device__ __forceinline__ float& el(float2 (&v)[2], int e) {
  return (e & 1) ? v[e >> 1].y : v[e >> 1].x;
}

// 8 row partials per lane -> lanes 4r .. 4r + 3 hold the total of row r in v[0] (the halving
// exchanges of rows_all8 without the final broadcast; the owners publish through shared memory)
__device__ __forceinline__ void rows_reduce8(float (&v)[8]) {
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  float a[4], b2[2], b1;
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float send = hi ? v[k] : v[4 + k], keep = hi ? v[4 + k] : v[k];
      a[k] = keep + __shfl_xor_sync(F, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float send = hi ? a[k] : a[2 + k], keep = hi ? a[2 + k] : a[k];
      b2[k] = keep + __shfl_xor_sync(F, send, 8);
    }
  }
  {
    const bool hi = lane & 4;
    const float send = hi ? b2[0] : b2[1], keep = hi ? b2[1] : b2[0];
    b1 = keep + __shfl_xor_sync(F, send, 4);
  }
  b1 += __shfl_xor_sync(F, b1, 2);
  b1 += __shfl_xor_sync(F, b1, 1);
  v[0] = b1;
}

__device__ __forceinline__ void rows_allreduce(float (&v)[16]) { rows_allreduce16(v); }
__device__ __forceinline__ void rows_allreduce(float (&v)[8]) { rows_all8<false>(v); }
__device__ __forceinline__ void rows_allmax(float (&v)[16]) { rows_allmax16(v); }
__device__ __forceinline__ void rows_allmax(float (&v)[8]) { rows_all8<true>(v); }

}  // namespace

template <bool kFull, bool kDelta>
__global__ void __launch_bounds__(kT, 1) small_solve_tc_kernel(SmallArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SmemTC& sm = *reinterpret_cast<SmemTC*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = p.n, np = p.np, m = p.m;
  const float inv_m = 1.0f / (float)m;
  // epilogue geometry: row = TMEM lane 32 (warp & 3) + lane, columns kEC (warp >> 2) ..
  const int erow = (warp & 3) * 32 + lane, ecol0 = (warp >> 2) * kEC;
  float (*colp)[kW][kS] = colp_of(sm);

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  uint32_t bar_phase = 0;

  for (int pair = blockIdx.x; pair < p.batch; pair += gridDim.x) {
    const float* A = p.A + (int64_t)pair * n * n;
    const float* Ap = p.Ap + (int64_t)pair * np * np;
    const float* Kp = p.K ? p.K + (int64_t)pair * n * np : nullptr;
    float* X = p.X + (int64_t)pair * n * np;

    // digit planes of the constant graphs (A' is GEMM1's M side, A is GEMM2's)
    split_rows_smem(Ap, np, np, sm.Pd, sm.eP);
    split_rows_smem(A, n, n, sm.Ad, sm.eA);
    // Y register tile: rows kRW w + r, cols 4l + e, as two float2 pairs (e = 0,1 | 2,3) so the
    // sweep runs on the packed fp32x2 pipe (FADD2)
    float2 y[kRW][2];
#pragma unroll
    for (int r = 0; r < kRW; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = warp * kRW + r, j = 4 * lane + e;
        el(y[r], e) = (p.Y && i < m && j < m) ? p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] : 0.f;
      }

    int it = 0, conv = 0, total_sweeps = 0, degen = 0;
    float rho = 0.f;
    float2 xr[kRW][2];          // X in the Y-tile layout (kept for the blend and the next digits)
#pragma unroll
    for (int r = 0; r < kRW; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = warp * kRW + r, j = 4 * lane + e;
        el(xr[r], e) = (i < n && j < np) ? X[(int64_t)i * np + j] : 0.f;
      }
    split_tile_smem(xr, sm.Wd, sm.eW);
#ifdef FPFP_SS_PROF
    long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define SSP(k) do { const long long t_ = clock64(); tp[k] += t_ - tq; tq = t_; } while (0)
#else
#define SSP(k) do { } while (0)
#endif
    for (; it < p.max_iter1;) {
      // ---- U = A' X^T (line 3, first product): X rows (N side) are in Wd / eW
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (warp == 0) {   // warp-uniform: descriptors stay in uniform registers
        tc_fence_after();
        if (elect_one()) issue_product(sm.Pd, sm.Wd, tmem, &sm.bar);
        __syncwarp();
      }
      mbar_wait(&sm.bar, bar_phase);
      bar_phase ^= 1;
      tc_fence_after();
      SSP(0);
      if (threadIdx.x < kS) sm.cscale[threadIdx.x] = pow2(sm.eW[threadIdx.x] - 14);   // X exps
      __syncthreads();
      // U -> fp32 staging rows (row = TMEM lane), then digits with the scale of the whole row
      const float mx = product_to_smem(tmem, pow2(sm.eP[erow]), sm.cscale, &sm.G[erow][ecol0]);
      sm.wmax[warp >> 2][erow] = mx;
      tc_fence_before();
      __syncthreads();                                     // U staged; X digits / exps consumed
      {
        float rmx = sm.wmax[0][erow];
#pragma unroll
        for (int g = 1; g < kW / 4; ++g) rmx = fmaxf(rmx, sm.wmax[g][erow]);
        const int e = frexp_exp(rmx);
        if (warp < 4) sm.eW[erow] = e;
        const float inv = exp2i(-e);
#pragma unroll 4
        for (int j = 0; j < kEC; j += 4) {
          const float4 g = *reinterpret_cast<const float4*>(&sm.G[erow][ecol0 + j]);
          const float q[4] = {g.x, g.y, g.z, g.w};
          int w1, w2, w3;
          digits4(q, inv, w1, w2, w3);
          const int o = swz(erow, ecol0 + j);
          *reinterpret_cast<int*>(&sm.Wd[0][o]) = w1;
          *reinterpret_cast<int*>(&sm.Wd[1][o]) = w2;
          *reinterpret_cast<int*>(&sm.Wd[2][o]) = w3;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      SSP(1);
      // ---- G = A U^T + lambda K (line 3, second product)
      if (warp == 0) {   // warp-uniform: descriptors stay in uniform registers
        tc_fence_after();
        if (elect_one()) issue_product(sm.Ad, sm.Wd, tmem, &sm.bar);
        __syncwarp();
      }
      mbar_wait(&sm.bar, bar_phase);
      bar_phase ^= 1;
      tc_fence_after();
      SSP(2);
      if (threadIdx.x < kS) sm.cscale[threadIdx.x] = pow2(sm.eW[threadIdx.x] - 14);
      __syncthreads();
      product_to_smem(tmem, pow2(sm.eA[erow]), sm.cscale, &sm.G[erow][ecol0]);   // G staged
      if (Kp && erow < n) {                               // + lambda K (line 3)
        for (int j = 0; j < kEC && ecol0 + j < np; ++j)
          sm.G[erow][ecol0 + j] += p.lam * Kp[(int64_t)erow * np + ecol0 + j];
      }
      tc_fence_before();
      __syncthreads();
      // Y[0:n, 0:n'] = G ; slack entries keep their values (reading A3)
#pragma unroll
      for (int r = 0; r < kRW; ++r) {
        const int i = warp * kRW + r;
        if (kFull) {
          const float4 g = *reinterpret_cast<const float4*>(&sm.G[i][4 * lane]);
          y[r][0] = make_float2(g.x, g.y);
          y[r][1] = make_float2(g.z, g.w);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (i < n && 4 * lane + e < np) el(y[r], e) = sm.G[i][4 * lane + e];
        }
      }
      __syncthreads();   // G is read; the column partials of the sweeps reuse its space

      SSP(3);
      // ---- projection loop (P1 + P2 per sweep), sums of the current Y first. Per sweep: the
      // update and the sums of its output on the packed fp32x2 pipe; a warp's 8 row sums by a
      // transposed butterfly, published in shared memory with its column partials; one barrier;
      // the column partials combined by 4 warps (one thread per column); one barrier.
      int buf = 0;
      auto sums = [&](const float2 (&yy)[kRW][2]) {
        float rp[kRW];
        float2 c01 = make_float2(0.f, 0.f), c23 = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < kRW; ++r) {
          const float2 t = __fadd2_rn(yy[r][0], yy[r][1]);
          rp[r] = t.x + t.y;
          c01 = __fadd2_rn(c01, yy[r][0]);
          c23 = __fadd2_rn(c23, yy[r][1]);
        }
        rows_reduce8(rp);                         // lanes 4r..4r+3 now hold the sum of row r
        if ((lane & 3) == 0) sm.rsum[buf][warp][lane >> 2] = rp[0];
        *reinterpret_cast<float4*>(&colp[buf][warp][4 * lane]) = make_float4(c01.x, c01.y, c23.x, c23.y);
      };
      sums(y);
      float dmax = 0.f;
      if (lane == 0) sm.dl[buf][warp] = 0.f;
      __syncthreads();
      int s = 0;
      float delta = 0.f;
      for (;;) {
        if (threadIdx.x < kS) {   // the kW warp partials of column t (conflict-free rows)
          float c0 = 0.f, c1 = 0.f;
#pragma unroll
          for (int w = 0; w < kW; w += 2) {
            c0 += colp[buf][w][threadIdx.x];
            c1 += colp[buf][w + 1][threadIdx.x];
          }
          sm.csum[threadIdx.x] = c0 + c1;
        }
        __syncthreads();
        const float4 cs4 = *reinterpret_cast<const float4*>(&sm.csum[4 * lane]);
        const float4 rs_lo = *reinterpret_cast<const float4*>(&sm.rsum[buf][warp][0]);
        const float4 rs_hi = *reinterpret_cast<const float4*>(&sm.rsum[buf][warp][4]);
        const float sigma = warp_sum((cs4.x + cs4.y) + (cs4.z + cs4.w));
        const float tconst = (1.0f + sigma * inv_m) * inv_m;
        const float2 inv2 = make_float2(-inv_m, -inv_m);
        const float2 ncu01 = __fmul2_rn(make_float2(cs4.x, cs4.y), inv2);   // -c_j / m
        const float2 ncu23 = __fmul2_rn(make_float2(cs4.z, cs4.w), inv2);
        const float rsr[8] = {rs_lo.x, rs_lo.y, rs_lo.z, rs_lo.w, rs_hi.x, rs_hi.y, rs_hi.z, rs_hi.w};
        buf ^= 1;
        dmax = 0.f;
#pragma unroll
        for (int r = 0; r < kRW; ++r) {
          const int i = warp * kRW + r;
          const float ti = tconst - rsr[r] * inv_m;
          const float2 t2 = make_float2(ti, ti);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 yo = y[r][h];
            float2 z = __fadd2_rn(__fadd2_rn(yo, t2), h ? ncu23 : ncu01);    // P1: (y + t_i) - c_j/m
            z.x = fmaxf(z.x, 0.f);                                            // P2
            z.y = fmaxf(z.y, 0.f);
            if (!kFull) {
              const int j = 4 * lane + 2 * h;
              if (!(i < m && j < m)) z.x = 0.f;
              if (!(i < m && j + 1 < m)) z.y = 0.f;
            }
            if (kDelta) dmax = fmaxf(dmax, fmaxf(fabsf(z.x - yo.x), fabsf(z.y - yo.y)));
            y[r][h] = z;
          }
        }
        sums(y);
        if (kDelta) {
          dmax = warp_max(dmax);
          if (lane == 0) sm.dl[buf][warp] = dmax;
        }
        __syncthreads();
        delta = 0.f;
        if (kDelta) {
#pragma unroll
          for (int w = 0; w < kW; ++w) delta = fmaxf(delta, sm.dl[buf][w]);
        }
        ++s;
        if (delta < p.eps2 || s >= p.max_iter2) break;
      }
      total_sweeps += s;
      SSP(4);

      // ---- blend + rescale (lines 8-9) on X (registers), row maxima for the next X digits
      float2 xt[kRW][2];
      float rmx[kRW];
      const float2 a2 = make_float2(p.alpha, p.alpha), b2 = make_float2(1.0f - p.alpha, 1.0f - p.alpha);
#pragma unroll
      for (int r = 0; r < kRW; ++r) {
        const int i = warp * kRW + r;
        rmx[r] = 0.f;                         // X~ >= 0: 0 is the identity of the max
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          xt[r][h] = __ffma2_rn(a2, y[r][h], __fmul2_rn(b2, xr[r][h]));
          if (kFull) {
            rmx[r] = fmaxf(rmx[r], fmaxf(xt[r][h].x, xt[r][h].y));
          } else {
            const int j = 4 * lane + 2 * h;
            if (i < n && j < np) rmx[r] = fmaxf(rmx[r], xt[r][h].x);
            if (i < n && j + 1 < np) rmx[r] = fmaxf(rmx[r], xt[r][h].y);
          }
        }
      }
      rows_allmax(rmx);
      float mu = rmx[0];
#pragma unroll
      for (int r = 1; r < kRW; ++r) mu = fmaxf(mu, rmx[r]);
      if (lane == 0) sm.red[warp] = mu;
      __syncthreads();
      mu = 0.f;
#pragma unroll
      for (int w = 0; w < kW; ++w) mu = fmaxf(mu, sm.red[w]);
      __syncthreads();
      if (!(mu > 1e-30f)) { degen = 1; break; }   // degenerate guard (reading A7), X unchanged
      // X / max X as a product with the reciprocal (<= 1 ulp from the quotient)
      const float inv_scale = p.rescale ? 1.0f / mu : 1.0f;
      float rl = 0.f;
      const float2 is2 = make_float2(inv_scale, inv_scale);
#pragma unroll
      for (int r = 0; r < kRW; ++r) {
        const int i = warp * kRW + r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 xn = __fmul2_rn(xt[r][h], is2);
          const int j = 4 * lane + 2 * h;
          if (kFull || (i < n && j < np)) {
            rl = fmaxf(rl, fabsf(xn.x - xr[r][h].x));
            xr[r][h].x = xn.x;
          }
          if (kFull || (i < n && j + 1 < np)) {
            rl = fmaxf(rl, fabsf(xn.y - xr[r][h].y));
            xr[r][h].y = xn.y;
          }
        }
      }
      SSP(6);
      // digits of the new X for the next GEMM1; row max of X = (row max of X~) / scale (rounding
      // and the division are monotonic, so this is the max of the stored values)
      {
#pragma unroll
        for (int r = 0; r < kRW; ++r) {
          const int row = warp * kRW + r;
          const int e = frexp_exp(rmx[r] * inv_scale);
          if (lane == 0) sm.eW[row] = e;
          int w1, w2, w3;
          const float v4[4] = {xr[r][0].x, xr[r][0].y, xr[r][1].x, xr[r][1].y};
          digits4(v4, exp2i(-e), w1, w2, w3);   // columns 4 lane .. 4 lane + 3: packed
          const int o = swz(row, 4 * lane);
          *reinterpret_cast<int*>(&sm.Wd[0][o]) = w1;
          *reinterpret_cast<int*>(&sm.Wd[1][o]) = w2;
          *reinterpret_cast<int*>(&sm.Wd[2][o]) = w3;
        }
      }
      rl = warp_max(rl);
      if (lane == 0) sm.red[warp] = rl;
      __syncthreads();
      rho = 0.f;
#pragma unroll
      for (int w = 0; w < kW; ++w) rho = fmaxf(rho, sm.red[w]);
      __syncthreads();
      ++it;
      SSP(5);
      if (rho < p.eps1) { conv = 1; break; }
    }
#ifdef FPFP_SS_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0 && pair == 0)
      printf("ss-prof pair 0: per outer (clk): gemm1 %lld  U-epi+digits %lld  gemm2 %lld  G-epi+stage %lld  sweeps %lld  blend %lld  X-digits+rho %lld\n",
             tp[0] / it, tp[1] / it, tp[2] / it, tp[3] / it, tp[4] / it, tp[6] / it, tp[5] / it);
#endif

    // write back X (and Y when slack exists)
#pragma unroll
    for (int r = 0; r < kRW; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = warp * kRW + r, j = 4 * lane + e;
        if (i < n && j < np) X[(int64_t)i * np + j] = el(xr[r], e);
      }
    if (p.Y) {
#pragma unroll
      for (int r = 0; r < kRW; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = warp * kRW + r, j = 4 * lane + e;
          if (i < m && j < m) p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] = el(y[r], e);
        }
    }
    if (threadIdx.x == 0) {
      p.iters[pair] = it; p.conv[pair] = conv; p.sweeps[pair] = total_sweeps;
      p.rho[pair] = rho; p.degen[pair] = degen;
    }
    __syncthreads();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

size_t small_tc_smem_bytes() { return sizeof(SmemTC) + 1024; }

cudaError_t launch_small_solve_tc(const SmallArgs& a, int grid, cudaStream_t s) {
  const bool full = a.n == kS && a.np == kS;
  const bool delta = a.eps2 > 0.0f;
  void (*k)(SmallArgs) = full ? (delta ? small_solve_tc_kernel<true, true> : small_solve_tc_kernel<true, false>)
                              : (delta ? small_solve_tc_kernel<false, true> : small_solve_tc_kernel<false, false>);
  const int bytes = (int)small_tc_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  k<<<grid, kT, bytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fpfp
