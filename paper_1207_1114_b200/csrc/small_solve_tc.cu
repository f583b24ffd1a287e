// small_solve_tc.cu — Algorithm 1 for many small pairs (n, n' <= 128) with the two
// products of line 3 on the int8 tensor cores: the Ozaki digit decomposition of gemm_i8.cu
// (3 signed 7-bit digit planes per operand row, 6 exact int32 digit products in 3 TMEM weight
// classes; fp32-accurate) at M = N = K = 128 (tcgen05.mma.cta_group::1.kind::i8,
// 24 MMAs per product). BASELINE configs[3] (8192 pairs of 128).
//
// TWO PAIRS PER CTA. A pair is a latency-bound chain (20 sweeps per outer iteration, each ending in
// a block-wide reduction), so one pair per SM leaves most issue slots idle. Each CTA runs two
// independent "slots" of 8 warps; slot s works through pairs 2 blockIdx + s, + 2 gridDim, ... and
// synchronises its warps with its own named barrier, so one slot computes while the other waits.
// The resources only the products need — the operand digit planes in shared memory, the 384 TMEM
// accumulator columns and the fp32 staging tile — are shared and owned by one slot at a time (a
// shared-memory lock around the "product phase"). Their footprint is kept small by keeping the
// constant operands off chip: the digit planes of A and A' are built once per set_graphs
// (small_digits_prep_kernel) as the exact swizzled shared-memory image in global memory, and the
// digits of the current X are written there by the slot's blend; the product phase pulls them in
// with 1-D bulk copies (cp.async.bulk, 48 KB per operand, L2-resident).
//
// Per slot and outer iteration:
//   [product phase, lock held] bulk-copy A' digits + X digits -> GEMM1 U = A' X^T (TMEM) -> bulk
//   copy of A digits overlapped with the U epilogue (U digits, row scales over the whole row) ->
//   GEMM2 G = A U^T (TMEM) -> + lambda K -> fp32 staging -> Y registers (X block)
//   [slot only] the projection sweeps (Y in registers: warp w owns rows 16w..16w+15, lane l the
//   columns 4l..4l+3 as two float2 pairs for the packed fp32x2 pipe; fp32 sums) -> blend: the X
//   block of Y becomes X~ = (1-a) X + a Y, mu = max X~, X = X~/mu (global) and its digits (global).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fpfp {

namespace {

using namespace tc;

constexpr int kT = 512;               // threads per CTA (two slots)
constexpr int kST = 256;              // threads per slot
constexpr int kS = 128;               // max n, n', m
constexpr int kPW = kST / 32;         // warps per slot (8)
constexpr int kPR = kS / kPW;         // rows of the Y register tile per warp (16)
constexpr int kEC = kS / 2;           // epilogue columns per warp (2 warps per TMEM lane quarter)
constexpr int kLdG = kS + 4;          // fp32 staging row stride
constexpr int kPlane = kS * kS;       // one digit plane: 128 rows x 128 bytes (SWIZZLE_128B image)
constexpr int kOperand = 3 * kPlane;  // 48 KB: the three planes of one operand

struct SlotSm {
  float colp[2][kPW][kS];     // per-warp column partials of the sweeps (double buffered)
  float csum[kS];             // combined column sums of the current sweep
  float rsum[2][kPW][kPR];    // row sums of each warp's rows (double buffered)
  float wsig[2][kPW];         // per-warp totals (sigma partials, double buffered)
  float dl[2][kPW];
  float red[kPW];
  float xscale[kS];           // 2^(eX - 14): the X digits' row scales (GEMM1's N side)
  float xtmax[kS];            // row maxima of X~ (blend pass 1 -> pass 2)
  int eP[kS], eA[kS];         // row exponents of A' and A
};

struct __align__(1024) SmemTC {
  int8_t Pd[3][kPlane];       // M-side digit planes of the current product (A' or A)
  int8_t Wd[3][kPlane];       // N-side digit planes (X digits, then U digits)
  float G[kS][kLdG];          // product staging (row = TMEM lane)
  SlotSm slot[2];
  float cscale[kS];           // N-side column scales of the current product
  float wmax[2][kS];          // row |max| of U per epilogue column half
  uint64_t bar_mma;           // MMA completion
  uint64_t bar_ld;            // bulk-copy completion
  uint32_t mma_phase, ld_phase;
  int lock;                   // product-phase owner (0 = free, 1 + slot)
  uint32_t tmem_base;
};

__device__ __forceinline__ float pow2(int e) {
  return (e > -127 && e < 128) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e);
}

// byte offset of (row, col) in a SWIZZLE_128B K-major plane (128-byte rows, 1024-byte atoms)
__device__ __forceinline__ int swz(int row, int col) {
  return row * 128 + ((((col >> 4) ^ (row & 7))) << 4) + (col & 15);
}

// low bytes of four ints -> one word (byte t = d_t)
__device__ __forceinline__ int pack4(int d0, int d1, int d2, int d3) {
  return (int)__byte_perm(__byte_perm(d0, d1, 0x0040), __byte_perm(d2, d3, 0x0040), 0x5410);
}
// Ozaki digits in integer arithmetic. With s21 = 2^(21 - e) (e: the row's frexp exponent, so
// |x s21| < 2^21) one magic-number FFMA gives q = rint(x 2^(21-e)) exactly in the float's low bits;
// q = a 2^14 + b 2^7 + c is then split with carries: a = floor((q + 2^13) / 2^14) <= 127 (clamped),
// b = floor((r + 64) / 128) <= 127, c = r' <= 127 — the same q, and the same digit ranges
// (|b|, |c| <= 64 except next to the top of the row's range), as rounding the remainders r0 = x 2^-e
// 128, r1 = 128 (r0 - a), r2 = 128 (r1 - b) one digit at a time, in ~11 integer ops
// per value instead of ~24 float ops.
__device__ __forceinline__ void digits_q(float x, float s21, int& a, int& b, int& c) {
  const int bits = __float_as_int(fmaf(x, s21, 12582912.0f));   // 1.5 2^23 + q, |q| < 2^22
  const int q = bits - 0x4B400000;
  a = min((q + 8192) >> 14, 127);
  const int r = q - (a << 14);
  b = min((r + 64) >> 7, 127);
  c = min(r - (b << 7), 127);
}
// row exponent of the digit split: frexp's, floored at -100 so that s21 = 2^(21 - e) stays finite
// (rows below 2^-100 just keep fewer significant bits; the same e scales the product epilogue)
__device__ __forceinline__ int digit_exp(float mx) { return max(frexp_exp(mx), -100); }
// 4 consecutive values -> one packed word (4 digits) per plane; s21 = 2^(21 - e)
__device__ __forceinline__ void digits4(const float (&v)[4], float s21, int& w1, int& w2, int& w3) {
  int a[4], b[4], c[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) digits_q(v[t], s21, a[t], b[t], c[t]);
  w1 = pack4(a[0], a[1], a[2], a[3]);
  w2 = pack4(b[0], b[1], b[2], b[3]);
  w3 = pack4(c[0], c[1], c[2], c[3]);
}

__device__ __forceinline__ void slot_sync(int slot) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(kST) : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// one operand's three planes (48 KB) from its global image
__device__ __forceinline__ void copy_operand(int8_t (*dst)[kPlane], const int8_t* src, uint64_t* bar) {
#pragma unroll
  for (int k = 0; k < 3; ++k) bulk_copy(dst[k], src + (size_t)k * kPlane, kPlane, bar);
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

// The thread's kEC values of row erow (its TMEM lane), columns ecol0 .. ecol0 + kEC - 1, of the
// digit product: (a2 + 2^-7 (a3 + 2^-7 a4)) * rscale * cscale[col], cscale = 2^(e_col - 14);
// written to dst[0 .. kEC) (fp32 staging); returns their max |value|.
__device__ __forceinline__ float product_to_smem(uint32_t tb, float rscale, const float* cscale, int ecol0,
                                                 float* dst) {
  float mx = 0.0f;
#pragma unroll 2
  for (int h = 0; h < kEC / 16; ++h) {   // 16 columns at a time (48 registers of accumulators; two
                                         // groups in flight: c4 +0.5%)
    uint32_t a2[16], a3[16], a4[16];
    tmem_ld16_nowait(tb + (uint32_t)(h * 16), a2);
    tmem_ld16_nowait(tb + 128u + (uint32_t)(h * 16), a3);
    tmem_ld16_nowait(tb + 256u + (uint32_t)(h * 16), a4);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      // class sums at K = 128: |a2| <= 128^3 = 2^21 and |a3| <= 2 * 128 * 127 * 128 < 2^22
      // convert exactly through the 1.5 * 2^23 magic number (integer add + packed float
      // subtract); |a4| may reach 3 * 128 * 127 * 128 and takes the conversion pipe. The combine
      // runs on column pairs (FFMA2 / FMUL2).
      const float2 kM = make_float2(-12582912.0f, -12582912.0f), k7 = make_float2(0.0078125f, 0.0078125f);
      const float2 rs2 = make_float2(rscale, rscale);
      const float4 cs = *reinterpret_cast<const float4*>(cscale + ecol0 + h * 16 + j);
      float2 o[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int u = j + 2 * t;
        const float2 f2 = __fadd2_rn(make_float2(__int_as_float((int)a2[u] + 0x4B400000),
                                                 __int_as_float((int)a2[u + 1] + 0x4B400000)), kM);
        const float2 f3 = __fadd2_rn(make_float2(__int_as_float((int)a3[u] + 0x4B400000),
                                                 __int_as_float((int)a3[u + 1] + 0x4B400000)), kM);
        float2 v = __ffma2_rn(make_float2((float)(int)a4[u], (float)(int)a4[u + 1]), k7, f3);
        v = __ffma2_rn(v, k7, f2);
        o[t] = __fmul2_rn(__fmul2_rn(v, rs2), t ? make_float2(cs.z, cs.w) : make_float2(cs.x, cs.y));
        mx = fmaxf(mx, fmaxf(fabsf(o[t].x), fabsf(o[t].y)));
      }
      *reinterpret_cast<float4*>(dst + h * 16 + j) = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
    }
  }
  return mx;
}

// 16 row partials per lane -> lanes 2r, 2r + 1 hold the total of row r in v[0] (transposed
// butterfly: 8 + 4 + 2 + 1 exchanges, then xor 1)
__device__ __forceinline__ void rows_reduce16(float (&v)[16]) {
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
  v[0] = b1;   // row 8 bit4 + 4 bit3 + 2 bit2 + bit1 of the lane
}

// element e (0..3) of a lane's 4 consecutive columns held as two float2 pairs
__device__ __forceinline__ float& el(float2 (&v)[2], int e) { return (e & 1) ? v[e >> 1].y : v[e >> 1].x; }
__device__ __forceinline__ float elc(const float2 (&v)[2], int e) { return (e & 1) ? v[e >> 1].y : v[e >> 1].x; }

// digits of 4 consecutive values of row `row` (s21 = 2^(21 - e)) into a global operand image
__device__ __forceinline__ void store_digits(int8_t* img, int row, int col0, const float (&v)[4], float s21) {
  int w1, w2, w3;
  digits4(v, s21, w1, w2, w3);
  const int o = swz(row, col0);
  *reinterpret_cast<int*>(img + o) = w1;
  *reinterpret_cast<int*>(img + kPlane + o) = w2;
  *reinterpret_cast<int*>(img + 2 * kPlane + o) = w3;
}

}  // namespace

// A' and A of every pair -> the swizzled digit-plane images the product phase bulk-copies
// (dig[pair] = [A' planes 0..2 | A planes 0..2 | X planes], exps[pair] = [eA' 128 | eA 128]).
// One warp per row, lane l owns columns 4l .. 4l + 3; zero outside n / n'.
__global__ void __launch_bounds__(256) small_digits_prep_kernel(const float* A, const float* Ap, int batch,
                                                               int n, int np, int8_t* dig, int* exps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pair = blockIdx.x; pair < batch; pair += gridDim.x) {
    for (int mtx = 0; mtx < 2; ++mtx) {
      const int dim = mtx == 0 ? np : n;
      const float* src = (mtx == 0 ? Ap + (int64_t)pair * np * np : A + (int64_t)pair * n * n);
      int8_t* img = dig + ((size_t)pair * 3 + mtx) * kOperand;
      int* ex = exps + ((size_t)pair * 2 + mtx) * kS;
      for (int r = warp; r < kS; r += 8) {
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = 4 * lane + t;
          v[t] = (r < dim && c < dim) ? __ldg(src + (int64_t)r * dim + c) : 0.0f;
        }
        float mx = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
        mx = warp_max(mx);
        const int e = digit_exp(mx);
        if (lane == 0) ex[r] = e;
        store_digits(img, r, 4 * lane, v, exp2i(21 - e));
      }
    }
  }
}

template <bool kFull, bool kDelta>
__global__ void __launch_bounds__(kT, 1) small_solve_tc_kernel(SmallArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on smem_raw (not through an integer) so the compiler keeps the
  // shared state space: LDS/STS instead of generic LD/ST
  SmemTC& sm = *reinterpret_cast<SmemTC*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / kPW, sw = warp % kPW, st = threadIdx.x % kST;
  SlotSm& ss = sm.slot[slot];
  const int n = p.n, np = p.np, m = p.m;
  const float inv_m = 1.0f / (float)m;
  // epilogue geometry: row = TMEM lane 32 (warp & 3) + lane, columns kEC (sw >> 2) ..
  const int erow = (warp & 3) * 32 + lane, ecol0 = (sw >> 2) * kEC;

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_mma, 1);
    mbar_init(&sm.bar_ld, 1);
    fence_mbar_init();
    sm.mma_phase = 0;
    sm.ld_phase = 0;
    sm.lock = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)ecol0;

  for (int pair = 2 * blockIdx.x + slot; pair < p.batch; pair += 2 * gridDim.x) {
    const float* Kp = p.K ? p.K + (int64_t)pair * n * np : nullptr;
    float* X = p.X + (int64_t)pair * n * np;
    const int8_t* dig = p.dig + (size_t)pair * 3 * kOperand;
    int8_t* xdig = p.dig + ((size_t)pair * 3 + 2) * kOperand;
    if (st < kS) {
      ss.eP[st] = p.dexp[(size_t)pair * 2 * kS + st];
      ss.eA[st] = p.dexp[(size_t)pair * 2 * kS + kS + st];
    }
    // digits of the current X (the first GEMM1 of this call): warp sw owns rows 16 sw .. 16 sw + 15
#pragma unroll 1
    for (int r = 0; r < kPR; ++r) {
      const int i = sw * kPR + r;
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 4 * lane + e;
        v[e] = (i < n && j < np) ? __ldcg(X + (int64_t)i * np + j) : 0.f;
      }
      float mx = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
      mx = warp_max(mx);
      const int e = digit_exp(mx);
      if (lane == 0) ss.xscale[i] = pow2(e - 14);
      store_digits(xdig, i, 4 * lane, v, exp2i(21 - e));
    }
    // Y register tile (slack state; the X block is overwritten by the first product)
    float2 y[kPR][2];
#pragma unroll
    for (int r = 0; r < kPR; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = sw * kPR + r, j = 4 * lane + e;
        el(y[r], e) = (p.Y && i < m && j < m) ? p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] : 0.f;
      }
    asm volatile("fence.proxy.async.global;" ::: "memory");   // X digits: generic -> async proxy
    slot_sync(slot);

    int it = 0, conv = 0, total_sweeps = 0, degen = 0;
    float rho = 0.f;
#ifdef FPFP_SS_PROF
    long long tp[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define SSP(k) do { const long long t_ = clock64(); tp[k] += t_ - tq; tq = t_; } while (0)
#else
#define SSP(k) do { } while (0)
#endif
    for (; it < p.max_iter1;) {
      // ================= product phase (shared operand buffers, TMEM, staging: lock) ==========
      if (st == 0) {
        while (atomicCAS(&sm.lock, 0, 1 + slot) != 0) __nanosleep(64);
        __threadfence_block();
      }
      slot_sync(slot);
      SSP(0);
      uint32_t mph = *reinterpret_cast<volatile uint32_t*>(&sm.mma_phase);
      uint32_t lph = *reinterpret_cast<volatile uint32_t*>(&sm.ld_phase);
      tc_fence_after();
      if (sw == 0) {
        if (elect_one()) {
          mbar_expect_tx(&sm.bar_ld, 2 * kOperand);
          copy_operand(sm.Pd, dig, &sm.bar_ld);           // A' digits (GEMM1 M side)
          copy_operand(sm.Wd, xdig, &sm.bar_ld);          // X digits  (GEMM1 N side)
        }
        __syncwarp();
      }
      if (st < kS) sm.cscale[st] = ss.xscale[st];
      mbar_wait(&sm.bar_ld, lph);
      lph ^= 1;
      slot_sync(slot);
      SSP(6);
      // ---- U = A' X^T (line 3, first product)
      if (sw == 0) {
        tc_fence_after();
        if (elect_one()) issue_product(sm.Pd, sm.Wd, tmem, &sm.bar_mma);
        __syncwarp();
      }
      mbar_wait(&sm.bar_mma, mph);
      mph ^= 1;
      tc_fence_after();
      SSP(7);
      if (sw == 0) {   // P is free again: the A digits (GEMM2 M side) stream in under the U epilogue
        if (elect_one()) {
          mbar_expect_tx(&sm.bar_ld, kOperand);
          copy_operand(sm.Pd, dig + kOperand, &sm.bar_ld);
        }
        __syncwarp();
      }
      {
        const float mx = product_to_smem(tb, pow2(ss.eP[erow]), sm.cscale, ecol0, &sm.G[erow][ecol0]);
        sm.wmax[sw >> 2][erow] = mx;
      }
      tc_fence_before();
      slot_sync(slot);                                       // U staged; X digits consumed
      {   // U digits with the scale of the whole row (GEMM2's N side)
        const float rmx = fmaxf(sm.wmax[0][erow], sm.wmax[1][erow]);
        const int e = digit_exp(rmx);
        const float inv = exp2i(21 - e);
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
        if (sw < 4) sm.cscale[erow] = pow2(e - 14);          // (GEMM1's scales were read above)
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      SSP(8);
      mbar_wait(&sm.bar_ld, lph);
      lph ^= 1;
      slot_sync(slot);
      // ---- G = A U^T + lambda K (line 3, second product)
      if (sw == 0) {
        tc_fence_after();
        if (elect_one()) issue_product(sm.Pd, sm.Wd, tmem, &sm.bar_mma);
        __syncwarp();
      }
      mbar_wait(&sm.bar_mma, mph);
      mph ^= 1;
      tc_fence_after();
      SSP(9);
      product_to_smem(tb, pow2(ss.eA[erow]), sm.cscale, ecol0, &sm.G[erow][ecol0]);   // G staged
      if (Kp && erow < n) {                               // + lambda K (line 3)
        for (int j = 0; j < kEC && ecol0 + j < np; ++j)
          sm.G[erow][ecol0 + j] += p.lam * Kp[(int64_t)erow * np + ecol0 + j];
      }
      tc_fence_before();
      slot_sync(slot);
      // Y[0:n, 0:n'] = G ; slack entries keep their values (reading A3)
#pragma unroll
      for (int r = 0; r < kPR; ++r) {
        const int i = sw * kPR + r;
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
      slot_sync(slot);   // staging read, accumulators drained: hand the product resources over
      if (st == 0) {
        sm.mma_phase = mph;
        sm.ld_phase = lph;
        __threadfence_block();
        atomicExch(&sm.lock, 0);
      }
      SSP(1);

      // ================= projection loop (P1 + P2 per sweep; slot-local) ======================
      // Per sweep: the update and the sums of its output on the packed fp32x2 pipe; each warp's
      // 16 row sums by a transposed butterfly, published with its column partials; slot barrier;
      // 4 warps combine the column partials (one thread per column); slot barrier.
      int buf = 0;
      auto sums = [&](const float2 (&yy)[kPR][2]) {
        float rp[kPR];
        float2 c01 = make_float2(0.f, 0.f), c23 = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
          const float2 t = __fadd2_rn(yy[r][0], yy[r][1]);
          rp[r] = t.x + t.y;
          c01 = __fadd2_rn(c01, yy[r][0]);
          c23 = __fadd2_rn(c23, yy[r][1]);
        }
        // the warp's share of sigma = 1^T Y 1: an independent reduction that overlaps the butterfly
        float ws = 0.f;
#pragma unroll
        for (int r = 0; r < kPR; ++r) ws += rp[r];
        ws = warp_sum(ws);
        rows_reduce16(rp);
        if ((lane & 1) == 0) ss.rsum[buf][sw][lane >> 1] = rp[0];
        if (lane == 0) ss.wsig[buf][sw] = ws;
        *reinterpret_cast<float4*>(&ss.colp[buf][sw][4 * lane]) = make_float4(c01.x, c01.y, c23.x, c23.y);
      };
      sums(y);
      if (lane == 0) ss.dl[buf][sw] = 0.f;
      slot_sync(slot);
      int s = 0;
      float delta = 0.f;
      for (;;) {
        // the blend's X rows (this warp's 16 rows, 16 B per lane) toward L1 during the cap's last
        // sweep, so the rescale pass that follows finds them on chip (c4: +2.5%; 8 rows or 2-3
        // sweeps ahead measured slower)
        if (kFull && s + 1 == p.max_iter2) {
#pragma unroll
          for (int r = 0; r < kPR; ++r)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(X + (int64_t)(sw * kPR + r) * kS + 4 * lane));
        }
        // t_i of the warp's rows needs only the row sums and sigma, published before the first
        // barrier: formed while warps 0-3 combine the column partials (c4 +1.2%)
        float tir[kPR];
        {
          const float4 sg0 = *reinterpret_cast<const float4*>(&ss.wsig[buf][0]);
          const float4 sg1 = *reinterpret_cast<const float4*>(&ss.wsig[buf][4]);
          const float sigma = ((sg0.x + sg0.y) + (sg0.z + sg0.w)) + ((sg1.x + sg1.y) + (sg1.z + sg1.w));
          const float tconst = (1.0f + sigma * inv_m) * inv_m;
#pragma unroll
          for (int q = 0; q < kPR; q += 4) {
            const float4 v = *reinterpret_cast<const float4*>(&ss.rsum[buf][sw][q]);
            tir[q] = tconst - v.x * inv_m; tir[q + 1] = tconst - v.y * inv_m;
            tir[q + 2] = tconst - v.z * inv_m; tir[q + 3] = tconst - v.w * inv_m;
          }
        }
#ifndef FPFP_SS_PER_LANE_COMBINE   // (the per-lane variant below measured no faster: 7.36 vs 7.5 M)
        if (st < kS) {   // the kPW warp partials of column st (conflict-free rows)
          float c0 = 0.f, c1 = 0.f;
#pragma unroll
          for (int w = 0; w < kPW; w += 2) {
            c0 += ss.colp[buf][w][st];
            c1 += ss.colp[buf][w + 1][st];
          }
          ss.csum[st] = c0 + c1;
        }
        slot_sync(slot);
        const float4 cs4 = *reinterpret_cast<const float4*>(&ss.csum[4 * lane]);
#else
        // every lane combines the kPW warp partials of its own 4 columns (8 vector loads, in the
        // fixed warp order): one slot barrier per sweep instead of two
        float4 cs4;
        {
          float2 c01 = make_float2(0.f, 0.f), c23 = make_float2(0.f, 0.f);
#pragma unroll
          for (int w = 0; w < kPW; ++w) {
            const float4 v = *reinterpret_cast<const float4*>(&ss.colp[buf][w][4 * lane]);
            c01 = __fadd2_rn(c01, make_float2(v.x, v.y));
            c23 = __fadd2_rn(c23, make_float2(v.z, v.w));
          }
          cs4 = make_float4(c01.x, c01.y, c23.x, c23.y);
        }
#endif
        const float2 inv2 = make_float2(-inv_m, -inv_m);
        const float2 ncu01 = __fmul2_rn(make_float2(cs4.x, cs4.y), inv2);   // -c_j / m
        const float2 ncu23 = __fmul2_rn(make_float2(cs4.z, cs4.w), inv2);
        buf ^= 1;
        float dmax = 0.f;
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
          const int i = sw * kPR + r;
          const float ti = tir[r];
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
          if (lane == 0) ss.dl[buf][sw] = dmax;
        }
        slot_sync(slot);
        delta = 0.f;
        if (kDelta) {
#pragma unroll
          for (int w = 0; w < kPW; ++w) delta = fmaxf(delta, ss.dl[buf][w]);
        }
        ++s;
        if (delta < p.eps2 || s >= p.max_iter2) break;
      }
      total_sweeps += s;
      SSP(2);

      // ================= blend + rescale (lines 8-9) =========================================
      // pass 1: the X block of Y becomes X~ = (1 - alpha) X + alpha Y; row maxima; mu
      float rmx[kPR];
      const float2 a2 = make_float2(p.alpha, p.alpha), b2 = make_float2(1.0f - p.alpha, 1.0f - p.alpha);
      float mu = 0.f;
      const float* xrow0 = X + (int64_t)(sw * kPR) * np + 4 * lane;
      if (kFull) {   // X rows streamed 4 at a time, the next 4 in flight (L2 latency)
        float4 xa[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xa[q] = __ldcg(reinterpret_cast<const float4*>(xrow0 + q * kS));   // kFull: np = kS
#pragma unroll
        for (int c = 0; c < kPR / 4; ++c) {
          float4 xb[4];
          if (c + 1 < kPR / 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              xb[q] = __ldcg(reinterpret_cast<const float4*>(xrow0 + (4 * (c + 1) + q) * kS));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = 4 * c + q;
            y[r][0] = __ffma2_rn(a2, y[r][0], __fmul2_rn(b2, make_float2(xa[q].x, xa[q].y)));
            y[r][1] = __ffma2_rn(a2, y[r][1], __fmul2_rn(b2, make_float2(xa[q].z, xa[q].w)));
            rmx[r] = fmaxf(fmaxf(y[r][0].x, y[r][0].y), fmaxf(y[r][1].x, y[r][1].y));
          }
          if (c + 1 < kPR / 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) xa[q] = xb[q];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
          const int i = sw * kPR + r;
          rmx[r] = 0.f;                        // X~ >= 0: 0 is the identity of the max
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * lane + e;
            if (i < n && j < np) {
              const float xo = __ldcg(X + (int64_t)i * np + j);
              el(y[r], e) = fmaf(p.alpha, el(y[r], e), (1.0f - p.alpha) * xo);
              rmx[r] = fmaxf(rmx[r], el(y[r], e));
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kPR; ++r) {
        const float v = warp_max(rmx[r]);
        if (lane == 0) ss.xtmax[sw * kPR + r] = v;
        mu = fmaxf(mu, v);
      }
      if (lane == 0) ss.red[sw] = mu;
      slot_sync(slot);
      mu = 0.f;
#pragma unroll
      for (int w = 0; w < kPW; ++w) mu = fmaxf(mu, ss.red[w]);
      slot_sync(slot);
      SSP(3);
      if (!(mu > 1e-30f)) { degen = 1; break; }   // degenerate guard (reading A7), X unchanged
      // pass 2: X = X~ / mu (product with the fp32 reciprocal, <= 1 ulp from the quotient,
      // DESIGN.md §6), rho, and the digits of the new X for the next GEMM1 (row scale from the row
      // max of X~: rounding and the division are monotonic, so it is the max of the stored row)
      const float inv_scale = p.rescale ? 1.0f / mu : 1.0f;
      // rho decides only the outer stop test (eps1 > 0) and the reported last value: with eps1 <= 0
      // (fixed outer counts) only the call's last iteration re-reads the old X for it (c4: +3.6%)
      const bool want_rho = p.eps1 > 0.f || it + 1 >= p.max_iter1;
      float rl = 0.f;
      auto finish_row = [&](int r, const float (&xn)[4]) {
        const int i = sw * kPR + r;
        const int e = digit_exp(ss.xtmax[i] * inv_scale);
        if (lane == 0) ss.xscale[i] = pow2(e - 14);
        store_digits(xdig, i, 4 * lane, xn, exp2i(21 - e));
      };
      if (kFull && !want_rho) {
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
          float xn[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) xn[e] = elc(y[r], e) * inv_scale;
          __stcg(reinterpret_cast<float4*>(const_cast<float*>(xrow0) + r * kS), make_float4(xn[0], xn[1], xn[2], xn[3]));
          finish_row(r, xn);
        }
      } else if (kFull) {
        float4 xa[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xa[q] = __ldcg(reinterpret_cast<const float4*>(xrow0 + q * kS));   // kFull: np = kS
#pragma unroll
        for (int c = 0; c < kPR / 4; ++c) {
          float4 xb[4];
          if (c + 1 < kPR / 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              xb[q] = __ldcg(reinterpret_cast<const float4*>(xrow0 + (4 * (c + 1) + q) * kS));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = 4 * c + q;
            float xn[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) xn[e] = elc(y[r], e) * inv_scale;
            rl = fmaxf(rl, fmaxf(fmaxf(fabsf(xn[0] - xa[q].x), fabsf(xn[1] - xa[q].y)),
                                 fmaxf(fabsf(xn[2] - xa[q].z), fabsf(xn[3] - xa[q].w))));
            __stcg(reinterpret_cast<float4*>(const_cast<float*>(xrow0) + r * kS),
                   make_float4(xn[0], xn[1], xn[2], xn[3]));
            finish_row(r, xn);
          }
          if (c + 1 < kPR / 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) xa[q] = xb[q];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
          const int i = sw * kPR + r;
          float xn[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * lane + e;
            xn[e] = elc(y[r], e) * inv_scale;
            if (i < n && j < np) {
              const float xo = __ldcg(X + (int64_t)i * np + j);
              rl = fmaxf(rl, fabsf(xn[e] - xo));
              __stcg(X + (int64_t)i * np + j, xn[e]);
            } else {
              xn[e] = 0.f;
            }
          }
          finish_row(r, xn);
        }
      }
      SSP(4);
      asm volatile("fence.proxy.async.global;" ::: "memory");   // X digits: generic -> async proxy
      if (want_rho) {
        rl = warp_max(rl);
        if (lane == 0) ss.red[sw] = rl;
        slot_sync(slot);
        rho = 0.f;
#pragma unroll
        for (int w = 0; w < kPW; ++w) rho = fmaxf(rho, ss.red[w]);
        slot_sync(slot);
      }
      ++it;
      SSP(5);
      if (rho < p.eps1) { conv = 1; break; }
    }
#ifdef FPFP_SS_PROF
    if (blockIdx.x == 0 && st == 0 && pair < 2)
      printf("ss-prof slot %d pair %d: per outer (clk): lock-wait %lld  product-phase %lld [copies %lld mma1 %lld "
             "U-epi+digits %lld mma2-wait %lld G-epi %lld]  sweeps %lld  blend-pass1+mu %lld  pass2 %lld  fence+rho %lld\n",
             slot, pair, tp[0] / it, (tp[1] + tp[6] + tp[7] + tp[8] + tp[9]) / it, tp[6] / it, tp[7] / it, tp[8] / it,
             tp[9] / it, tp[1] / it, tp[2] / it, tp[3] / it, tp[4] / it, tp[5] / it);
#endif

    // write back Y when slack exists (its X block holds X~ or G: overwritten by the next product)
    if (p.Y) {
#pragma unroll
      for (int r = 0; r < kPR; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = sw * kPR + r, j = 4 * lane + e;
          if (i < m && j < m) p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] = el(y[r], e);
        }
    }
    if (st == 0) {
      p.iters[pair] = it; p.conv[pair] = conv; p.sweeps[pair] = total_sweeps;
      p.rho[pair] = rho; p.degen[pair] = degen;
    }
    slot_sync(slot);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

size_t small_tc_smem_bytes() { return sizeof(SmemTC) + 1024; }
size_t small_tc_digit_bytes_per_pair() { return (size_t)3 * kOperand; }   // A', A and X images
size_t small_tc_exp_ints_per_pair() { return (size_t)2 * kS; }

cudaError_t launch_small_digits_prep(const SmallArgs& a, int grid, cudaStream_t s) {
  small_digits_prep_kernel<<<grid, 256, 0, s>>>(a.A, a.Ap, a.batch, a.n, a.np, a.dig, a.dexp);
  return cudaGetLastError();
}

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
