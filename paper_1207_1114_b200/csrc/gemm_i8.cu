// gemm_i8.cu — the two products of Algorithm 1 line 3, U = A' X^T and
// Y[0:n,0:n'] = A U^T + lambda K, on the int8 tensor cores (tcgen05.mma.kind::i8) with an
// Ozaki-style exact digit decomposition (FASTPFP_OPT_PRECISION = 3, DESIGN.md §6 "Ozaki int8").
//
// Every operand row r (K contiguous) is stored as a power-of-two scale 2^e_r and three signed
// 7-bit digit planes:  x_rk = 2^e_r * (d1_rk 2^-7 + d2_rk 2^-14 + d3_rk 2^-21) + O(2^-22 2^e_r),
// with e_r = frexp exponent of max_k |x_rk| (so |x / 2^e| < 1) and d_k = clamp(rint(r_k 128), +-127),
// r_{k+1} = r_k 128 - d_k. The product of two such rows is
//   sum_k P_ik Q_jk = 2^(eP_i + eQ_j) * sum_{p+q <= 4} 2^-7(p+q) (Dp_i . Dq_j)
// where every digit dot product is an EXACT int32: a weight class sums at most 3 digit products of
// |d| <= 127, so K <= 2^15 keeps |sum| <= 3 * 127^2 * 2^15 < 2^31.
// The six digit pairs fall into three weight classes w = p + q = 2, 3, 4, accumulated in three
// int32 TMEM accumulators; the epilogue combines them in fp32 (2^-14 (a2 + 2^-7 (a3 + 2^-7 a4)))
// and applies the exact power-of-two scales. Dropped pairs (p + q >= 5) and the digit truncation
// contribute <= 2^-21 relative to the row scales, the same order as an fp32 accumulation
// (measured: tests/diagnostics/ozaki_drift.py, drift from the fp64 oracle equal to fp32's).
//
// Kernel shape: persistent, one CTA pair (cta_group::2) per 256 x 128 output tile; each CTA stages
// 128 rows of P and 64 rows of Q per 128-byte K block (3 digit planes each, TMA SWIZZLE_128B,
// 3-stage mbarrier ring, 72 KB per stage = the whole shared memory); the MMA warp runs its loop
// warp-uniformly and one elected lane issues 6 x 4 UMMAs (K = 32 int8 each) per stage from uniform
// registers (a single-lane branch cost an R2UR round trip per MMA: 13% of the GEMM); 3 x 128 TMEM
// columns hold the accumulators (single-buffered: 384 of 512 columns); 4 epilogue warps read them
// into registers (one output row per thread), release TMEM at once, and store from registers
// while the next tile's main loop runs; a CTA's last tile goes through the (then idle) operand ring
// for coalesced row stores. The int8 pipe runs 8192 MAC/clk/SM, 4x the TF32 rate.
// Measured at c5 (ncu): tensor pipe 97% active; the SM clock sits at 1.6-1.7 GHz under this load
// (power), so the GEMM is bound by the tensor pipe at the power-limited clock.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <cstdio>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fpfp {

namespace {

using namespace tc;

constexpr int kBKb = 128;                 // K bytes (int8 elements) per stage: one 128 B swizzle row
constexpr int kPRows = 128;               // P rows per CTA
constexpr int kStages = 3;
constexpr int kPBox = kPRows * kBKb;      // 16 KB: one P digit plane, this CTA's 128 rows
constexpr int kHBox = 64 * kBKb;          // 8 KB: half a Q plane (this CTA's 64 rows)
// stage: P1 P2 P3 | H1 H2 H3 (this CTA's halves of the three Q planes)
constexpr int kOffH = 3 * kPBox;
constexpr int kStageBytes = kOffH + 3 * kHBox;       // 72 KB
constexpr int kThreads = 256;
constexpr int kTileM = 256, kTileN = 128;
constexpr uint32_t kTmemCols = 512;       // 3 x 128 used

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

struct I8Params {
  int M, N, K;
  int q3d, qk;                    // Q planes are [K/qk][N][qk] blocks (3-D tensor maps) when q3d
  const int* eP; const int* eQ;   // per-row exponents
  int epi;
  float* C; int64_t ldC;
  const float* D; int64_t ldD; float lam;
  const float* D2; int64_t ldD2; float scale;
  unsigned* rowmax;               // kEpiRowMax: atomicMax of |C| bits per row (M side)
  const int* done;
};

#ifndef FPFP_I8_GROUP
#define FPFP_I8_GROUP 8   // M tiles per raster group (experiment switch)
#endif
__device__ __forceinline__ void tile_coords_i8(int t, int num_m, int num_n, int& mt, int& nt) {
  constexpr int kGroup = FPFP_I8_GROUP;
  const int per_group = kGroup * num_n;
  const int g = t / per_group;
  const int first_m = g * kGroup;
  const int gsz = min(num_m - first_m, kGroup);
  const int r = t - g * per_group;
  mt = first_m + r % gsz;
  nt = r / gsz;
}

__device__ __forceinline__ float pow2f(int e) {
  // exact 2^e for the normal range, ldexpf otherwise
  return (e > -127 && e < 128) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e);
}

__global__ void __launch_bounds__(kThreads, 1)
gemm_i8_kernel(const __grid_constant__ CUtensorMap mP1, const __grid_constant__ CUtensorMap mP2,
               const __grid_constant__ CUtensorMap mP3, const __grid_constant__ CUtensorMap mQ1,
               const __grid_constant__ CUtensorMap mQ2, const __grid_constant__ CUtensorMap mQ3,
               I8Params p) {
  if (p.done && *p.done) return;  // uniform across the grid

  // D = S32, A = B = signed int8, K-major, M = 256 (pair), N = 128
  constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTileN >> 3) << 17) |
                              ((uint32_t)(kTileM >> 4) << 24);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar;
  __shared__ __align__(8) uint64_t tempty_bar;
  __shared__ uint32_t tmem_base_sm;
  __shared__ float s_cscale[2][kTileN];   // double-buffered by tile parity

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int num_m = (int)ceil_div(p.M, kTileM), num_n = (int)ceil_div(p.N, kTileN);
  const int num_tiles = num_m * num_n;
  const int num_kb = (int)ceil_div(p.K, kBKb);
  const int cid = (int)cluster_id_x();
  const int ncl = (int)num_clusters_x();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 4 * 2);
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sm)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sm;

  if (warp == 0) {
    // ===================== TMA producer (one elected lane per CTA) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        int mt, nt;
        tile_coords_i8(t, num_m, num_n, mt, nt);
        const int prow = mt * kTileM + (int)rank * kPRows;
        const int qhalf = nt * kTileN + (int)rank * 64;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t bar = mapa(smem_u32(&full_bar[stage]), 0);   // the leader's barrier
#ifdef FPFP_I8_NOTMA   // experiment: MMA rate alone (operands stale)
          if (leader) mbar_expect_tx(&full_bar[stage], 0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          continue;
#endif
          if (leader) mbar_expect_tx(&full_bar[stage], kStageBytes * 2);
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          const int kc = kb * kBKb;
          tma_load<2>(&mP1, base + 0 * kPBox, bar, kc, prow);
          tma_load<2>(&mP2, base + 1 * kPBox, bar, kc, prow);
          tma_load<2>(&mP3, base + 2 * kPBox, bar, kc, prow);
          if (p.q3d) {   // row-sharded GEMM2: K walks the gathered rank blocks
            const int blk = kc / p.qk, kin = kc - blk * p.qk;
            tma_load3<2>(&mQ1, base + kOffH + 0 * kHBox, bar, kin, qhalf, blk);
            tma_load3<2>(&mQ2, base + kOffH + 1 * kHBox, bar, kin, qhalf, blk);
            tma_load3<2>(&mQ3, base + kOffH + 2 * kHBox, bar, kin, qhalf, blk);
          } else {
            tma_load<2>(&mQ1, base + kOffH + 0 * kHBox, bar, kc, qhalf);
            tma_load<2>(&mQ2, base + kOffH + 1 * kHBox, bar, kc, qhalf);
            tma_load<2>(&mQ3, base + kOffH + 2 * kHBox, bar, kc, qhalf);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, one lane) =====================
    // the whole warp runs the loop (warp-uniform control flow, descriptors in uniform registers);
    // one elected lane issues the MMAs and commits
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_phase = 0;
#ifdef FPFP_I8_CLK
      const long long c_start = clock64();
      unsigned long long gc_start;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gc_start));
#endif
#ifdef FPFP_I8_PROF
      long long t_empty = 0, t_full = 0, t_start = clock64();
      unsigned long long g_start;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
      int ntl = 0;
#endif
      for (int t = cid; t < num_tiles; t += ncl) {
#ifdef FPFP_I8_PROF
        long long w0 = clock64();
#endif
        mbar_wait(&tempty_bar, acc_phase ^ 1);   // epilogue drained the accumulators
#ifdef FPFP_I8_PROF
        t_empty += clock64() - w0;
#endif
        tc_fence_after();
        const uint32_t acc2 = tmem_base, acc3 = tmem_base + 128, acc4 = tmem_base + 256;
        for (int kb = 0; kb < num_kb; ++kb) {
#ifdef FPFP_I8_PROF
          long long w1 = clock64();
#endif
          mbar_wait(&full_bar[stage], phase);
#ifdef FPFP_I8_PROF
          t_full += clock64() - w1;
#endif
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kBKb / 32; ++k) {   // K = 32 int8 (32 bytes) per MMA
            const uint32_t off = (uint32_t)k * 32u;
            const uint64_t p1 = smem_desc(base + 0 * kPBox + off);
            const uint64_t p2 = smem_desc(base + 1 * kPBox + off);
            const uint64_t p3 = smem_desc(base + 2 * kPBox + off);
            const uint64_t q1 = smem_desc(base + kOffH + 0 * kHBox + off);
            const uint64_t q2 = smem_desc(base + kOffH + 1 * kHBox + off);
            const uint64_t q3 = smem_desc(base + kOffH + 2 * kHBox + off);
            const uint32_t acc = (kb == 0 && k == 0) ? 0u : 1u;
#ifdef FPFP_I8_NOMMA   // experiment: operand delivery alone
            if (acc < 2) continue;
#endif
            // the six digit products by weight class w = p + q
            mma_i8(acc2, p1, q1, kIdesc, acc);   // w = 2
            mma_i8(acc3, p1, q2, kIdesc, acc);   // w = 3
            mma_i8(acc4, p1, q3, kIdesc, acc);   // w = 4
            mma_i8(acc3, p2, q1, kIdesc, 1u);
            mma_i8(acc4, p2, q2, kIdesc, 1u);
            mma_i8(acc4, p3, q1, kIdesc, 1u);
          }
          umma_commit<2>(&empty_bar[stage]);     // frees the smem slot in both CTAs
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit<2>(&tfull_bar);   // accumulators ready (both CTAs)
        __syncwarp();
        acc_phase ^= 1;
#ifdef FPFP_I8_PROF
        ++ntl;
#endif
      }
#ifdef FPFP_I8_CLK
      {
        unsigned long long gc_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gc_end));
        const long long c_end = clock64();
        if (cid == 0 && lane == 0) printf("i8-clk %lld clk in %llu ns (%.0f MHz)\n", c_end - c_start, gc_end - gc_start,
                             (double)(c_end - c_start) * 1e3 / (double)(gc_end - gc_start));
      }
#endif
#ifdef FPFP_I8_PROF
      unsigned long long g_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
      if ((cid == 0 || cid == 37) && lane == 0)
        printf("i8-prof cluster %d: tiles %d total %lld clk in %llu ns (%.0f MHz), wait-accumulator %lld, wait-operands %lld, issue %lld\n",
               cid, ntl, clock64() - t_start, g_end - g_start, (double)(clock64() - t_start) * 1e3 / (double)(g_end - g_start),
               t_empty, t_full, clock64() - t_start - t_empty - t_full);
#endif
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    // E1: TMEM -> registers, combined into the 128 fp32 outputs of this thread's row, then TMEM is
    //     released so the MMAs of the next tile start at once;
    // E2: the row is written from registers (adding lambda K / the PG term), overlapping the next
    //     tile's main loop. No shared-memory staging: the whole ring is operand stages.
    const int ew = warp & 3;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader = mapa(smem_u32(&tempty_bar), 0);
    for (int t = cid; t < num_tiles; t += ncl) {
      int mt, nt;
      tile_coords_i8(t, num_m, num_n, mt, nt);
      const int rbase = mt * kTileM + (int)rank * kPRows;
      const int cbase = nt * kTileN;
      const int lrow = ew * 32 + lane;
      const int row = rbase + lrow;
      float* cs = s_cscale[acc_phase];
      // column scales 2^(eQ_j - 14) of this tile, staged while the main loop still runs
      cs[lrow] = cbase + lrow < p.N ? pow2f(__ldg(p.eQ + cbase + lrow) - 14) : 0.0f;
      const float rscale = row < p.M ? pow2f(p.eP[row]) : 0.0f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait_sleep(&tfull_bar, acc_phase, 256);   // a whole main loop away: do not spin
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16);
      float o[kTileN];
      float rmax = 0.0f;
#pragma unroll
      for (int cc = 0; cc < kTileN / 16; ++cc) {
        uint32_t a2[16], a3[16], a4[16];
        tmem_ld16_nowait(tb + (uint32_t)(cc * 16), a2);
        tmem_ld16_nowait(tb + 128u + (uint32_t)(cc * 16), a3);
        tmem_ld16_nowait(tb + 256u + (uint32_t)(cc * 16), a4);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // 2^-14 (a2 + 2^-7 (a3 + 2^-7 a4)) * 2^eP * 2^eQ (exact power-of-two scalings)
          float v = fmaf((float)(int)a4[j], 0.0078125f, (float)(int)a3[j]);
          v = fmaf(v, 0.0078125f, (float)(int)a2[j]);
          v = (v * rscale) * cs[cc * 16 + j];
          o[cc * 16 + j] = v;
          rmax = fmaxf(rmax, fabsf(v));   // columns past N carry scale 0
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader);   // accumulators free
      if (t + ncl >= num_tiles) {
        // this CTA's last tile: every operand stage is idle once the accumulators are complete
        // (no further loads are issued), so the tile is staged through shared memory and written
        // with coalesced row stores. Matters when a CTA has few tiles (n ~ 1000: one tile each,
        // the epilogue is the whole tail of the kernel); rows of one thread are 512 B apart.
        if (p.epi == kEpiRowMax && row < p.M) atomicMax(p.rowmax + row, __float_as_uint(rmax));
        float* stile = reinterpret_cast<float*>(smem);   // [128][128] fp32, float4 c at c ^ (row & 31)
        float* srow = stile + lrow * kTileN;
#pragma unroll
        for (int c4 = 0; c4 < kTileN / 4; ++c4)
          *reinterpret_cast<float4*>(srow + ((c4 ^ (lrow & 31)) * 4)) =
              make_float4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int col = cbase + lane * 4;    // lane l owns columns 4l .. 4l + 3 of every row
        const bool cfull = col + 4 <= p.N;
        const bool add_d = (p.epi == kEpiAxpy || p.epi == kEpiPG) && p.D;
        for (int r0 = ew; r0 < kPRows; r0 += 32) {
          // 8 rows per batch: their lambda K (and PG X) loads are issued before any store (C may
          // alias D as far as the compiler knows, which would serialise load / store pairs)
          float4 dv[8], xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int grow = rbase + r0 + 4 * u;
            const bool ok = cfull && grow < p.M;
            dv[u] = (add_d && ok) ? __ldg(reinterpret_cast<const float4*>(p.D + (int64_t)grow * p.ldD + col))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            xv[u] = (p.epi == kEpiPG && ok)
                        ? __ldg(reinterpret_cast<const float4*>(p.D2 + (int64_t)grow * p.ldD2 + col))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = r0 + 4 * u;
            const int grow = rbase + r;
            if (grow >= p.M) break;
            float4 v = *reinterpret_cast<const float4*>(stile + r * kTileN + ((lane ^ (r & 31)) * 4));
            float* ve = reinterpret_cast<float*>(&v);
            if (cfull) {
              v.x += p.lam * dv[u].x; v.y += p.lam * dv[u].y; v.z += p.lam * dv[u].z; v.w += p.lam * dv[u].w;
              if (p.epi == kEpiPG) {   // Projected Gradient: X + alpha (A X A' + lambda K)
                v.x = p.scale * v.x + xv[u].x; v.y = p.scale * v.y + xv[u].y;
                v.z = p.scale * v.z + xv[u].z; v.w = p.scale * v.w + xv[u].w;
              }
              *reinterpret_cast<float4*>(p.C + (int64_t)grow * p.ldC + col) = v;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                if (col + e >= p.N) break;
                float x = ve[e];
                if (add_d) x += p.lam * p.D[(int64_t)grow * p.ldD + col + e];
                if (p.epi == kEpiPG) x = p.scale * x + p.D2[(int64_t)grow * p.ldD2 + col + e];
                p.C[(int64_t)grow * p.ldC + col + e] = x;
              }
            }
          }
        }
      } else if (row < p.M) {
        if (p.epi == kEpiRowMax) atomicMax(p.rowmax + row, __float_as_uint(rmax));
        float* crow = p.C + (int64_t)row * p.ldC + cbase;
        const bool add_d = (p.epi == kEpiAxpy || p.epi == kEpiPG) && p.D;
        const float* drow = add_d ? p.D + (int64_t)row * p.ldD + cbase : nullptr;
        const float* xrow = p.epi == kEpiPG ? p.D2 + (int64_t)row * p.ldD2 + cbase : nullptr;
        if (cbase + kTileN <= p.N) {
#pragma unroll
          for (int c = 0; c < kTileN; c += 4) {
            float4 v = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
            if (drow) {
              const float4 dv = __ldg(reinterpret_cast<const float4*>(drow + c));
              v.x += p.lam * dv.x; v.y += p.lam * dv.y; v.z += p.lam * dv.z; v.w += p.lam * dv.w;
            }
            if (xrow) {   // Projected Gradient: X + alpha (A X A' + lambda K)
              const float4 xv = __ldg(reinterpret_cast<const float4*>(xrow + c));
              v.x = p.scale * v.x + xv.x; v.y = p.scale * v.y + xv.y;
              v.z = p.scale * v.z + xv.z; v.w = p.scale * v.w + xv.w;
            }
            *reinterpret_cast<float4*>(crow + c) = v;
          }
        } else {
#pragma unroll
          for (int c = 0; c < kTileN; ++c) {
            if (cbase + c < p.N) {
              float x = o[c];
              if (drow) x += p.lam * drow[c];
              if (xrow) x = p.scale * x + xrow[c];
              crow[c] = x;
            }
          }
        }
      }
      acc_phase ^= 1;
    }
  }

  // teardown
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ---- digit split: one warp per row ----------------------------------------------------------
// rowmax (nullable): precomputed |max| bits per row (GEMM1's kEpiRowMax); else computed here.
__device__ __forceinline__ int pack4i(int d0, int d1, int d2, int d3) {
  return (d0 & 0xFF) | ((d1 & 0xFF) << 8) | ((d2 & 0xFF) << 16) | ((d3 & 0xFF) << 24);
}

// 4 consecutive values -> one packed word (4 digits) per plane at o[0..2] + k (k % 4 == 0, in range)
__device__ __forceinline__ void digits_store4(float4 q, float inv, int8_t* o1, int8_t* o2, int8_t* o3, int k) {
  int a0, b0, c0, a1, b1, c1, a2, b2, c2, a3, b3, c3;
  ozaki_digits3(q.x, inv, a0, b0, c0);
  ozaki_digits3(q.y, inv, a1, b1, c1);
  ozaki_digits3(q.z, inv, a2, b2, c2);
  ozaki_digits3(q.w, inv, a3, b3, c3);
  *reinterpret_cast<int*>(o1 + k) = pack4i(a0, a1, a2, a3);
  *reinterpret_cast<int*>(o2 + k) = pack4i(b0, b1, b2, b3);
  *reinterpret_cast<int*>(o3 + k) = pack4i(c0, c1, c2, c3);
}

// one warp per row; 4 float4 loads in flight per lane (HBM-bound at c5: 4 B read + 3 B written)
__global__ void split_i8_kernel(const float* __restrict__ src, int64_t lds, int rows, int K,
                                const unsigned* __restrict__ rowmax, int8_t* __restrict__ d1,
                                int8_t* __restrict__ d2, int8_t* __restrict__ d3, int64_t ldd,
                                int* __restrict__ ex, const int* done) {
  if (done && *done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  const int Kv = K & ~3;                 // float4-vectorised part
  for (int r = gw; r < rows; r += nw) {
    const float* x = src + (int64_t)r * lds;
    float mx;
    if (rowmax) {
      mx = __uint_as_float(rowmax[r]);
    } else {
      mx = 0.0f;
      int k = lane * 4;
      for (; k + 384 < Kv; k += 512) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(x + k + 128 * u));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
      }
      for (; k < Kv; k += 128) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + k));
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      for (int e = Kv + lane; e < K; e += 32) mx = fmaxf(mx, fabsf(x[e]));
      mx = warp_max(mx);
    }
    const int e = frexp_exp(mx);     // mx = f 2^e, f in [0.5, 1): |x / 2^e| < 1
    if (lane == 0) ex[r] = e;
    const float inv = exp2i(-e);
    int8_t* o1 = d1 + (int64_t)r * ldd;
    int8_t* o2 = d2 + (int64_t)r * ldd;
    int8_t* o3 = d3 + (int64_t)r * ldd;
    int k = lane * 4;
    for (; k + 384 < Kv; k += 512) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(x + k + 128 * u));
#pragma unroll
      for (int u = 0; u < 4; ++u) digits_store4(v[u], inv, o1, o2, o3, k + 128 * u);
    }
    for (; k < Kv; k += 128) digits_store4(__ldg(reinterpret_cast<const float4*>(x + k)), inv, o1, o2, o3, k);
    for (int t = Kv + lane; t < K; t += 32) {
      int a, b, c;
      ozaki_digits3(x[t], inv, a, b, c);
      o1[t] = (int8_t)a; o2[t] = (int8_t)b; o3[t] = (int8_t)c;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
std::once_flag g_enc_once;

bool get_enc() {
  std::call_once(g_enc_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_enc != nullptr;
}

// rows x K int8 plane with row stride ld bytes; box = box_rows x 128 bytes, SW128
bool make_map_i8(CUtensorMap* m, const int8_t* base, int rows, int K, int64_t ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)kBKb, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// [blocks][rows][qk] int8 plane blocks (row stride ld bytes, block stride bstride bytes)
bool make_map3_i8(CUtensorMap* m, const int8_t* base, int rows, int qk, int blocks, int64_t ld,
                  int64_t bstride, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)qk, (cuuint64_t)rows, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)bstride};
  cuuint32_t box[3] = {(cuuint32_t)kBKb, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool gemm_i8_supported(const I8Gemm& g) {
  if (!get_enc()) return false;
  if (g.M < 1 || g.N < 1 || g.K < 1 || g.K > (1 << 15)) return false;   // int32 class sums
  for (int k = 0; k < 3; ++k)
    if (!g.P[k] || !g.Q[k] || (reinterpret_cast<uintptr_t>(g.P[k]) % 16) || (reinterpret_cast<uintptr_t>(g.Q[k]) % 16))
      return false;
  if (g.q_blocks > 1 && (g.q_block_k % kBKb != 0 || (int64_t)g.q_block_k * g.q_blocks != g.K ||
                         g.q_block_stride % 16 != 0))
    return false;
  return (g.ldP % 16 == 0) && (g.ldQ % 16 == 0) && (g.ldC % 4 == 0) && g.eP && g.eQ;
}

cudaError_t launch_gemm_i8(const I8Gemm& g, cudaStream_t s, int device) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  CUtensorMap mp[3];
  const bool q3d = g.q_blocks > 1;
  for (int k = 0; k < 3; ++k)
    if (!make_map_i8(&mp[k], g.P[k], g.M, g.K, g.ldP, kPRows)) return cudaErrorInvalidValue;
  // Q planes: 64-row half boxes (the N = 128 operands, split between the CTAs of the pair)
  CUtensorMap mq[3];
  auto mk = [&](CUtensorMap* m, const int8_t* base, int box_rows) {
    return q3d ? make_map3_i8(m, base, g.N, g.q_block_k, g.q_blocks, g.ldQ, g.q_block_stride, box_rows)
               : make_map_i8(m, base, g.N, g.K, g.ldQ, box_rows);
  };
  for (int k = 0; k < 3; ++k)
    if (!mk(&mq[k], g.Q[k], 64)) return cudaErrorInvalidValue;
  I8Params p{g.M, g.N, g.K, q3d ? 1 : 0, q3d ? g.q_block_k : 0, g.eP, g.eQ, g.epi, g.C, g.ldC, g.D,
             g.ldD, g.lam, g.D2, g.ldD2, g.scale, g.rowmax, g.done};
  const size_t smem = (size_t)kStages * kStageBytes + 1024;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t tiles = ceil_div(g.M, kTileM) * ceil_div(g.N, kTileN);
  const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, sms / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * 2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_i8_kernel, mp[0], mp[1], mp[2], mq[0], mq[1], mq[2], p);
}

cudaError_t launch_split_i8(const float* src, int64_t lds, int rows, int K, const unsigned* rowmax,
                            int8_t* const d[3], int64_t ldd, int* ex, const int* done, cudaStream_t s) {
  const int warps = 8;
  const int grid = (int)std::min<int64_t>(4096, std::max<int64_t>(1, ceil_div(rows, warps)));
  split_i8_kernel<<<grid, warps * 32, 0, s>>>(src, lds, rows, K, rowmax, d[0], d[1], d[2], ldd, ex, done);
  return cudaGetLastError();
}

}  // namespace fpfp
