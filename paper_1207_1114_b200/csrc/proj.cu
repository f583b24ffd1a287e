// proj.cu — the projection loop (Algorithm 1 lines 4-7) and the blend/rescale
// (lines 8-9) as ONE persistent cooperative kernel per outer iteration.
//
// Y is the m x m slacked matrix. One sweep is P2(P1(Y)) with the closed forms
//   P1(Y)_ij = Y_ij + (1 + sigma/m - r_i - c_j)/m,  r = Y 1, c = Y^T 1, sigma = 1^T Y 1  ({P1}, P:300-302
//   with 1^T Y 1 as in Alg. 1 line 5, reading A2),   P2(Z) = (Z + |Z|)/2 = max(Z, 0)  ({P2})
// and delta = max|Y_new - Y_old|. Every Z_ij needs the global sums of the previous Y,
// so a sweep is: [tile pass: read Y, write Z, emit fp64 partial row/col sums of Z and a partial
// delta] -> grid barrier -> [reduce partials to r, c, sigma] -> grid barrier. That is the minimum
// of one HBM read + one HBM write of Y per sweep (DESIGN.md §Kernels "proj"). The sums of the
// fresh GEMM output are taken by a read-only pass first. The inner loop (convergence test on
// delta) runs on the device: every block computes the same delta from the same partials.
//
// Numerics: Y is stored in fp32; r, c, sigma and the P1 correction are
// evaluated in fp64 (the first P1 after a GEMM cancels values ~1e2-1e3 down to O(1/m)), then the
// result is rounded once to fp32. Reductions are two-stage with a fixed order (no float atomics),
// so results are bitwise reproducible for a given grid.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fpfp {

namespace {

constexpr int kWarps = kProjThreads / kWarp;  // 8
constexpr int kQ = kProjTC / 128;             // float4 chunks per lane per row
#ifndef FPFP_PROJ_DEPTH
#define FPFP_PROJ_DEPTH 2
#endif

struct __align__(16) ProjSmem {
  double col[kWarps][kProjTC];  // 32 KB: per-warp column partials of one tile
  double red[kWarps];
  double bcast[4];
};

// Row staging for the tile pass (FPFP_PROJ_BULK, default on): every warp owns a ring of kSlots
// shared-memory row buffers filled by 1-D bulk async copies (cp.async.bulk, the TMA engine) on
// mbarriers, so kSlots rows per warp (8 KB per CTA per slot depth) are in flight without holding
// registers; the register-ring path (FPFP_PROJ_BULK=0) keeps kDepth rows of float4 loads instead.
#ifndef FPFP_PROJ_BULK
#define FPFP_PROJ_BULK 1
#endif
#ifndef FPFP_PROJ_SLOTS
#define FPFP_PROJ_SLOTS 8
#endif
constexpr int kSlots = FPFP_PROJ_SLOTS;   // a power of two (slot = seq % kSlots)
static_assert((kSlots & (kSlots - 1)) == 0, "kSlots must be a power of two");
#ifndef FPFP_PROJ_RING_FIRST
#define FPFP_PROJ_RING_FIRST 1
#endif
constexpr size_t kRingBytes = FPFP_PROJ_BULK ? (size_t)kWarps * kSlots * kProjTC * sizeof(float) : 0;

struct Ring {
  float* buf;          // [kWarps][kSlots][kProjTC] (dynamic shared memory)
  uint64_t* bar;       // [kWarps][kSlots]
  uint32_t seq;        // rows consumed by this warp so far (slot = seq % kSlots, parity = seq / kSlots)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ring_issue(uint64_t* bar, float* dst, const float* src, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void ring_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

// X~ = (1 - alpha) X + alpha Y in fp64 (Algorithm 1 line 8): one expression shared by every
// place that forms it, so the fused and the separate mu passes give identical values
__device__ __forceinline__ double blend_xt(double a, double b, float x, float y) {
  return __fma_rn(a, (double)y, b * (double)x);
}

// One tile pass over rows [rb*TR, ...) x cols [cb*512, ...) of Y.
//   kSweep = false: sums only (Z = Y), accumulated in fp64 (the fresh GEMM output cancels in the
//   first correction, reading A2 / DESIGN.md §6).
//   kSweep = true: Z = max(Y + t_i - u_j, 0) written back; the sums of Z for the next sweep are
//   accumulated in fp32 per lane (16 values of a row, <= 64 rows of a column) and in fp64 beyond:
//   their rounding (<= 2^-18 relative) is far below that of the fp32 storage of Y at the same sweep.
//   kFull: every column of the tile is inside m (no per-element bounds test).
//   kMu (last sweep of a fixed-count inner loop, single GPU): the pass also forms X~ from the fresh
//   Z of the X block and reduces max X~ (mu, line 9) and the per-row max |X~| of the fused X digits,
//   which saves the separate mu pass over X and Y[0:n, 0:n'] (finalize_mu).
template <bool kSweep, bool kFull = false, bool kMu = false>
__device__ __forceinline__ void tile_pass(const ProjArgs& p, int tile, double sigma, float& dmax,
                                          ProjSmem& sm, Ring& ring_st, double* mu_acc = nullptr) {
  const int rb = tile / p.CB, cb = tile - (tile / p.CB) * p.CB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = rb * p.TR;
  const int row1 = min(p.rows, row0 + p.TR);
  const int colbase = cb * kProjTC;
  const double inv_m = 1.0 / (double)p.m;
#if FPFP_PROJ_BULK && FPFP_PROJ_RING_FIRST
  // the first rows' bulk copies go out before the sum vectors are loaded (HBM and L2 latency overlap)
  constexpr int kDepth = kSlots;
  const uint32_t row_bytes = (uint32_t)min(kProjTC, (int)(p.ldY - colbase)) * 4u;
  float* wbuf = ring_st.buf + (size_t)warp * kSlots * kProjTC;
  uint64_t* wbar = ring_st.bar + warp * kSlots;
  const uint32_t seq0 = ring_st.seq;
  const int i0 = row0 + warp;
  const int nrows_w = i0 < row1 ? (row1 - i0 + kWarps - 1) / kWarps : 0;
  asm volatile("fence.proxy.async.global;" ::: "memory");   // Y written by the generic proxy
  if (lane == 0) {
#pragma unroll 1
    for (int k = 0; k < kDepth && k < nrows_w; ++k) {
      const uint32_t slot = (seq0 + k) % kSlots;
      ring_issue(wbar + slot, wbuf + slot * kProjTC, p.Y + (int64_t)(i0 + k * kWarps) * p.ldY + colbase,
                 row_bytes);
    }
  }
  __syncwarp();
#endif

  double u[kQ][4], colacc[kQ][4];
  float colf[kQ][4];
  bool inrow[kQ];  // float4 inside the allocated row (col < ldY)
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int j0 = colbase + q * 128 + lane * 4;
    inrow[q] = kFull || j0 < p.ldY;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + e;
      u[q][e] = (kSweep && (kFull || j < p.m)) ? __ldcg(p.c + j) * inv_m : 0.0;
      colacc[q][e] = 0.0;
      colf[q][e] = 0.0f;
    }
  }
  const double tconst = (1.0 + sigma * inv_m) * inv_m;  // (1/n + 1^T Y 1 / n^2)
  // this warp's rows are row0 + warp + 8 t, t < TR/8 <= 64: lane l holds r for t = l and t = l + 32
  // (loaded up front, in parallel with the first rows of Y, then shuffled out row by row)
  double r_lo = 0.0, r_hi = 0.0;
  if (kSweep) {
    const int ia = row0 + warp + kWarps * lane, ib = ia + kWarps * 32;
    r_lo = ia < row1 ? __ldcg(p.r + ia) : 0.0;
    r_hi = ib < row1 ? __ldcg(p.r + ib) : 0.0;
  }

  // Software-pipelined over the warp's rows: a ring of kDepth (kSlots) rows stays in flight per
  // warp (memory-level parallelism is what bounds this kernel), each slot refilled with the row
  // kDepth steps ahead as soon as its own row has been corrected and stored.
#if FPFP_PROJ_BULK
#if !FPFP_PROJ_RING_FIRST
  constexpr int kDepth = kSlots;
  const uint32_t row_bytes = (uint32_t)min(kProjTC, (int)(p.ldY - colbase)) * 4u;
  float* wbuf = ring_st.buf + (size_t)warp * kSlots * kProjTC;
  uint64_t* wbar = ring_st.bar + warp * kSlots;
  const uint32_t seq0 = ring_st.seq;
  const int i0 = row0 + warp;
  const int nrows_w = i0 < row1 ? (row1 - i0 + kWarps - 1) / kWarps : 0;
  asm volatile("fence.proxy.async.global;" ::: "memory");   // Y written by the generic proxy
  if (lane == 0) {
#pragma unroll 1
    for (int k = 0; k < kDepth && k < nrows_w; ++k) {
      const uint32_t slot = (seq0 + k) % kSlots;
      ring_issue(wbar + slot, wbuf + slot * kProjTC, p.Y + (int64_t)(i0 + k * kWarps) * p.ldY + colbase,
                 row_bytes);
    }
  }
  __syncwarp();
#endif
  // rows are processed in groups of 4 so that their 4 row sums share one transposed warp
  // reduction (6 double shuffles per 4 rows instead of 5 per row)
  for (int tg = 0; tg < nrows_w; tg += 4) {
    double rq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u4 = 0; u4 < 4; ++u4) {
      const int t = tg + u4;
      if (t >= nrows_w) break;
      const int i = i0 + t * kWarps;
      const uint32_t slot = (seq0 + t) % kSlots;
      ring_wait(wbar + slot, ((seq0 + t) / kSlots) & 1u);
      float4 cur[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        cur[q] = inrow[q] ? *reinterpret_cast<const float4*>(wbuf + slot * kProjTC + q * 128 + lane * 4)
                          : make_float4(0, 0, 0, 0);
      __syncwarp();
      if (lane == 0 && t + kDepth < nrows_w) {   // refill this slot with the row kDepth ahead
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        ring_issue(wbar + slot, wbuf + slot * kProjTC,
                   p.Y + (int64_t)(i + kDepth * kWarps) * p.ldY + colbase, row_bytes);
      }
      float* rowp = p.Y + (int64_t)i * p.ldY + colbase + lane * 4;
#else
  constexpr int kDepth = FPFP_PROJ_DEPTH;
  auto load_row = [&](int i, float4 (&v)[kQ]) {
    const float* rowp = p.Y + (int64_t)i * p.ldY + colbase + lane * 4;
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      v[q] = inrow[q] ? __ldcg(reinterpret_cast<const float4*>(rowp + q * 128)) : make_float4(0, 0, 0, 0);
  };
  float4 ring[kDepth][kQ];
  const int i0 = row0 + warp;
#pragma unroll
  for (int k = 0; k < kDepth; ++k)
    if (i0 + k * kWarps < row1) load_row(i0 + k * kWarps, ring[k]);
  for (int base = i0; base < row1; base += kDepth * kWarps) {
#pragma unroll
    for (int k = 0; k < kDepth; ++k) {
      const int i = base + k * kWarps;
      if (i >= row1) break;
      float4 (&cur)[kQ] = ring[k];
      float* rowp = p.Y + (int64_t)i * p.ldY + colbase + lane * 4;
#endif
      double ti = 0.0;
      if (kSweep) {
        const int t = (i - row0 - warp) / kWarps;
        const double rlo = __shfl_sync(0xffffffffu, r_lo, t & 31);
        const double rhi = __shfl_sync(0xffffffffu, r_hi, t & 31);
        ti = tconst - (t < 32 ? rlo : rhi) * inv_m;
      }
      double racc = 0.0;
      float racc_f = 0.0f;
      // kMu: this row's X segment (issued before the element loop; L2/HBM latency overlaps it)
      float4 xq[kQ];
      const bool xrow = kMu && i < p.n;
      if (kMu) {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int j0 = colbase + q * 128 + lane * 4;
          xq[q] = (xrow && j0 < p.np) ? __ldcs(reinterpret_cast<const float4*>(p.X + (int64_t)i * p.ldX + j0))
                                      : make_float4(0, 0, 0, 0);
        }
      }
      double xrmax = 0.0;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        float* ve = reinterpret_cast<float*>(&cur[q]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = colbase + q * 128 + lane * 4 + e;
          const bool valid = kFull || j < p.m;
          const float y = ve[e];
          if (kSweep) {
            const double zd = ((double)y + ti) - u[q][e];          // P1, fp64
            // P2 after the one rounding to fp32: rounding is monotonic and 0 is exact, so
            // max(fl32(zd), 0) = fl32(max(zd, 0)); one FMNMX instead of an fp64 max + selects
            float z = fmaxf((float)zd, 0.0f);
            if (!valid) z = 0.0f;
            dmax = fmaxf(dmax, fabsf(z - y));                       // delta
            ve[e] = z;
            racc_f += z;
            colf[q][e] += z;
            if (kMu && xrow && j < p.np) {                          // line 8 on the fresh Z
              const double xt = blend_xt(p.alpha, 1.0 - p.alpha, reinterpret_cast<const float*>(&xq[q])[e], z);
              *mu_acc = fmax(*mu_acc, xt);
              xrmax = fmax(xrmax, fabs(xt));
            }
          } else {
            const double zz = valid ? (double)y : 0.0;
            racc += zz;
            colacc[q][e] += zz;
          }
        }
      }
      if (kSweep) racc = (double)racc_f;
      if (kMu && p.xrowmax) {   // per-row max |X~| of this segment (nonnegative doubles order as bits)
        const double v = warp_max(xrmax);
        if (lane == 0 && xrow) atomicMax(p.xrowmax + i, (unsigned long long)__double_as_longlong(v));
      }
      if (kSweep) {
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (inrow[q]) __stcg(reinterpret_cast<float4*>(rowp + q * 128), cur[q]);
      }
#if FPFP_PROJ_BULK
      rq[u4] = racc;
    }
    // transposed reduction of the 4 rows: after the xor-16 and xor-8 exchanges lane L holds a
    // partial of row 2*bit4(L) + bit3(L); xor 4, 2, 1 finish it; lanes 0, 8, 16, 24 write
    const bool b4 = lane & 16, b3 = lane & 8;
    double k0 = b4 ? rq[2] : rq[0], k1 = b4 ? rq[3] : rq[1];
    k0 += __shfl_xor_sync(0xffffffffu, b4 ? rq[0] : rq[2], 16);
    k1 += __shfl_xor_sync(0xffffffffu, b4 ? rq[1] : rq[3], 16);
    double k = b3 ? k1 : k0;
    k += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    const int rsel = (b4 ? 2 : 0) + (b3 ? 1 : 0);
    if ((lane & 7) == 0 && tg + rsel < nrows_w)
      p.rowpart[(int64_t)cb * p.rows + i0 + (tg + rsel) * kWarps] = k;
  }
  ring_st.seq = seq0 + (uint32_t)nrows_w;
#else
      const int ahead = i + kDepth * kWarps;
      if (ahead < row1) load_row(ahead, ring[k]);
      racc = warp_sum(racc);
      if (lane == 0) p.rowpart[(int64_t)cb * p.rows + i] = racc;
    }
  }
#endif
  // column partials of this tile: combine the 8 warps in a fixed order
#pragma unroll
  for (int q = 0; q < kQ; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      sm.col[warp][q * 128 + lane * 4 + e] = kSweep ? (double)colf[q][e] : colacc[q][e];
  __syncthreads();
  for (int jj = threadIdx.x; jj < kProjTC; jj += kProjThreads) {
    const int j = colbase + jj;
    if (j < p.m) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += sm.col[w][jj];
      p.colpart[(int64_t)rb * p.m + j] = s;
    }
  }
  __syncthreads();
}

constexpr int kRC = kProjReplayC;   // checkpoint interval: Y stored every kRC sweeps

#if FPFP_PROJ_BULK
// Replay pass (single GPU, p.replay; DESIGN.md §8 "checkpointed sweeps"). Sweep k's output is an
// elementwise function of an earlier stored Y and the correction vectors of the sweeps between:
// Z_k = max(Z_{k-1} + t^(k) - u^(k), 0) with t^(k), u^(k) from the sums of Z_{k-1}. So the inner
// loop stores Y only every other sweep: pass k reads the last stored Y (the checkpoint) and
// re-applies D = 1 or 2 sweeps in registers; it writes Z_k only when asked (`write`: the odd sweeps
// and the cap's last), and always emits the sums of Z_k and delta = max|Z_k - Z_{k-1}| like
// tile_pass. Per 2 sweeps: 2 reads + 1 write of Y instead of 2 reads + 2 writes. These sweeps follow
// the first of the outer iteration (the fp64 one, whose operand is the product), so their
// correction runs in fp32, as in the on-chip kernel: t_i = fl32(tconst - r_i/m),
// u_j = fl32(c_j/m), z = max(fl32(fl32(y + t_i) - u_j), 0). A re-applied sweep repeats the same
// fp32 operations on the same stored operand, so every pass sees the same Z values.
//   rs[d], cs[d], tc[d]: row sums, column sums and tconst = (1 + sigma/m)/m of the sums each
//   re-applied sweep d < D consumes (d = D - 1: this pass's sweep).
template <bool kFull, bool kMu>
__device__ __forceinline__ void replay_pass(const ProjArgs& p, int tile, int D, bool write,
                                            const double* const (&rs)[kRC], const double* const (&cs)[kRC],
                                            const double (&tc)[kRC], float& dmax, ProjSmem& sm, Ring& ring_st,
                                            double* mu_acc) {
  const int rb = tile / p.CB, cb = tile - (tile / p.CB) * p.CB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = rb * p.TR;
  const int row1 = min(p.rows, row0 + p.TR);
  const int colbase = cb * kProjTC;
  const double inv_m = 1.0 / (double)p.m;
#if FPFP_PROJ_RING_FIRST
  const uint32_t row_bytes = (uint32_t)min(kProjTC, (int)(p.ldY - colbase)) * 4u;
  float* wbuf = ring_st.buf + (size_t)warp * kSlots * kProjTC;
  uint64_t* wbar = ring_st.bar + warp * kSlots;
  const uint32_t seq0 = ring_st.seq;
  const int i0 = row0 + warp;
  const int nrows_w = i0 < row1 ? (row1 - i0 + kWarps - 1) / kWarps : 0;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (lane == 0) {
#pragma unroll 1
    for (int k = 0; k < kSlots && k < nrows_w; ++k) {
      const uint32_t slot = (seq0 + k) % kSlots;
      ring_issue(wbar + slot, wbuf + slot * kProjTC, p.Y + (int64_t)(i0 + k * kWarps) * p.ldY + colbase,
                 row_bytes);
    }
  }
  __syncwarp();
#endif

  float u[kRC][kQ][4], colf[kQ][4];
  bool inrow[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int j0 = colbase + q * 128 + lane * 4;
    inrow[q] = kFull || j0 < p.ldY;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + e;
      const bool v = kFull || j < p.m;
#pragma unroll
      for (int d = 0; d < kRC; ++d) u[d][q][e] = (v && d < D) ? (float)(__ldcg(cs[d] + j) * inv_m) : 0.0f;
      colf[q][e] = 0.0f;
    }
  }
  double r_lo[kRC], r_hi[kRC];
  {
    const int ia = row0 + warp + kWarps * lane, ib = ia + kWarps * 32;
#pragma unroll
    for (int d = 0; d < kRC; ++d) {
      r_lo[d] = (d < D && ia < row1) ? __ldcg(rs[d] + ia) : 0.0;
      r_hi[d] = (d < D && ib < row1) ? __ldcg(rs[d] + ib) : 0.0;
    }
  }

#if !FPFP_PROJ_RING_FIRST
  const uint32_t row_bytes = (uint32_t)min(kProjTC, (int)(p.ldY - colbase)) * 4u;
  float* wbuf = ring_st.buf + (size_t)warp * kSlots * kProjTC;
  uint64_t* wbar = ring_st.bar + warp * kSlots;
  const uint32_t seq0 = ring_st.seq;
  const int i0 = row0 + warp;
  const int nrows_w = i0 < row1 ? (row1 - i0 + kWarps - 1) / kWarps : 0;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (lane == 0) {
#pragma unroll 1
    for (int k = 0; k < kSlots && k < nrows_w; ++k) {
      const uint32_t slot = (seq0 + k) % kSlots;
      ring_issue(wbar + slot, wbuf + slot * kProjTC, p.Y + (int64_t)(i0 + k * kWarps) * p.ldY + colbase,
                 row_bytes);
    }
  }
  __syncwarp();
#endif
  for (int tg = 0; tg < nrows_w; tg += 4) {
    double rq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u4 = 0; u4 < 4; ++u4) {
      const int t = tg + u4;
      if (t >= nrows_w) break;
      const int i = i0 + t * kWarps;
      const uint32_t slot = (seq0 + t) % kSlots;
      ring_wait(wbar + slot, ((seq0 + t) / kSlots) & 1u);
      float4 cur[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        cur[q] = inrow[q] ? *reinterpret_cast<const float4*>(wbuf + slot * kProjTC + q * 128 + lane * 4)
                          : make_float4(0, 0, 0, 0);
      __syncwarp();
      if (lane == 0 && t + kSlots < nrows_w) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        ring_issue(wbar + slot, wbuf + slot * kProjTC, p.Y + (int64_t)(i + kSlots * kWarps) * p.ldY + colbase,
                   row_bytes);
      }
      float* rowp = p.Y + (int64_t)i * p.ldY + colbase + lane * 4;
      float tf[kRC];
#pragma unroll
      for (int d = 0; d < kRC; ++d) {
        const double rlo = __shfl_sync(0xffffffffu, r_lo[d], t & 31);
        const double rhi = __shfl_sync(0xffffffffu, r_hi[d], t & 31);
        tf[d] = (float)(tc[d] - (t < 32 ? rlo : rhi) * inv_m);
      }
      float racc_f = 0.0f;
      float4 xq[kQ];
      const bool xrow = kMu && i < p.n;
      if (kMu) {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int j0 = colbase + q * 128 + lane * 4;
          xq[q] = (xrow && j0 < p.np) ? __ldcs(reinterpret_cast<const float4*>(p.X + (int64_t)i * p.ldX + j0))
                                      : make_float4(0, 0, 0, 0);
        }
      }
      double xrmax = 0.0;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        float* ve = reinterpret_cast<float*>(&cur[q]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = colbase + q * 128 + lane * 4 + e;
          const bool valid = kFull || j < p.m;
          float zp = ve[e];
          float z = fmaxf((zp + tf[0]) - u[0][q][e], 0.0f);   // P1 + P2 (fp32)
#pragma unroll
          for (int d = 1; d < kRC; ++d)
            if (d < D) {
              zp = z;
              z = fmaxf((zp + tf[d]) - u[d][q][e], 0.0f);
            }
          if (!valid) {   // outside m: stays 0 (delta as tile_pass: against the stored value)
            z = 0.0f;
            zp = ve[e];
          }
          dmax = fmaxf(dmax, fabsf(z - zp));                   // delta
          ve[e] = z;
          racc_f += z;
          colf[q][e] += z;
          if (kMu && xrow && j < p.np) {
            const double xt = blend_xt(p.alpha, 1.0 - p.alpha, reinterpret_cast<const float*>(&xq[q])[e], z);
            *mu_acc = fmax(*mu_acc, xt);
            xrmax = fmax(xrmax, fabs(xt));
          }
        }
      }
      if (kMu && p.xrowmax) {
        const double v = warp_max(xrmax);
        if (lane == 0 && xrow) atomicMax(p.xrowmax + i, (unsigned long long)__double_as_longlong(v));
      }
      if (write) {
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (inrow[q]) __stcg(reinterpret_cast<float4*>(rowp + q * 128), cur[q]);
      }
      rq[u4] = (double)racc_f;
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    double k0 = b4 ? rq[2] : rq[0], k1 = b4 ? rq[3] : rq[1];
    k0 += __shfl_xor_sync(0xffffffffu, b4 ? rq[0] : rq[2], 16);
    k1 += __shfl_xor_sync(0xffffffffu, b4 ? rq[1] : rq[3], 16);
    double k = b3 ? k1 : k0;
    k += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    const int rsel = (b4 ? 2 : 0) + (b3 ? 1 : 0);
    if ((lane & 7) == 0 && tg + rsel < nrows_w)
      p.rowpart[(int64_t)cb * p.rows + i0 + (tg + rsel) * kWarps] = k;
  }
  ring_st.seq = seq0 + (uint32_t)nrows_w;
#pragma unroll
  for (int q = 0; q < kQ; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) sm.col[warp][q * 128 + lane * 4 + e] = (double)colf[q][e];
  __syncthreads();
  for (int jj = threadIdx.x; jj < kProjTC; jj += kProjThreads) {
    const int j = colbase + jj;
    if (j < p.m) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += sm.col[w][jj];
      p.colpart[(int64_t)rb * p.m + j] = s;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void replay_tile(const ProjArgs& p, int t, int D, bool write, bool mu_fused,
                                            const double* const (&rs)[kRC], const double* const (&cs)[kRC],
                                            const double (&tc)[kRC], float& dmax, ProjSmem& sm, Ring& ring,
                                            double& mu) {
  const int rb = t / p.CB, cb = t - rb * p.CB;
  const bool full = (cb + 1) * kProjTC <= p.m;
  if (mu_fused && rb * p.TR < p.n && cb * kProjTC < p.np) {
    if (full) replay_pass<true, true>(p, t, D, write, rs, cs, tc, dmax, sm, ring, &mu);
    else replay_pass<false, true>(p, t, D, write, rs, cs, tc, dmax, sm, ring, &mu);
  } else {
    if (full) replay_pass<true, false>(p, t, D, write, rs, cs, tc, dmax, sm, ring, nullptr);
    else replay_pass<false, false>(p, t, D, write, rs, cs, tc, dmax, sm, ring, nullptr);
  }
}
#endif

// one sweep over a tile: the bounds-free variant when all 512 columns are inside m
__device__ __forceinline__ void sweep_tile(const ProjArgs& p, int t, double sigma, float& dmax,
                                           ProjSmem& sm, Ring& ring) {
  const int cb = t - (t / p.CB) * p.CB;
  if ((cb + 1) * kProjTC <= p.m) tile_pass<true, true>(p, t, sigma, dmax, sm, ring);
  else tile_pass<true, false>(p, t, sigma, dmax, sm, ring);
}
// the last sweep with the fused mu pass (tiles with no row of the X block take the plain sweep)
__device__ __forceinline__ void sweep_tile_mu(const ProjArgs& p, int t, double sigma, float& dmax,
                                              ProjSmem& sm, Ring& ring, double& mu) {
  const int rb = t / p.CB, cb = t - rb * p.CB;
  if (rb * p.TR >= p.n || cb * kProjTC >= p.np) { sweep_tile(p, t, sigma, dmax, sm, ring); return; }
  if ((cb + 1) * kProjTC <= p.m) tile_pass<true, true, true>(p, t, sigma, dmax, sm, ring, &mu);
  else tile_pass<true, false, true>(p, t, sigma, dmax, sm, ring, &mu);
}

// r_i = sum_cb rowpart[cb][i], c_j = sum_rb colpart[rb][j]; one warp per index: lane l sums the
// partials l, l+32, ... and an xor tree combines the lanes (a fixed order => deterministic).
// Per-block partial of sigma = sum of the c_j this block produced (fixed assignment of j to blocks).
__device__ __forceinline__ void reduce_phase(const ProjArgs& p, ProjSmem& sm, double* r_out = nullptr,
                                             double* c_out = nullptr) {
  if (!r_out) r_out = p.r;
  if (!c_out) c_out = p.c;
  // one thread per column / row, partials summed in block order (coalesced across threads,
  // independent loads in flight; fixed order => deterministic)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  double local = 0.0;
  for (int j = gt; j < p.m; j += nt) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int rb = 0;
    for (; rb + 4 <= p.RB; rb += 4) {
      s0 += __ldcg(p.colpart + (int64_t)(rb + 0) * p.m + j);
      s1 += __ldcg(p.colpart + (int64_t)(rb + 1) * p.m + j);
      s2 += __ldcg(p.colpart + (int64_t)(rb + 2) * p.m + j);
      s3 += __ldcg(p.colpart + (int64_t)(rb + 3) * p.m + j);
    }
    for (; rb < p.RB; ++rb) s0 += __ldcg(p.colpart + (int64_t)rb * p.m + j);
    const double s = (s0 + s1) + (s2 + s3);
    c_out[j] = s;
    local += s;
  }
  for (int i = gt; i < p.rows; i += nt) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int cb = 0;
    for (; cb + 4 <= p.CB; cb += 4) {
      s0 += __ldcg(p.rowpart + (int64_t)(cb + 0) * p.rows + i);
      s1 += __ldcg(p.rowpart + (int64_t)(cb + 1) * p.rows + i);
      s2 += __ldcg(p.rowpart + (int64_t)(cb + 2) * p.rows + i);
      s3 += __ldcg(p.rowpart + (int64_t)(cb + 3) * p.rows + i);
    }
    for (; cb < p.CB; ++cb) s0 += __ldcg(p.rowpart + (int64_t)cb * p.rows + i);
    r_out[i] = (s0 + s1) + (s2 + s3);
  }
  local = warp_sum(local);
  if (lane == 0) sm.red[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += sm.red[w];
    p.sig_part[blockIdx.x] = s;
  }
  __syncthreads();
}

// sigma = sum_b sig_part[b] (fixed order; identical in every block), broadcast through smem.
__device__ __forceinline__ double grid_sigma(const ProjArgs& p, ProjSmem& sm) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += p.sig_part[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) sm.bcast[0] = s;
  }
  __syncthreads();
  const double v = sm.bcast[0];
  __syncthreads();
  return v;
}

template <typename T>
__device__ __forceinline__ T block_max(T v, ProjSmem& sm, T init) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm.red[warp] = (double)v;
  __syncthreads();
  T r = init;
  if (threadIdx.x == 0) {
    for (int w = 0; w < kWarps; ++w) r = max(r, (T)sm.red[w]);
    sm.bcast[1] = (double)r;
  }
  __syncthreads();
  r = (T)sm.bcast[1];
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T grid_max(const T* parts, ProjSmem& sm, T init) {
  if (threadIdx.x < 32) {
    T v = init;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) v = max(v, parts[b]);
    v = warp_max(v);
    if (threadIdx.x == 0) sm.bcast[2] = (double)v;
  }
  __syncthreads();
  const T r = (T)sm.bcast[2];
  __syncthreads();
  return r;
}

// Block 0 folds the per-block sigma partials (fixed order) into c[m] (the dist all-reduce buffer).
__device__ __forceinline__ void publish_sigma(const ProjArgs& p, ProjSmem& sm) {
  if (blockIdx.x == 0) {
    const double sg = grid_sigma(p, sm);
    if (threadIdx.x == 0) p.c[p.m] = sg;
  }
}

// X~ = (1 - alpha) X + alpha Y[0:n, 0:n'] (Algorithm 1 line 8) and its local max (line 9's mu).
__device__ __forceinline__ double finalize_mu(const ProjArgs& p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ftiles = p.RBx * p.CBx;
  const double a = p.alpha, b = 1.0 - p.alpha;
  double mu_loc = -INFINITY;
  for (int t = blockIdx.x; t < ftiles; t += gridDim.x) {
    const int rb = t / p.CBx, cb = t - (t / p.CBx) * p.CBx;
    const int row1 = min(p.n, (rb + 1) * p.TR);
    for (int i = rb * p.TR + warp; i < row1; i += kWarps) {
      double rmx = 0.0;   // max |X~| of this row segment (for the fused digit planes)
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int j0 = cb * kProjTC + q * 128 + lane * 4;
        if (j0 >= p.np) continue;
        const float4 xv = *reinterpret_cast<const float4*>(p.X + (int64_t)i * p.ldX + j0);
        const float4 yv = *reinterpret_cast<const float4*>(p.Y + (int64_t)i * p.ldY + j0);
        const float* xe = reinterpret_cast<const float*>(&xv);
        const float* ye = reinterpret_cast<const float*>(&yv);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (j0 + e < p.np) {
            const double xt = blend_xt(a, b, xe[e], ye[e]);
            mu_loc = fmax(mu_loc, xt);
            rmx = fmax(rmx, fabs(xt));
          }
      }
      if (p.xrowmax) {
        rmx = warp_max(rmx);
        // nonnegative doubles order as their bit patterns
        if (lane == 0) atomicMax(p.xrowmax + i, (unsigned long long)__double_as_longlong(rmx));
      }
    }
  }
  return mu_loc;
}

// X = X~ / mu (if rescale), TF32 split of X, local max |X_new - X_old|.
__device__ __forceinline__ float finalize_apply(const ProjArgs& p, double mu) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ftiles = p.RBx * p.CBx;
  const double a = p.alpha, b = 1.0 - p.alpha;
  // X~ / mu as a product with the fp64 reciprocal (one DMUL instead of a DDIV per element; the
  // result rounded to fp32 equals fl32(X~ / mu) except within 2^-53 of an fp32 rounding boundary)
  const double rcp = p.rescale ? 1.0 / mu : 1.0;
  float rho_loc = 0.0f;
  for (int t = blockIdx.x; t < ftiles; t += gridDim.x) {
    const int rb = t / p.CBx, cb = t - (t / p.CBx) * p.CBx;
    const int row1 = min(p.n, (rb + 1) * p.TR);
    for (int i = rb * p.TR + warp; i < row1; i += kWarps) {
      // fused digits of the new X (int8 path): the row's scale is the exponent of
      // max_j |fl32(X~_ij / mu)| = fl32(max_j |X~_ij| / mu) (rounding is monotonic), i.e. exactly
      // what split_i8_kernel would derive from the stored row
      float dinv = 0.0f;
      if (p.xd[0]) {
        const float rmax = (float)(__longlong_as_double((long long)p.xrowmax[i]) * rcp);
        const int ex = frexp_exp(rmax);
        dinv = exp2i(-ex);
        if (cb == 0 && lane == 0) p.xe[i] = ex;
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int j0 = cb * kProjTC + q * 128 + lane * 4;
        if (j0 >= p.np) continue;
        float* xp = p.X + (int64_t)i * p.ldX + j0;
        float4 xv = *reinterpret_cast<const float4*>(xp);
        const float4 yv = *reinterpret_cast<const float4*>(p.Y + (int64_t)i * p.ldY + j0);
        float* xe = reinterpret_cast<float*>(&xv);
        const float* ye = reinterpret_cast<const float*>(&yv);
        float4 bv, sv;
        float* be = reinterpret_cast<float*>(&bv);
        float* se = reinterpret_cast<float*>(&sv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float xn = 0.0f;
          if (j0 + e < p.np) {
            const double xt = blend_xt(a, b, xe[e], ye[e]);
            xn = (float)(xt * rcp);
            // fl32(|xn - xo|) directly in fp32: IEEE subtraction rounds the exact difference, the
            // same value the former fp64 difference rounded to fp32 gave (2 conversions fewer)
            rho_loc = fmaxf(rho_loc, fabsf(xn - xe[e]));
          }
          xe[e] = xn;
          be[e] = tf32_rna(xn);
          se[e] = tf32_rna(xn - be[e]);
        }
        *reinterpret_cast<float4*>(xp) = xv;
        if (p.xd[0]) {   // 4 consecutive columns -> one packed word per digit plane
          int a4[4], b4[4], c4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) ozaki_digits3(xe[e], dinv, a4[e], b4[e], c4[e]);
          const int64_t o = (int64_t)i * p.ldxd + j0;
          auto pk = [](const int (&d)[4]) {
            return (d[0] & 0xFF) | ((d[1] & 0xFF) << 8) | ((d[2] & 0xFF) << 16) | ((d[3] & 0xFF) << 24);
          };
          *reinterpret_cast<int*>(p.xd[0] + o) = pk(a4);
          *reinterpret_cast<int*>(p.xd[1] + o) = pk(b4);
          *reinterpret_cast<int*>(p.xd[2] + o) = pk(c4);
        }
        if (p.split) {
          *reinterpret_cast<float4*>(p.Xb + (int64_t)i * p.ldX + j0) = bv;
          *reinterpret_cast<float4*>(p.Xs + (int64_t)i * p.ldX + j0) = sv;
        }
      }
    }
  }
  return rho_loc;
}

// Tile schedule of one pass (pass index `pass`, counted from the launch): with p.tile_ctr every block
// fetches tiles from one atomic counter. Each pass costs the counter exactly ntiles + gridDim.x
// increments (every block's last fetch fails), and passes are separated by grid barriers, so pass
// `pass` owns the counter range [pass (ntiles + grid), ...) without resetting it.
template <typename F>
__device__ __forceinline__ void for_tiles(const ProjArgs& p, int ntiles, unsigned pass, unsigned* s_tile,
                                          F&& body) {
  if (!p.tile_ctr) {
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) body(t);
    return;
  }
  const unsigned base = pass * (unsigned)(ntiles + gridDim.x);
  for (;;) {
    if (threadIdx.x == 0) *s_tile = atomicAdd(p.tile_ctr, 1u) - base;
    __syncthreads();
    const unsigned t = *s_tile;
    __syncthreads();
    if (t >= (unsigned)ntiles) break;
    body((int)t);
  }
}

__global__ void __launch_bounds__(kProjThreads, 2) proj_kernel(ProjArgs p) {
  if (*p.done) return;  // an earlier iteration of this launch batch converged (uniform)
  cg::grid_group grid = cg::this_grid();
  __shared__ ProjSmem sm;
  Ring ring{nullptr, nullptr, 0};
#if FPFP_PROJ_BULK
  extern __shared__ __align__(128) float ring_smem[];
  __shared__ __align__(8) uint64_t ring_bar[kWarps * kSlots];
  ring.buf = ring_smem;
  ring.bar = ring_bar;
  if (threadIdx.x < kWarps * kSlots)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&ring_bar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
#endif
  const int ntiles = p.RB * p.CB;
  float dummy = 0.0f;
  __shared__ unsigned s_tile;

  // ------------------------------------------------------------------ distributed phases
  if (p.mode == kProjSums) {            // sums of the local rows of Y -> c_local, r, sigma_local
    for_tiles(p, ntiles, 0u, &s_tile, [&](int t) { tile_pass<false>(p, t, 0.0, dummy, sm, ring); });
    grid.sync();
    reduce_phase(p, sm);
    grid.sync();
    publish_sigma(p, sm);
    return;
  }
  if (p.mode == kProjOneSweep) {        // one P1+P2 sweep with the global c, sigma = c[m]
    if (p.inner) {                      // device-side inner stop test (reading A5)
      if (p.inner[1]) return;
      if (p.inner[0] > 0 && p.scal[0] < p.eps2) {   // same values in every block: uniform
        grid.sync();                    // every block has read inner[] before it changes
        if (blockIdx.x == 0 && threadIdx.x == 0) p.inner[1] = 1;
        return;
      }
    }
    const double sigma = p.c[p.m];
    float dmax = 0.0f;
    for_tiles(p, ntiles, 0u, &s_tile, [&](int t) { sweep_tile(p, t, sigma, dmax, sm, ring); });
    dmax = block_max(dmax, sm, 0.0f);
    if (threadIdx.x == 0) p.dlt_part[blockIdx.x] = dmax;
    grid.sync();
    reduce_phase(p, sm);
    grid.sync();
    publish_sigma(p, sm);
    if (blockIdx.x == 0) {
      const float d = grid_max(p.dlt_part, sm, 0.0f);
      if (threadIdx.x == 0) {
        p.scal[0] = (double)d;
        if (p.inner) p.inner[0] += 1;
      }
    }
    return;
  }
  if (p.mode == kProjFinMu) {           // local max of X~
    double mu_loc = block_max(finalize_mu(p), sm, (double)-INFINITY);
    if (threadIdx.x == 0) p.mu_part[blockIdx.x] = mu_loc;
    grid.sync();
    if (blockIdx.x == 0) {
      const double mu = grid_max(p.mu_part, sm, (double)-INFINITY);
      if (threadIdx.x == 0) p.scal[1] = mu;
    }
    return;
  }
  if (p.mode == kProjFinApply) {        // apply with the global mu = scal[1]
    const double mu = p.scal[1];
    if (!(mu > 1e-300)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) p.scal[2] = -1.0;   // degenerate marker
      return;
    }
    float rho_loc = block_max(finalize_apply(p, mu), sm, 0.0f);
    if (threadIdx.x == 0) p.rho_part[blockIdx.x] = rho_loc;
    grid.sync();
    if (blockIdx.x == 0) {
      const float rho = grid_max(p.rho_part, sm, 0.0f);
      if (threadIdx.x == 0) p.scal[2] = (double)rho;
    }
    return;
  }

  // ------------------------------------------------------------------ single GPU: everything
  unsigned pass = 0;
  if (p.do_sums) {
    // sums of the current Y (fresh GEMM block + retained slack)
    for_tiles(p, ntiles, pass++, &s_tile, [&](int t) { tile_pass<false>(p, t, 0.0, dummy, sm, ring); });
    grid.sync();
    reduce_phase(p, sm);
    grid.sync();
  }
  double sigma = grid_sigma(p, sm);

  int sweeps = 0;
  float delta = 0.0f;
  bool mu_fused = false;
  double mu_loc = -INFINITY;
  // checkpointed sweeps (replay_pass): the sums of generation g (of Z_g) live in buffer g & 1
#if FPFP_PROJ_BULK
  const bool replay = p.replay != 0;
#else
  const bool replay = false;
#endif
  // generation g (the sums of Z_g) lives in slot g % kRC of r [kRC][rows], c [kRC][m + 1], sig
  auto rbuf = [&](int g) { return p.r + (int64_t)(g % kRC) * p.rows; };
  auto cbuf = [&](int g) { return p.c + (int64_t)(g % kRC) * (p.m + 1); };
  double sig[kRC];
  sig[0] = sigma;
  bool stored = true;   // Z of the last sweep is in Y
#ifdef FPFP_PROJ_PROF
  unsigned long long pt[4] = {0, 0, 0, 0}, tmin = ~0ull, tmax = 0;
  auto gt = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  unsigned long long tq = gt();
#endif
  for (;;) {
    float dmax = 0.0f;
    const int k = sweeps + 1;   // this sweep
    // the cap's last sweep is known in advance: it also reduces mu (the eps2 stop is not)
    mu_fused = p.do_finalize && sweeps + 1 >= p.max_iter2;
    if (!replay || k == 1) {
      if (mu_fused) {
        for_tiles(p, ntiles, pass++, &s_tile, [&](int t) { sweep_tile_mu(p, t, sigma, dmax, sm, ring, mu_loc); });
      } else {
        for_tiles(p, ntiles, pass++, &s_tile, [&](int t) { sweep_tile(p, t, sigma, dmax, sm, ring); });
      }
    } else {
#if FPFP_PROJ_BULK
      // the stored checkpoints are Z_1, Z_{1+kRC}, Z_{1+2kRC}, ... and the cap's last sweep: sweep k
      // re-applies D = k - (last checkpoint before k) sweeps and is stored when D == kRC
      const int D = (k - 2) % kRC + 1;
      const bool write = D == kRC || sweeps + 1 >= p.max_iter2;
      const int g0 = k - D;   // generation of the checkpoint
      const double* rs[kRC];
      const double* cs[kRC];
      double tc[kRC];
      const double inv_m = 1.0 / (double)p.m;
#pragma unroll
      for (int d = 0; d < kRC; ++d) {
        const int g = g0 + min(d, D - 1);
        rs[d] = rbuf(g);
        cs[d] = cbuf(g);
        tc[d] = (1.0 + sig[g % kRC] * inv_m) * inv_m;
      }
      for_tiles(p, ntiles, pass++, &s_tile,
                [&](int t) { replay_tile(p, t, D, write, mu_fused, rs, cs, tc, dmax, sm, ring, mu_loc); });
      stored = write;
#endif
    }
    dmax = block_max(dmax, sm, 0.0f);
    if (threadIdx.x == 0) p.dlt_part[blockIdx.x] = dmax;
#ifdef FPFP_PROJ_PROF
    { const unsigned long long t = gt(); pt[0] += t - tq; tmin = min(tmin, t - tq); tmax = max(tmax, t - tq); tq = t; }
#endif
    grid.sync();
#ifdef FPFP_PROJ_PROF
    { const unsigned long long t = gt(); pt[1] += t - tq; tq = t; }
#endif
    if (replay) reduce_phase(p, sm, rbuf(k), cbuf(k));
    else reduce_phase(p, sm);
#ifdef FPFP_PROJ_PROF
    { const unsigned long long t = gt(); pt[2] += t - tq; tq = t; }
#endif
    grid.sync();
    sigma = grid_sigma(p, sm);
    sig[k % kRC] = sigma;
    delta = grid_max(p.dlt_part, sm, 0.0f);
#ifdef FPFP_PROJ_PROF
    { const unsigned long long t = gt(); pt[3] += t - tq; tq = t; }
#endif
    ++sweeps;
    if ((double)delta < p.eps2 || sweeps >= p.max_iter2) break;  // uniform across blocks
  }
#if FPFP_PROJ_BULK
  if (!stored) {   // stopped on delta after a sweep that was not stored: store Z_k
    const int k = sweeps;
    const int D = (k - 2) % kRC + 1, g0 = k - D;
    const double* rs[kRC];
    const double* cs[kRC];
    double tc[kRC];
    const double inv_m = 1.0 / (double)p.m;
#pragma unroll
    for (int d = 0; d < kRC; ++d) {
      const int g = g0 + min(d, D - 1);
      rs[d] = rbuf(g);
      cs[d] = cbuf(g);
      tc[d] = (1.0 + sig[g % kRC] * inv_m) * inv_m;
    }
    float dd = 0.0f;
    for_tiles(p, ntiles, pass++, &s_tile,
              [&](int t) { replay_tile(p, t, D, true, false, rs, cs, tc, dd, sm, ring, mu_loc); });
    grid.sync();
  }
#endif

#ifdef FPFP_PROJ_PROF
  if ((blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && threadIdx.x == 0)
    printf("proj-prof block %d: per sweep (ns): tiles %llu [min %llu max %llu]  sync1 %llu  reduce %llu  sync2+scalars %llu\n",
           blockIdx.x, pt[0] / sweeps, tmin, tmax, pt[1] / sweeps, pt[2] / sweeps, pt[3] / sweeps);
#endif
  if (!p.do_finalize) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.iter_out->valid = 1;
      p.iter_out->sweeps = sweeps;
      p.iter_out->delta = (double)delta;
    }
    return;
  }

  // ---- Algorithm 1 line 8: X~ = (1 - alpha) X + alpha Y[0:n, 0:n'];  line 9: X = X~ / max X~
  // (mu and the row maxima come from the last sweep when it was the cap's; else one more pass)
  if (!mu_fused) mu_loc = finalize_mu(p);
  mu_loc = block_max(mu_loc, sm, (double)-INFINITY);
  if (threadIdx.x == 0) p.mu_part[blockIdx.x] = mu_loc;
  grid.sync();
  const double mu = grid_max(p.mu_part, sm, (double)-INFINITY);
  if (!(mu > 1e-300)) {  // degenerate guard (reading A7): X left unchanged, loop stops
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.iter_out->valid = 1; p.iter_out->sweeps = sweeps; p.iter_out->degenerate = 1;
      p.iter_out->delta = (double)delta; p.iter_out->mu = mu; p.iter_out->rho = 0.0;
      *p.done = 1;
    }
    return;
  }
  float rho_loc = block_max(finalize_apply(p, mu), sm, 0.0f);
  if (threadIdx.x == 0) p.rho_part[blockIdx.x] = rho_loc;
  grid.sync();
  if (blockIdx.x == 0) {
    const float rho = grid_max(p.rho_part, sm, 0.0f);
    if (threadIdx.x == 0) {
      p.iter_out->valid = 1; p.iter_out->sweeps = sweeps; p.iter_out->degenerate = 0;
      p.iter_out->delta = (double)delta; p.iter_out->mu = mu; p.iter_out->rho = (double)rho;
      const int conv = (double)rho < p.eps1;
      p.iter_out->converged = conv;
      if (conv) *p.done = 1;
    }
  }
}

__global__ void split_kernel(const float* __restrict__ src, int64_t lds, float* __restrict__ big,
                             float* __restrict__ small, int64_t ldd, int rows, int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / cols), j = (int)(k - (k / cols) * cols);
    const float a = src[(int64_t)i * lds + j];
    const float hb = tf32_rna(a);
    big[(int64_t)i * ldd + j] = hb;
    small[(int64_t)i * ldd + j] = tf32_rna(a - hb);
  }
}

__global__ void check_sym_kernel(const float* __restrict__ A, int64_t lda, int n, int* flags) {
  const int64_t total = (int64_t)n * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (k / n) * n);
    const float a = A[(int64_t)i * lda + j];
    if (!isfinite(a)) atomicOr(flags, 2);
    if (j > i && a != A[(int64_t)j * lda + i]) atomicOr(flags, 1);
  }
}

__global__ void check_finite_kernel(const float* __restrict__ A, int64_t lda, int rows, int cols,
                                    int* flags) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / cols), j = (int)(k - (k / cols) * cols);
    if (!isfinite(A[(int64_t)i * lda + j])) atomicOr(flags, 2);
  }
}

__global__ void fill_kernel(float* A, int64_t lda, int rows, int cols, float v) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / cols), j = (int)(k - (k / cols) * cols);
    A[(int64_t)i * lda + j] = v;
  }
}

// zero every entry of Y (rows x m) outside the X block [0:n, 0:n'] (slack_mode = reset)
__global__ void zero_slack_kernel(float* Y, int64_t ldY, int rows, int m, int n, int np,
                                  const int* done) {
  if (done && *done) return;
  const int64_t total = (int64_t)rows * m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / m), j = (int)(k - (k / m) * m);
    if (i >= n || j >= np) Y[(int64_t)i * ldY + j] = 0.0f;
  }
}

// out2[0] = sum X∘G, out2[1] = sum X∘K (fp64). Grid reduction in a fixed order: block b sums rows
// b, b + kDotBlocks, ... (lanes stride the columns) into part[2b], part[2b+1]; dot2_finish adds the
// partials in block order, so the value is reproducible for a given shape.
__global__ void __launch_bounds__(256) dot2_kernel(const float* X, const float* G, const float* K,
                                                   int64_t ld, int rows, int cols, double* part) {
  double s0 = 0.0, s1 = 0.0;
  for (int i = blockIdx.x; i < rows; i += gridDim.x) {
    const float* x = X + (int64_t)i * ld;
    const float* g = G + (int64_t)i * ld;
    const float* k = K ? K + (int64_t)i * ld : nullptr;
    for (int j = threadIdx.x; j < cols; j += blockDim.x) {
      const double xv = x[j];
      s0 += xv * (double)g[j];
      if (k) s1 += xv * (double)k[j];
    }
  }
  __shared__ double r0[8], r1[8];
  s0 = warp_sum(s0); s1 = warp_sum(s1);
  if ((threadIdx.x & 31) == 0) { r0[threadIdx.x >> 5] = s0; r1[threadIdx.x >> 5] = s1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) { a += r0[w]; b += r1[w]; }
    part[2 * blockIdx.x] = a; part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void dot2_finish(const double* part, int nblk, double* out2) {
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < nblk; ++q) { a += part[2 * q]; b += part[2 * q + 1]; }
    out2[0] = a; out2[1] = b;
  }
}

inline int grid_for(int64_t total) {
  return (int)std::min<int64_t>(4096, std::max<int64_t>(1, ceil_div(total, 256)));
}

}  // namespace

int proj_replay_default() {
  static const int v = [] {
    const char* e = getenv("FPFP_PROJ_REPLAY");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

int proj_max_grid(int device) {
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
  cudaFuncSetAttribute(proj_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, proj_kernel, kProjThreads, kRingBytes);
  return sms * std::max(per_sm, 0);
}

cudaError_t launch_proj(const ProjArgs& a, int grid, cudaStream_t s) {
  ProjArgs copy = a;
  void* args[] = {&copy};
  cudaError_t e = cudaFuncSetAttribute(proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(proj_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel((void*)proj_kernel, dim3(grid), dim3(kProjThreads), args, kRingBytes, s);
}

cudaError_t launch_split(const float* src, int64_t lds, float* big, float* small, int64_t ldd,
                         int rows, int cols, cudaStream_t s) {
  split_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(src, lds, big, small, ldd, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_check_sym(const float* A, int64_t lda, int n, int* flags, cudaStream_t s) {
  check_sym_kernel<<<grid_for((int64_t)n * n), 256, 0, s>>>(A, lda, n, flags);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* A, int64_t lda, int rows, int cols, int* flags,
                                cudaStream_t s) {
  check_finite_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(A, lda, rows, cols, flags);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* A, int64_t lda, int rows, int cols, float v, cudaStream_t s) {
  fill_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(A, lda, rows, cols, v);
  return cudaGetLastError();
}

cudaError_t launch_zero_slack(float* Y, int64_t ldY, int rows, int m, int n, int np,
                              const int* done, cudaStream_t s) {
  zero_slack_kernel<<<grid_for((int64_t)rows * m), 256, 0, s>>>(Y, ldY, rows, m, n, np, done);
  return cudaGetLastError();
}

cudaError_t launch_dot2(const float* X, const float* G, const float* K, int64_t ld, int rows,
                        int cols, double* part, double* out2, cudaStream_t s) {
  const int nblk = std::max(1, std::min(rows, kDotBlocks));
  dot2_kernel<<<nblk, 256, 0, s>>>(X, G, K, ld, rows, cols, part);
  dot2_finish<<<1, 32, 0, s>>>(part, nblk, out2);
  return cudaGetLastError();
}

}  // namespace fpfp
