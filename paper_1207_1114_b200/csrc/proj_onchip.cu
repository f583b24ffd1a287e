// proj_onchip.cu — the projection loop (Algorithm 1 lines 4-7) plus blend/rescale
// (lines 8-9) for m small enough that Y fits in the GPU's aggregate shared memory (m <~ 2.7k:
// BASELINE configs[1] and [2], n ~ 1000). Same arithmetic as proj.cu (fp64 sums and correction,
// one rounding to fp32 per sweep), different schedule: Y is split into PR x PC tiles, one per CTA,
// read from HBM/L2 once, kept in shared memory across all sweeps and written back once.
//
// Each sweep: update the own tile with the row sums r_i (own rows), column sums c_j (own columns)
// and sigma of the previous Y; emit fp64 partial row/column sums of the new tile, its total and its
// delta to a double-buffered global exchange; ONE grid barrier; every CTA then re-reduces just the
// partials of its own rows / columns (PC and PR values each) and the PR*PC totals in a fixed order,
// so every CTA holds bit-identical r, c, sigma and delta (deterministic, no float atomics). The
// streaming kernel (proj.cu) needs two barriers per sweep; at n ~ 1000 the barrier is the cost.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fpfp {
namespace {

#ifndef FPFP_OC_THREADS
#define FPFP_OC_THREADS 256
#endif
constexpr int kThreads = FPFP_OC_THREADS;
#ifndef FPFP_OC_UNROLL
#define FPFP_OC_UNROLL 2
#endif
constexpr int kRowUnroll = FPFP_OC_UNROLL;   // rows of the element loop in flight per warp
constexpr int kWarps = kThreads / 32;

struct OcShared {
  double colsum[kWarps][kOnchipMaxTC];
  double r[kOnchipMaxTC];     // own rows' sums
  double c[kOnchipMaxTC];     // own columns' sums
  double red[kWarps];
  float dred[kWarps];
  double bc[4];
};

template <int NQ>   // column chunks of 32 per lane: TCo <= 32 * NQ
__global__ void __launch_bounds__(kThreads, 1) proj_onchip_kernel(OnchipArgs p) {
  if (*p.done) return;
  cg::grid_group grid = cg::this_grid();
  // The tile is held in fp64 on chip (no per-sweep rounding: closer to the fp64 definition than
  // the streaming kernel's fp32 storage); it is rounded to fp32 once, when written back.
  // Rows of the shared tile are padded to kLdt = 32 NQ columns: padded entries are 0 and their
  // column correction is +1e300, so P2 keeps them at 0 and the element loop needs no bounds test.
  constexpr int kLdt = 32 * NQ;
  extern __shared__ __align__(16) double tile[];   // [TRo][kLdt]
  __shared__ OcShared sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const int pr = b / p.PC, pc = b - (b / p.PC) * p.PC;
  const int r0 = pr * p.TRo, c0 = pc * p.TCo;
  const int nr = max(0, min(p.m, r0 + p.TRo) - r0);
  const int nc = max(0, min(p.m, c0 + p.TCo) - c0);
  const int nb = p.PR * p.PC;
  const double inv_m = 1.0 / (double)p.m;

  // load the tile
  for (int i = warp; i < nr; i += kWarps)
    for (int j = lane; j < kLdt; j += 32)
      tile[i * kLdt + j] = j < nc ? (double)p.Y[(int64_t)(r0 + i) * p.ldY + c0 + j] : 0.0;
  __syncthreads();

  // One fused pass over the tile: optionally apply the sweep (P1 then P2, fp64 correction, one
  // rounding), and emit the fp64 row / column partial sums, the tile total and the tile delta of
  // the resulting values to exchange buffer `buf`. Latency, not bandwidth, bounds this kernel at
  // n ~ 1000, so the element loop carries no cross-lane reduction and no fp64
  // max chain: warp w walks rows w, w+8, ...; lane l keeps its columns' partial sums in registers
  // and writes its per-row partial to shared memory (rowacc[i][l]); the 32 lane partials of a row
  // and the 8 warp partials of a column are then summed by one thread each, in a fixed order.
  // P2 is a sign test (max(z, 0) for finite z), the delta is tracked in fp32: rounding is
  // monotonic, so max_ij fl32(|dz|) = fl32(max_ij |dz|), the same value the fp64 max would give.
  double* rowacc = tile + (size_t)p.TRo * kLdt;   // [TRo][33]
#ifdef FPFP_OC_PROF
  long long pc_rows = 0, pc_cols = 0;
#endif
  auto pass = [&](bool update, int buf, double tconst) {
#ifdef FPFP_OC_PROF
    const long long c0_ = clock64();
#endif
    double cacc[NQ], cj[NQ];
    float dq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      cacc[q] = 0.0;
      dq[q] = 0.0f;
      const int j = lane + 32 * q;
      cj[q] = j < nc ? sh.c[j] * inv_m : 1e300;
    }
    if (update) {
#pragma unroll kRowUnroll
      for (int i = warp; i < nr; i += kWarps) {
        const double ti = tconst - sh.r[i] * inv_m;
        double* row = &tile[i * kLdt + lane];
        double y[NQ], z[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) y[q] = row[32 * q];
        double racc = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          double v = (y[q] + ti) - cj[q];                          // P1 (fp64)
          z[q] = __double2hiint(v) < 0 ? 0.0 : v;                  // P2
          dq[q] = fmaxf(dq[q], (float)fabs(z[q] - y[q]));
          racc += z[q];
          cacc[q] += z[q];
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) row[32 * q] = z[q];
        rowacc[i * 33 + lane] = racc;
      }
    } else {
#pragma unroll 2
      for (int i = warp; i < nr; i += kWarps) {
        const double* row = &tile[i * kLdt + lane];
        double racc = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const double y = row[32 * q];
          racc += y;
          cacc[q] += y;
        }
        rowacc[i * 33 + lane] = racc;
      }
    }
    float dmax = 0.0f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) dmax = fmaxf(dmax, dq[q]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) sh.colsum[warp][lane + 32 * q] = cacc[q];
    dmax = warp_max(dmax);
    if (lane == 0) sh.dred[warp] = dmax;
    __syncthreads();
#ifdef FPFP_OC_PROF
    const long long c1_ = clock64();
    pc_rows += c1_ - c0_;
#endif
    // row partials (own rows) and column partials (own columns), fixed order
    double rsum = 0.0;
    for (int t = threadIdx.x; t < nr; t += kThreads) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int l = 0; l < 32; l += 4) {
        s0 += rowacc[t * 33 + l]; s1 += rowacc[t * 33 + l + 1];
        s2 += rowacc[t * 33 + l + 2]; s3 += rowacc[t * 33 + l + 3];
      }
      const double rs = (s0 + s1) + (s2 + s3);
      if (nb == 1) sh.r[t] = rs;   // one tile: the sums stay on chip (the element loop is done)
      else p.rowp[((int64_t)buf * p.PC + pc) * p.m + r0 + t] = rs;
      rsum += rs;
    }
    for (int j = threadIdx.x; j < nc; j += kThreads) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += sh.colsum[w][j];
      if (nb == 1) sh.c[j] = s;
      else p.colp[((int64_t)buf * p.PR + pr) * p.m + c0 + j] = s;
    }
    rsum = warp_sum(rsum);
    if (lane == 0) sh.red[warp] = rsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      float d = 0.0f;
      for (int w = 0; w < kWarps; ++w) { t += sh.red[w]; d = fmaxf(d, sh.dred[w]); }
      if (nb == 1) {
        sh.bc[0] = t;
        sh.bc[1] = (double)d;
      } else {
        p.tot[buf * nb + b] = t;
        p.dlt[buf * nb + b] = d;
      }
    }
#ifdef FPFP_OC_PROF
    pc_cols += clock64() - c1_;
#endif
  };

  // r (own rows), c (own columns), sigma, delta from exchange buffer `buf`, in a fixed order.
  // Every load is independent and issued before any is consumed (one L2 round trip): thread t
  // sums the PC partials of row t and the PR partials of column t in registers; warp 7 sums the
  // tile totals and deltas. Loads bypass L1 (__ldcg): the buffers are rewritten every other sweep.
  constexpr int kMaxTilesPerLane = 5;   // PR * PC <= 160
  constexpr int kMaxP = 12;             // PR, PC <= 12
  auto absorb = [&](int buf, double& sigma, float& delta) {
    const int t = threadIdx.x;
    double rv[kMaxP], cv[kMaxP];
    const double* rsrc = p.rowp + (int64_t)buf * p.PC * p.m + r0 + t;
    const double* csrc = p.colp + (int64_t)buf * p.PR * p.m + c0 + t;
#pragma unroll
    for (int q = 0; q < kMaxP; ++q) {
      rv[q] = (t < nr && q < p.PC) ? __ldcg(rsrc + (int64_t)q * p.m) : 0.0;
      cv[q] = (t < nc && q < p.PR) ? __ldcg(csrc + (int64_t)q * p.m) : 0.0;
    }
    double tv[kMaxTilesPerLane];
    float dv[kMaxTilesPerLane];
    if (warp == kWarps - 1) {
#pragma unroll
      for (int u = 0; u < kMaxTilesPerLane; ++u) {
        const int k = lane + 32 * u;
        tv[u] = k < nb ? __ldcg(p.tot + buf * nb + k) : 0.0;
        dv[u] = k < nb ? __ldcg(p.dlt + buf * nb + k) : 0.0f;
      }
    }
    if (t < nr) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxP; ++q) s += rv[q];
      sh.r[t] = s;
    }
    if (t < nc) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxP; ++q) s += cv[q];
      sh.c[t] = s;
    }
    if (warp == kWarps - 1) {
      double s = 0.0;
      float d = 0.0f;
#pragma unroll
      for (int u = 0; u < kMaxTilesPerLane; ++u) { s += tv[u]; d = fmaxf(d, dv[u]); }
      s = warp_sum(s);
      d = warp_max(d);
      if (lane == 0) { sh.bc[0] = s; sh.bc[1] = (double)d; }
    }
    __syncthreads();
    sigma = sh.bc[0];
    delta = (float)sh.bc[1];
  };

  // Grid barrier for the exchange: a monotonic arrival counter (zeroed by the host before the
  // launch), release on arrival, acquire on the poll (cheaper than cg::grid sync's fence + reset).
  unsigned phase = 0;
  auto exchange_barrier = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++phase;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p.bar), "r"(1u) : "memory");
      const unsigned target = (unsigned)nb * phase;
      unsigned v;
#ifdef FPFP_OC_RELAXED_POLL
      // poll without acquire (an acquire load invalidates L1 on every try), then one acquire fence
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.bar) : "memory");
      } while (v < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.bar) : "memory");
      } while (v < target);
#endif
    }
    __syncthreads();
  };

  // a single tile (m <= kOnchipSingleTile) needs no exchange: its sums are already in shared memory
  auto exchange = [&](int bufx, double& sigma_, float& delta_) {
    if (nb == 1) {
      __syncthreads();
      sigma_ = sh.bc[0];
      delta_ = (float)sh.bc[1];
      return;
    }
    exchange_barrier();
    absorb(bufx, sigma_, delta_);
  };
  int buf = 0;
  double sigma;
  float delta;
  pass(false, buf, 0.0);
  exchange(buf, sigma, delta);

  int sweeps = 0;
#ifdef FPFP_OC_PROF
  long long pc_bar = 0, pc_abs = 0;
  pc_rows = pc_cols = 0;
#endif
  for (;;) {
    buf ^= 1;
    pass(true, buf, (1.0 + sigma * inv_m) * inv_m);
#ifdef FPFP_OC_PROF
    const long long b0_ = clock64();
#endif
    if (nb > 1) exchange_barrier();
#ifdef FPFP_OC_PROF
    const long long b1_ = clock64();
    pc_bar += b1_ - b0_;
#endif
    if (nb > 1) {
      absorb(buf, sigma, delta);
    } else {
      __syncthreads();
      sigma = sh.bc[0];
      delta = (float)sh.bc[1];
    }
#ifdef FPFP_OC_PROF
    pc_abs += clock64() - b1_;
#endif
    ++sweeps;
    if ((double)delta < p.eps2 || sweeps >= p.max_iter2) break;
  }
#ifdef FPFP_OC_PROF
  if ((b == 0 || b == nb - 1) && threadIdx.x == 0)
    printf("oc-prof block %d: %d sweeps, clk/sweep: element loop %lld, partials %lld, barrier %lld, absorb %lld\n",
           b, sweeps, pc_rows / sweeps, pc_cols / sweeps, pc_bar / sweeps, pc_abs / sweeps);
#endif

  // write the tile back in fp32 (slack persists across outer iterations, reading A3)
  for (int i = warp; i < nr; i += kWarps)
    for (int j = lane; j < nc; j += 32) p.Y[(int64_t)(r0 + i) * p.ldY + c0 + j] = (float)tile[i * kLdt + j];
  if (!p.do_finalize) {
    if (b == 0 && threadIdx.x == 0) {
      p.iter_out->valid = 1; p.iter_out->sweeps = sweeps; p.iter_out->delta = (double)delta;
    }
    return;
  }

  // ---- Algorithm 1 lines 8-9 on the tile's part of the X block
  const double a = p.alpha, bb = 1.0 - p.alpha;
  const int xr = max(0, min(p.n, r0 + p.TRo) - r0);
  const int xc = max(0, min(p.np, c0 + p.TCo) - c0);
  double mu_loc = -INFINITY;
  for (int i = warp; i < xr; i += kWarps)
    for (int j = lane; j < xc; j += 32) {
      const double xt = bb * (double)p.X[(int64_t)(r0 + i) * p.ldX + c0 + j] + a * tile[i * kLdt + j];
      mu_loc = fmax(mu_loc, xt);
    }
  mu_loc = warp_max(mu_loc);
  if (lane == 0) sh.red[warp] = mu_loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = -INFINITY;
    for (int w = 0; w < kWarps; ++w) mx = fmax(mx, sh.red[w]);
    p.mu_part[b] = mx;
  }
  grid.sync();
  if (warp == 0) {
    double mx = -INFINITY;
    for (int k = lane; k < nb; k += 32) mx = fmax(mx, p.mu_part[k]);
    mx = warp_max(mx);
    if (lane == 0) sh.bc[2] = mx;
  }
  __syncthreads();
  const double mu = sh.bc[2];
  if (!(mu > 1e-300)) {   // degenerate guard (reading A7)
    if (b == 0 && threadIdx.x == 0) {
      p.iter_out->valid = 1; p.iter_out->sweeps = sweeps; p.iter_out->degenerate = 1;
      p.iter_out->delta = (double)delta; p.iter_out->mu = mu; p.iter_out->rho = 0.0;
      *p.done = 1;
    }
    return;
  }
  const double rcp = p.rescale ? 1.0 / mu : 1.0;   // one reciprocal, a DMUL per element
  float rho_loc = 0.0f;
  for (int i = warp; i < xr; i += kWarps)
    for (int j = lane; j < xc; j += 32) {
      const int64_t o = (int64_t)(r0 + i) * p.ldX + c0 + j;
      const float xo = p.X[o];
      const double xt = bb * (double)xo + a * tile[i * kLdt + j];
      const float xn = (float)(xt * rcp);
      rho_loc = fmaxf(rho_loc, fabsf(xn - xo));   // = fl32(|xn - xo|), as the fp64 difference rounded
      p.X[o] = xn;
      const float hb = tf32_rna(xn);
      p.Xb[o] = hb;
      p.Xs[o] = tf32_rna(xn - hb);
    }
  rho_loc = warp_max(rho_loc);
  if (lane == 0) sh.red[warp] = (double)rho_loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.0f;
    for (int w = 0; w < kWarps; ++w) mx = fmaxf(mx, (float)sh.red[w]);
    p.rho_part[b] = mx;
  }
  grid.sync();
  if (b == 0 && warp == 0) {
    float mx = 0.0f;
    for (int k = lane; k < nb; k += 32) mx = fmaxf(mx, p.rho_part[k]);
    mx = warp_max(mx);
    if (lane == 0) {
      p.iter_out->valid = 1; p.iter_out->sweeps = sweeps; p.iter_out->degenerate = 0;
      p.iter_out->delta = (double)delta; p.iter_out->mu = mu; p.iter_out->rho = (double)mx;
      const int conv = (double)mx < p.eps1;
      p.iter_out->converged = conv;
      if (conv) *p.done = 1;
    }
  }
}

}  // namespace

static size_t onchip_smem(int TRo, int TCo, int PR, int PC) {
  (void)PR; (void)PC;
  const size_t ldt = (size_t)round_up(TCo, 32);                      // kLdt of the kernel
  return ((size_t)TRo * ldt + (size_t)TRo * 33) * sizeof(double);    // tile + lane row partials
}

using KernFn = void (*)(OnchipArgs);
static KernFn onchip_kernel_for(int TCo) {
  switch ((TCo + 31) / 32) {
    case 1: return proj_onchip_kernel<1>;
    case 2: return proj_onchip_kernel<2>;
    case 3: return proj_onchip_kernel<3>;
    case 4: return proj_onchip_kernel<4>;
    case 5: return proj_onchip_kernel<5>;
    case 6: return proj_onchip_kernel<6>;
    case 7: return proj_onchip_kernel<7>;
    default: return proj_onchip_kernel<8>;
  }
}

#ifndef FPFP_OC_SINGLE_TILE
#define FPFP_OC_SINGLE_TILE 128   // m up to which the whole Y is one CTA's tile (no grid exchange)
#endif
bool onchip_fits(int m, int num_sms, int& PR, int& PC, int& TRo, int& TCo) {
  int side = 1;
  while ((side + 1) * (side + 1) <= num_sms) ++side;          // 12 x 12 on 148 SMs
  const int want = (int)ceil_div(m, 32);                      // at least 32 x 32 per tile
  PR = PC = m <= FPFP_OC_SINGLE_TILE ? 1 : std::max(1, std::min(side, want));
  TRo = (int)ceil_div(m, PR);
  TCo = (int)round_up(ceil_div(m, PC), 4);
  if (TCo > kOnchipMaxTC || TRo > kOnchipMaxTC || PR * PC > 160 || PR > 12 || PC > 12) return false;
  const size_t smem = onchip_smem(TRo, TCo, PR, PC);
  if (smem > 190 * 1024) return false;
  // every tile's CTA must be co-resident (cooperative launch); static + dynamic shared memory
  // beyond 48 KB needs the opt-in attribute
  KernFn k = onchip_kernel_for(TCo);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem) != cudaSuccess)
    return false;
  return (int64_t)per_sm * num_sms >= (int64_t)PR * PC;
}

cudaError_t launch_proj_onchip(const OnchipArgs& a, cudaStream_t s) {
  const size_t smem = onchip_smem(a.TRo, a.TCo, a.PR, a.PC);
  KernFn k = onchip_kernel_for(a.TCo);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  OnchipArgs copy = a;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel((void*)k, dim3(a.PR * a.PC), dim3(kThreads), args, smem, s);
}

}  // namespace fpfp
