// ga.cu — FastGA's normalisation step: the stabilised exponential of the
// Graduated-Assignment update `{GAO3}` X = exp(beta A X A') (Appendix "FastGA"; the
// exponent A X A' + lambda K comes from the same two tcgen05 GEMMs as FastPFP) followed by the
// slack-padded Sinkhorn normalisation and the outer-iteration bookkeeping, as ONE
// persistent cooperative kernel per outer iteration. Readings G1-G8 are listed in DESIGN.md §3b.
//
// Sinkhorn in scaling form: with E_ij = exp(beta (Q^_ij - c_i)) (c_i = row max of the padded
// compatibility Q^, slack entries Q^ = 0), the s-th sweep output is S^s = diag(u^s) E diag(v^s),
//   u^s_i = 1 / sum_j E_ij v^{s-1}_j       (rows to 1)      v^0 = 1
//   v^s_j = 1 / sum_i u^s_i E_ij            (columns to 1),
// exactly the literal row-then-column normalisation of S^{s-1} (the row factor of S^{s-1} cancels).
// delta_s = max_ij E_ij |u^s_i v^s_j - u^{s-1}_i v^{s-1}_j| = max|S^s - S^{s-1}| (reading G4).
//
// E is stored once per outer iteration in fp64 (m x m, HBM; L2-resident at m ~ 1k) so that entries
// far below the row maximum survive until the column step rescales them (reading G8); u, v and
// all sums are fp64. One sweep is two passes over E with one grid barrier after each:
//   pass R: one warp per full row: u_i = 1 / sum_j E_ij v_j  (+ the lagged delta_{s-1})
//   pass C: one block per chunk of W columns (all rows): v_j = 1 / sum_i u_i E_ij
// so no partial sums cross blocks: every sum has one fixed order (bitwise reproducible). The
// final pass writes X = u E v on the n x n' block with its TF32 split for the next GEMM1 and
// rho = max|X_new - X_old|. u and v are double-buffered by sweep parity for the lagged delta.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fpfp {

namespace {

constexpr int kGaThreads = 256;
constexpr int kGaWarps = kGaThreads / kWarp;

struct GaSmem {
  double col[kGaWarps][32];
  double red[kGaWarps];
};

__device__ __forceinline__ double block_max_d(double v, GaSmem& sm) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sm.red[warp] = v;
  __syncthreads();
  double r = sm.red[0];
  for (int w = 1; w < kGaWarps; ++w) r = max(r, sm.red[w]);
  return r;
}

__device__ __forceinline__ double grid_max_d(const double* parts, GaSmem& sm) {
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kGaThreads) v = max(v, __ldcg(parts + b));
  return block_max_d(v, sm);
}

// compatibility of padded entry (i, j): the GEMM output on the n x n' block, 0 on slack (G2)
__device__ __forceinline__ double qhat(const GaArgs& p, int i, int j) {
  return (i < p.n && j < p.np) ? (double)__ldcg(p.Q + (int64_t)i * p.ldQ + j) : 0.0;
}

__device__ __forceinline__ double* ubuf(const GaArgs& p, int s) { return p.u + (int64_t)(s & 1) * p.ldE; }
__device__ __forceinline__ double* vbuf(const GaArgs& p, int s) { return p.v + (int64_t)(s & 1) * p.ldE; }

// pass R of sweep s+1 (one warp per row): u^{s+1}_i = 1 / sum_j E_ij v^s_j, written to ubuf(s+1);
// with lagged = true also returns this row's part of delta_s = max_j E_ij |u^s_i v^s_j -
// u^{s-1}_i v^{s-1}_j| (read before ubuf(s+1) = ubuf(s-1) is overwritten by this same warp).
__device__ __forceinline__ double pass_r(const GaArgs& p, int s, bool lagged) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kGaWarps + warp, nw = gridDim.x * kGaWarps;
  const double* v = vbuf(p, s);
  const double* vo = vbuf(p, s - 1);
  constexpr int kU = 8;   // loads in flight per lane (the pass is L2-latency bound at m ~ 1k)
  double dl = 0.0;
  for (int i = gw; i < p.m; i += nw) {
    const double* e = p.E + (int64_t)i * p.ldE;
    const double us = lagged ? __ldcg(ubuf(p, s) + i) : 0.0;
    const double uo = lagged ? __ldcg(ubuf(p, s - 1) + i) : 0.0;
    double acc = 0.0;
    for (int j0 = 0; j0 < p.m; j0 += 32 * kU) {
      double ev[kU], vj[kU], vk[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int j = j0 + q * 32 + lane;
        const bool ok = j < p.m;
        ev[q] = ok ? __ldcg(e + j) : 0.0;
        vj[q] = ok ? __ldcg(v + j) : 0.0;
        vk[q] = (ok && lagged) ? __ldcg(vo + j) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        acc += ev[q] * vj[q];
        if (lagged) dl = max(dl, ev[q] * fabs(us * vj[q] - uo * vk[q]));
      }
    }
    acc = warp_sum(acc);
    __syncwarp();
    if (lane == 0) ubuf(p, s + 1)[i] = 1.0 / acc;
  }
  return dl;
}

// pass C of sweep s (one block per chunk of W columns, all rows): v^s_j = 1 / sum_i u^s_i E_ij.
// Lane l of a warp covers column l % W of the chunk and rows (32/W) apart; the per-column sums
// are reduced over lanes (shuffles) and warps (shared memory) in a fixed order.
__device__ __forceinline__ void pass_c(const GaArgs& p, int s, GaSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = p.W, rpw = 32 / W;            // rows per warp step
  const int cl = lane % W, rl = lane / W;
  const double* u = ubuf(p, s);
  double* vout = vbuf(p, s);
  const int nchunks = (int)ceil_div(p.m, W);
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int j = ch * W + cl;
    double acc = 0.0;
    if (j < p.m) {
      constexpr int kU = 8;
      const int step = kGaWarps * rpw;
      for (int i0 = warp * rpw + rl; i0 < p.m; i0 += step * kU) {
        double ui[kU], ei[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
          const int i = i0 + q * step;
          ui[q] = i < p.m ? __ldcg(u + i) : 0.0;
          ei[q] = i < p.m ? __ldcg(p.E + (int64_t)i * p.ldE + j) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) acc += ui[q] * ei[q];
      }
    }
    for (int o = W; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane < W) sm.col[warp][lane] = acc;
    __syncthreads();
    if (threadIdx.x < W && ch * W + (int)threadIdx.x < p.m) {
      double c = 0.0;
      for (int w = 0; w < kGaWarps; ++w) c += sm.col[w][threadIdx.x];
      vout[ch * W + threadIdx.x] = 1.0 / c;
    }
    __syncthreads();
  }
}

}  // namespace

__global__ void __launch_bounds__(kGaThreads) ga_kernel(GaArgs p) {
  cg::grid_group grid = cg::this_grid();
  if (*p.done) return;  // earlier iteration converged (uniform across the grid)
  __shared__ GaSmem sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kGaWarps + warp, nw = gridDim.x * kGaWarps;
  const int m = p.m;

  // ---- E = exp(beta (Q^ - c_i)), one warp per row (G3); v^0 = 1 ----
  for (int i = gw; i < m; i += nw) {
    constexpr int kU = 8;
    double c = (i < p.n && p.np >= m) ? -INFINITY : 0.0;   // slack entries contribute Q^ = 0
    if (i < p.n)
      for (int j0 = 0; j0 < p.np; j0 += 32 * kU) {
        double q[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          const int j = j0 + k * 32 + lane;
          q[k] = j < p.np ? qhat(p, i, j) : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) c = max(c, q[k]);
      }
    c = warp_max(c);
    double* e = p.E + (int64_t)i * p.ldE;
    for (int j0 = 0; j0 < m; j0 += 32 * kU) {
      double q[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int j = j0 + k * 32 + lane;
        q[k] = j < m ? qhat(p, i, j) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int j = j0 + k * 32 + lane;
        if (j < m) e[j] = exp(p.beta * (q[k] - c));
      }
    }
    if (lane == 0) vbuf(p, 0)[i] = 1.0;
  }
  grid.sync();

  int s = 0;                // sweeps completed
  double delta = INFINITY;  // delta of the last completed sweep (G4: delta_1 = inf)
  bool stopped = false;
  for (;;) {
    const bool lagged = s >= 2;
    double dl = pass_r(p, s, lagged);       // u^{s+1}, delta_s
    if (lagged) {
      dl = block_max_d(dl, sm);
      if (threadIdx.x == 0) p.dlt_part[blockIdx.x] = dl;
    }
    grid.sync();
    if (lagged) {
      delta = grid_max_d(p.dlt_part, sm);
      if (delta < p.eps2) { stopped = true; break; }   // state s is final: ubuf(s), vbuf(s)
    }
    pass_c(p, s + 1, sm);                   // v^{s+1}
    grid.sync();
    ++s;
    if (s >= p.max_iter2) break;
  }

  // ---- final pass: X = u^s E v^s on the n x n' block and rho; delta_s at the cap (s >= 2) ----
  const bool need_delta = !stopped && s >= 2;
  const double* us_ = ubuf(p, s);
  const double* vs_ = vbuf(p, s);
  const double* uo_ = ubuf(p, s - 1);
  const double* vo_ = vbuf(p, s - 1);
  double rl = 0.0, dl = 0.0;
  for (int i = gw; i < m; i += nw) {
    const double* e = p.E + (int64_t)i * p.ldE;
    const double us = __ldcg(us_ + i);
    const double uo = need_delta ? __ldcg(uo_ + i) : 0.0;
    const int jend = need_delta ? m : (i < p.n ? p.np : 0);
    constexpr int kU = 4;
    for (int j0 = 0; j0 < jend; j0 += 32 * kU) {
      double ev[kU], vj[kU], vk[kU];
      float xo[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int j = j0 + k * 32 + lane;
        const bool ok = j < jend;
        ev[k] = ok ? __ldcg(e + j) : 0.0;
        vj[k] = ok ? __ldcg(vs_ + j) : 0.0;
        vk[k] = (ok && need_delta) ? __ldcg(vo_ + j) : 0.0;
        xo[k] = (ok && i < p.n && j < p.np) ? p.X[(int64_t)i * p.ldX + j] : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int j = j0 + k * 32 + lane;
        if (j >= jend) continue;
        if (need_delta) dl = max(dl, ev[k] * fabs(us * vj[k] - uo * vk[k]));
        if (i < p.n && j < p.np) {
          const float x = (float)(us * ev[k] * vj[k]);
          const int64_t o = (int64_t)i * p.ldX + j;
          rl = max(rl, fabs((double)x - (double)xo[k]));
          p.X[o] = x;
          const float hb = tf32_rna(x);
          p.Xb[o] = hb;
          p.Xs[o] = tf32_rna(x - hb);
        }
      }
    }
  }
  rl = block_max_d(rl, sm);
  if (need_delta) dl = block_max_d(dl, sm);
  if (threadIdx.x == 0) {
    p.rho_part[blockIdx.x] = rl;
    if (need_delta) p.dlt_part[blockIdx.x] = dl;
  }
  grid.sync();
  if (blockIdx.x == 0) {
    const double rho = grid_max_d(p.rho_part, sm);
    if (need_delta) delta = grid_max_d(p.dlt_part, sm);
    if (threadIdx.x == 0) {
      p.iter_out->valid = 1;
      p.iter_out->sweeps = s;
      p.iter_out->degenerate = 0;
      p.iter_out->delta = delta;
      p.iter_out->mu = p.beta;   // GA: the report's mu slot carries beta_t
      p.iter_out->rho = rho;
      const int conv = rho < p.eps1;
      p.iter_out->converged = conv;
      if (conv) *p.done = 1;
    }
  }
}

int ga_max_grid(int device) {
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ga_kernel, kGaThreads, 0);
  // one CTA per SM: the sweep is barrier-latency bound at m ~ 1k, and a grid barrier over more
  // resident CTAs costs more than the extra memory parallelism buys
  return per_sm >= 1 ? sms : 0;
}

// column-chunk width of pass C: the widest W in {32, 16, 8} that still gives every block a chunk
int ga_chunk_width(int m, int grid) {
  for (int w : {32, 16}) if (ceil_div(m, w) >= grid) return w;
  return 8;
}

cudaError_t launch_ga(const GaArgs& a, int grid, cudaStream_t s) {
  GaArgs copy = a;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel((void*)ga_kernel, dim3(grid), dim3(kGaThreads), args, 0, s);
}

}  // namespace fpfp
