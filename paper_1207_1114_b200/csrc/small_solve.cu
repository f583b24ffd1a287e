// small_solve.cu — Algorithm 1 for many small pairs (n, n' <= 128), one pair per CTA,
// entirely on chip: BASELINE configs[3] (8192 pairs of 128) and configs[0] (batch of one n = 64).
//
// Per outer iteration (all in one CTA, no host involvement):
//   T = X A'   (= (A' X^T)^T, A' symmetric)          line 3, SIMT fp32 from shared memory
//   G = A T + lambda K -> Y[0:n, 0:n']               (A symmetric: its rows are the columns needed)
//   repeat Y = max(Y + (1 + sigma/m - r_i - c_j)/m, 0) until max|dY| < eps2 or I_1   lines 4-7
//   X~ = (1-alpha) X + alpha Y[0:n,0:n'];  X = X~ / max X~;  rho = max|dX|          lines 8-9
// Y (m x m, m = max(n, n') <= 128) lives in registers across the whole solve: warp w owns rows
// 16w..16w+15, lane l owns columns l, l+32, l+64, l+96, so row sums are warp reductions and column
// sums one shared-memory exchange per sweep. X is kept transposed in shared memory (Xt[k][i])
// so both GEMMs read their operands along contiguous rows; A, A' rows stream through a cp.async
// double buffer (they stay L2-resident while a CTA works on its pair).
//
// Numerics: at n <= 128 the products are O(10^1-10^2) and the fp32-storage emulation of the
// projection with fp32 sums drifts < 1e-6 from the fp64 oracle on the c4 recipe, so
// the projection arithmetic is fp32 here (the large-m kernel, proj.cu, uses fp64 sums).
#include <algorithm>

#include "common.cuh"

namespace fpfp {

namespace {

constexpr int kT = 256;           // threads
constexpr int kS = 128;           // max n, n', m
constexpr int kLd = kS + 4;       // padded shared-memory row (floats)
constexpr int kKc = 16;           // rows of A / A' per staging chunk

struct SmallSmem {
  float Xt[kS][kLd];              // X transposed: Xt[k][i] = X[i][k]
  float T[kS][kLd];               // T = X A' (row-major), then G = A T + lambda K
  float stage[2][kKc][kLd];       // A / A' row chunks
  float colp[2][8][kS];           // per-warp column partial sums (double buffered)
  float dl[2][8];                 // per-warp delta partials
  float red[8];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// stage rows [k0, k0+16) of a rows x cols row-major matrix (ld = cols) into dst; zero outside.
// 16-byte cp.async when rows are 16-byte aligned (cols % 4 == 0), plain loads otherwise.
__device__ __forceinline__ void stage_rows(float (*dst)[kLd], const float* src, int rows, int cols,
                                           int k0) {
  // 16 rows x 32 float4 = 512 float4, 2 per thread
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int idx = threadIdx.x + kT * h;
    const int r = idx >> 5, q = (idx & 31) * 4;
    const int gr = k0 + r;
    if ((cols & 3) == 0) {
      const bool ok = gr < rows && q < cols;
      cp_async16(&dst[r][q], ok ? src + (int64_t)gr * cols + q : src, ok);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        dst[r][q + e] = (gr < rows && q + e < cols) ? src[(int64_t)gr * cols + q + e] : 0.f;
    }
  }
}

// C[i][j] = sum_k Pt[k][i] * Q[k][j] over k < K, 8 x 8 register tile per thread.
// Pt from shared memory (Xt) or from the staged chunk; Q likewise.
template <bool kPtStaged>
__device__ __forceinline__ void gemm_acc(float (&acc)[8][8], const float (*Pres)[kLd],
                                         const float (*Qres)[kLd], const float* Gsrc, int Grows,
                                         int Gcols, int K, SmallSmem& sm) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  const int nch = (K + kKc - 1) / kKc;
  stage_rows(sm.stage[0], Gsrc, Grows, Gcols, 0);
  cp_async_commit();
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait_all();
    __syncthreads();
    if (ch + 1 < nch) {
      stage_rows(sm.stage[(ch + 1) & 1], Gsrc, Grows, Gcols, (ch + 1) * kKc);
      cp_async_commit();
    }
    const float (*st)[kLd] = sm.stage[ch & 1];
    const int kmax = min(kKc, K - ch * kKc);
    for (int kk = 0; kk < kmax; ++kk) {
      const int k = ch * kKc + kk;
      const float* prow = kPtStaged ? st[kk] : Pres[k];
      const float* qrow = kPtStaged ? Qres[k] : st[kk];
      const float4 a0 = *reinterpret_cast<const float4*>(prow + ty * 8);
      const float4 a1 = *reinterpret_cast<const float4*>(prow + ty * 8 + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(qrow + tx * 8);
      const float4 b1 = *reinterpret_cast<const float4*>(qrow + tx * 8 + 4);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
  }
  __syncthreads();
}

}  // namespace



namespace {

// All 32 lanes hold partial sums v[0..15] of 16 rows; on return every lane holds the full sums.
// Transpose-butterfly (each stage halves the values a lane carries: 8+4+2+1+1 shuffles) followed by
// 16 broadcasts: 32 shuffles instead of 16 x 5. Fixed tree => deterministic.
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
  // the lane with bits (16, 8, 4, 2) = (r3, r2, r1, r0) now holds row r = 8 r3 + 4 r2 + 2 r1 + r0
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int src = (((r >> 3) & 1) << 4) | (((r >> 2) & 1) << 3) | (((r >> 1) & 1) << 2) | ((r & 1) << 1);
    v[r] = __shfl_sync(F, b1, src);
  }
}

// kFull: n = n' = m = 128 (no bounds masks); kDelta: eps2 > 0 (the inner stop needs delta)
template <bool kFull, bool kDelta>
__global__ void __launch_bounds__(kT, 1) small_solve_kernel(SmallArgs p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SmallSmem& sm = *reinterpret_cast<SmallSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int n = p.n, np = p.np, m = p.m;
  const float inv_m = 1.0f / (float)m;

  for (int pair = blockIdx.x; pair < p.batch; pair += gridDim.x) {
    const float* A = p.A + (int64_t)pair * n * n;
    const float* Ap = p.Ap + (int64_t)pair * np * np;
    const float* Kp = p.K ? p.K + (int64_t)pair * n * np : nullptr;
    float* X = p.X + (int64_t)pair * n * np;

    // X -> Xt (transposed, zero padded)
    for (int idx = threadIdx.x; idx < kS * kS; idx += kT) {
      const int i = idx / kS, k = idx % kS;   // Xt[k][i] = X[i][k]
      sm.Xt[k][i] = (i < n && k < np) ? X[(int64_t)i * np + k] : 0.f;
    }
    // Y register tile: rows 16w+r, cols l+32e
    float y[16][4];
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = warp * 16 + r, j = lane + 32 * e;
        y[r][e] = (p.Y && i < m && j < m) ? p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] : 0.f;
      }
    __syncthreads();

    int it = 0, conv = 0, total_sweeps = 0, degen = 0;
    float rho = 0.f;
    for (; it < p.max_iter1;) {
      float acc[8][8];
      // ---- T = X A' : Pt = Xt (resident), Q = A' rows (staged), K over n'
      gemm_acc<false>(acc, sm.Xt, nullptr, Ap, np, np, np, sm);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        *reinterpret_cast<float4*>(&sm.T[ty * 8 + i][tx * 8]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(&sm.T[ty * 8 + i][tx * 8 + 4]) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
      __syncthreads();
      // ---- G = A T (+ lambda K): Pt = A rows (staged; A symmetric), Q = T (resident), K over n
      gemm_acc<true>(acc, nullptr, sm.T, A, n, n, n, sm);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gi = ty * 8 + i;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int gj = tx * 8 + j;
          if (Kp && gi < n && gj < np) acc[i][j] += p.lam * Kp[(int64_t)gi * np + gj];
        }
        *reinterpret_cast<float4*>(&sm.T[gi][tx * 8]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(&sm.T[gi][tx * 8 + 4]) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
      __syncthreads();
      // Y[0:n, 0:n'] = G ; slack entries keep their values (reading A3)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = warp * 16 + r;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (i < n && lane + 32 * e < np) y[r][e] = sm.T[i][lane + 32 * e];
      }

      // ---- projection loop (P1 + P2 per sweep), sums of the current Y first
      int buf = 0;
      float rs[16], cs[4];
      auto sums = [&](float (&yy)[16][4]) {
        // row partials (4 columns per lane) -> all-lane xor reduction per row
#pragma unroll
        for (int r = 0; r < 16; ++r) rs[r] = (yy[r][0] + yy[r][1]) + (yy[r][2] + yy[r][3]);
        rows_allreduce16(rs);
        // column partials over this warp's 16 rows
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float s = 0.f;
#pragma unroll
          for (int r = 0; r < 16; ++r) s += yy[r][e];
          sm.colp[buf][warp][lane + 32 * e] = s;
        }
      };
      sums(y);
      float dmax = 0.f;
      if (lane == 0) sm.dl[buf][warp] = 0.f;
      __syncthreads();
      int s = 0;
      float delta = 0.f;
      for (;;) {
        // combine column partials (fixed warp order), sigma
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float c = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) c += sm.colp[buf][w][lane + 32 * e];
          cs[e] = c;
        }
        const float sigma = warp_sum((cs[0] + cs[1]) + (cs[2] + cs[3]));
        const float tconst = (1.0f + sigma * inv_m) * inv_m;
        float cu[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) cu[e] = cs[e] * inv_m;
        buf ^= 1;
        dmax = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int i = warp * 16 + r;
          const float ti = tconst - rs[r] * inv_m;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = lane + 32 * e;
            const float yo = y[r][e];
            const float z = (kFull || (i < m && j < m)) ? fmaxf((yo + ti) - cu[e], 0.f) : 0.f;  // P1, P2
            if (kDelta) dmax = fmaxf(dmax, fabsf(z - yo));
            y[r][e] = z;
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
          for (int w = 0; w < 8; ++w) delta = fmaxf(delta, sm.dl[buf][w]);
        }
        ++s;
        if (delta < p.eps2 || s >= p.max_iter2) break;
      }
      total_sweeps += s;

      // ---- blend + rescale (lines 8-9); X~ kept in registers over this thread's tile
      float xt[16][4];
      float mu = -INFINITY;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = warp * 16 + r;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = lane + 32 * e;
          const bool ok = i < n && j < np;
          const float xo = ok ? sm.Xt[j][i] : 0.f;
          xt[r][e] = (1.0f - p.alpha) * xo + p.alpha * y[r][e];
          if (ok) mu = fmaxf(mu, xt[r][e]);
        }
      }
      mu = warp_max(mu);
      if (lane == 0) sm.red[warp] = mu;
      __syncthreads();
      mu = -INFINITY;
#pragma unroll
      for (int w = 0; w < 8; ++w) mu = fmaxf(mu, sm.red[w]);
      __syncthreads();
      if (!(mu > 1e-30f)) { degen = 1; break; }   // degenerate guard (reading A7), X unchanged
      const float scale = p.rescale ? mu : 1.0f;
      float rl = 0.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = warp * 16 + r;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = lane + 32 * e;
          if (i < n && j < np) {
            const float xn = xt[r][e] / scale;
            rl = fmaxf(rl, fabsf(xn - sm.Xt[j][i]));
            sm.Xt[j][i] = xn;
          }
        }
      }
      rl = warp_max(rl);
      if (lane == 0) sm.red[warp] = rl;
      __syncthreads();
      rho = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) rho = fmaxf(rho, sm.red[w]);
      __syncthreads();
      ++it;
      if (rho < p.eps1) { conv = 1; break; }
    }

    // write back X (and Y when slack exists)
    for (int idx = threadIdx.x; idx < n * np; idx += kT) {
      const int i = idx / np, k = idx % np;
      X[idx] = sm.Xt[k][i];
    }
    if (p.Y) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = warp * 16 + r, j = lane + 32 * e;
          if (i < m && j < m) p.Y[(int64_t)pair * m * m + (int64_t)i * m + j] = y[r][e];
        }
    }
    if (threadIdx.x == 0) {
      p.iters[pair] = it; p.conv[pair] = conv; p.sweeps[pair] = total_sweeps;
      p.rho[pair] = rho; p.degen[pair] = degen;
    }
    __syncthreads();
  }
}

// Greedy discretization of one small pair per CTA: min(n, n') rounds of a block-wide
// argmax over the live entries under the strict order (value desc, row asc, col asc).
__global__ void __launch_bounds__(kT) small_greedy_kernel(const float* X, int batch, int n, int np,
                                                          int32_t* assign) {
  __shared__ unsigned char row_dead[kS], col_dead[kS];
  __shared__ float bv[8];
  __shared__ int bi[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pair = blockIdx.x; pair < batch; pair += gridDim.x) {
    const float* Xp = X + (int64_t)pair * n * np;
    for (int i = threadIdx.x; i < kS; i += kT) { row_dead[i] = 0; col_dead[i] = 0; }
    for (int i = threadIdx.x; i < n; i += kT) assign[(int64_t)pair * n + i] = -1;
    __syncthreads();
    const int need = min(n, np);
    for (int pick = 0; pick < need; ++pick) {
      float best = -INFINITY;
      int bidx = 0x7fffffff;
      for (int idx = threadIdx.x; idx < n * np; idx += kT) {
        const int i = idx / np, j = idx % np;
        if (row_dead[i] || col_dead[j]) continue;
        const float v = Xp[idx];
        if (v > best || (v == best && idx < bidx)) { best = v; bidx = idx; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
      }
      if (lane == 0) { bv[warp] = best; bi[warp] = bidx; }
      __syncthreads();
      if (threadIdx.x == 0) {
        float b = bv[0]; int k = bi[0];
        for (int w = 1; w < 8; ++w)
          if (bv[w] > b || (bv[w] == b && bi[w] < k)) { b = bv[w]; k = bi[w]; }
        const int i = k / np, j = k % np;
        assign[(int64_t)pair * n + i] = j;
        row_dead[i] = 1;
        col_dead[j] = 1;
      }
      __syncthreads();
    }
  }
}

}  // namespace

size_t small_smem_bytes() { return sizeof(SmallSmem); }

cudaError_t launch_small_solve(const SmallArgs& a, int grid, cudaStream_t s) {
  const bool full = a.n == kS && a.np == kS;
  const bool delta = a.eps2 > 0.0f;
  void (*k)(SmallArgs) = full ? (delta ? small_solve_kernel<true, true> : small_solve_kernel<true, false>)
                              : (delta ? small_solve_kernel<false, true> : small_solve_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmallSmem));
  if (e != cudaSuccess) return e;
  k<<<grid, kT, sizeof(SmallSmem), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_small_greedy(const float* X, int batch, int n, int np, int32_t* assign, int grid,
                                cudaStream_t s) {
  small_greedy_kernel<<<grid, kT, 0, s>>>(X, batch, n, np, assign);
  return cudaGetLastError();
}

}  // namespace fpfp
