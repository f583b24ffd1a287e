// discretize.cu — greedy discretization (Algorithm 1 line 11) on the GPU.
//
// The paper's greedy repeatedly takes the largest live X_ij and strikes row i and column j
// (Steps 1-3). Under a STRICT total order on entries — (value desc, row asc, col asc),
// reading A12 — that sequential result equals the result of repeatedly matching, in parallel, all
// "locally dominant" live entries: (i, j) such that j is the best live column of row i AND i is the
// best live row of column j. (The order's maximum live entry is always locally dominant, so every
// round makes progress, and a locally dominant entry is picked by the sequential greedy before any
// entry that competes with it.) Each round:
//   1. row pass  (one warp per row whose best column died): rbest[i] = argmax over live columns,
//   2. col pass  (first round: tiled over all rows; later: one warp per column whose best row died),
//   3. match     rbest[i] = j and cbest[j] = i  =>  assign[i] = j, strike row i and column j.
// For FastPFP's near-permutation outputs a handful of rounds suffice. Pathological tie chains (e.g.
// a constant matrix needs min(n, n') rounds) are cut off after kMaxRounds rounds or when a round
// matches < 1/64 of the remaining pairs; the remaining live sub-matrix is then finished on the host
// by the literal sort-and-scan of Steps 1-3 (same order), so the result is always exact.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fastpfp.h"
#include "common.cuh"

namespace fpfp {
namespace {

constexpr int kMaxRounds = 64;

// strict order: a beats b  <=>  va > vb, or va == vb and ka < kb (ka, kb: the row or column index)
__device__ __forceinline__ bool beats(float va, int ka, float vb, int kb) {
  return va > vb || (va == vb && ka < kb);
}

__device__ __forceinline__ void warp_argmax(float& v, int& k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int ok = __shfl_xor_sync(0xffffffffu, k, o);
    if (beats(ov, ok, v, k)) { v = ov; k = ok; }
  }
}

struct GreedyState {
  const float* X; int64_t ld; int n, np;
  uint8_t* row_dead; uint8_t* col_dead;
  int* rbest; int* cbest;
  int* assign;
  int* counters;   // [0] matched so far, [1] rows to recompute, [2] cols to recompute
};

// rows whose best column is unknown or dead
__global__ void row_pass(GreedyState g, int full) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < g.n; i += nw) {
    if (g.row_dead[i]) continue;
    const int cur = g.rbest[i];
    if (!full && cur >= 0 && !g.col_dead[cur]) continue;
    const float* row = g.X + (int64_t)i * g.ld;
    float bv = -INFINITY;
    int bk = 0x7fffffff;
    for (int j = lane; j < g.np; j += 32) {
      if (g.col_dead[j]) continue;
      const float v = row[j];
      if (beats(v, j, bv, bk)) { bv = v; bk = j; }
    }
    warp_argmax(bv, bk);
    if (lane == 0) g.rbest[i] = bk == 0x7fffffff ? -1 : bk;
  }
}

// first round: per (row tile, column) partial argmax, then per-column reduction in tile order
__global__ void col_pass_tiles(GreedyState g, int tr, float* pv, int* pk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int rt = blockIdx.y;
  if (j >= g.np) return;
  float bv = -INFINITY;
  int bk = 0x7fffffff;
  if (!g.col_dead[j]) {
    const int i1 = min(g.n, (rt + 1) * tr);
    for (int i = rt * tr; i < i1; ++i) {
      if (g.row_dead[i]) continue;
      const float v = g.X[(int64_t)i * g.ld + j];
      if (beats(v, i, bv, bk)) { bv = v; bk = i; }
    }
  }
  pv[(int64_t)rt * g.np + j] = bv;
  pk[(int64_t)rt * g.np + j] = bk;
}

__global__ void col_pass_reduce(GreedyState g, int ntiles, const float* pv, const int* pk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.np) return;
  float bv = -INFINITY;
  int bk = 0x7fffffff;
  for (int t = 0; t < ntiles; ++t) {
    const float v = pv[(int64_t)t * g.np + j];
    const int k = pk[(int64_t)t * g.np + j];
    if (beats(v, k, bv, bk)) { bv = v; bk = k; }
  }
  g.cbest[j] = (g.col_dead[j] || bk == 0x7fffffff) ? -1 : bk;
}

// later rounds: one warp per live column whose best row died
__global__ void col_pass_warp(GreedyState g) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = gw; j < g.np; j += nw) {
    if (g.col_dead[j]) continue;
    const int cur = g.cbest[j];
    if (cur >= 0 && !g.row_dead[cur]) continue;
    float bv = -INFINITY;
    int bk = 0x7fffffff;
    for (int i = lane; i < g.n; i += 32) {
      if (g.row_dead[i]) continue;
      const float v = g.X[(int64_t)i * g.ld + j];
      if (beats(v, i, bv, bk)) { bv = v; bk = i; }
    }
    warp_argmax(bv, bk);
    if (lane == 0) g.cbest[j] = bk == 0x7fffffff ? -1 : bk;
  }
}

// match mutually-best pairs; they are disjoint (cbest[j] names one row)
__global__ void match_pass(GreedyState g) {
  int local = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    if (g.row_dead[i]) continue;
    const int j = g.rbest[i];
    if (j >= 0 && g.cbest[j] == i) {
      g.assign[i] = j;
      g.row_dead[i] = 1;
      g.col_dead[j] = 1;
      ++local;
    }
  }
  if (local) atomicAdd(&g.counters[0], local);
}

__global__ void init_pass(GreedyState g) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(g.n, g.np); i += gridDim.x * blockDim.x) {
    if (i < g.n) { g.row_dead[i] = 0; g.rbest[i] = -1; g.assign[i] = -1; }
    if (i < g.np) { g.col_dead[i] = 0; g.cbest[i] = -1; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) g.counters[0] = 0;
}

template <typename T>
cudaError_t dalloc(T*& p, size_t count) { return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)); }

}  // namespace
}  // namespace fpfp

using namespace fpfp;

// Host finish of Steps 1-3 on the live sub-matrix (literal sort-and-scan in the same order).
static void host_finish(const float* X, int64_t ldX, int n, int np, std::vector<uint8_t>& row_dead,
                        std::vector<uint8_t>& col_dead, int32_t* assign, int matched, cudaStream_t s,
                        std::string& msg, int& rc) {
  std::vector<int> rows, cols;
  for (int i = 0; i < n; ++i) if (!row_dead[i]) rows.push_back(i);
  for (int j = 0; j < np; ++j) if (!col_dead[j]) cols.push_back(j);
  std::vector<float> hx((size_t)n * np);
  cudaError_t e = cudaMemcpy2DAsync(hx.data(), (size_t)np * sizeof(float), X, ldX * sizeof(float),
                                    (size_t)np * sizeof(float), n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { msg = cudaGetErrorString(e); rc = FASTPFP_ECUDA; return; }
  std::vector<int64_t> order;
  order.reserve(rows.size() * cols.size());
  for (int i : rows) for (int j : cols) order.push_back((int64_t)i * np + j);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (hx[a] != hx[b]) return hx[a] > hx[b];
    return a < b;   // row-major flat index: smaller row, then smaller column
  });
  const int need = std::min(n, np);
  for (size_t k = 0; k < order.size() && matched < need; ++k) {
    const int i = (int)(order[k] / np), j = (int)(order[k] % np);
    if (!row_dead[i] && !col_dead[j]) {
      assign[i] = j; row_dead[i] = 1; col_dead[j] = 1; ++matched;
    }
  }
}

int fpfp_discretize_device(fastpfp_handle* /*h*/, const float* X, int64_t ldX, int n, int np,
                           int32_t* assign, cudaStream_t s, std::string& msg) {
  GreedyState g{};
  g.X = X; g.ld = ldX; g.n = n; g.np = np;
  const int tr = 256;
  const int ntiles = (int)ceil_div(n, tr);
  float* pv = nullptr;
  int* pk = nullptr;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  A(dalloc(g.row_dead, n)); A(dalloc(g.col_dead, np)); A(dalloc(g.rbest, n)); A(dalloc(g.cbest, np));
  A(dalloc(g.assign, n)); A(dalloc(g.counters, 4));
  A(dalloc(pv, (size_t)ntiles * np)); A(dalloc(pk, (size_t)ntiles * np));
  int rc = FASTPFP_OK;
  const int need = std::min(n, np);
  int matched = 0;
  if (e == cudaSuccess) {
    const int blocks = (int)std::min<int64_t>(4096, ceil_div(std::max(n, np), 256));
    init_pass<<<blocks, 256, 0, s>>>(g);
    for (int round = 0; round < kMaxRounds && matched < need; ++round) {
      row_pass<<<(int)std::min<int64_t>(8192, ceil_div((int64_t)n * 32, 256)), 256, 0, s>>>(g, round == 0);
      if (round == 0) {
        col_pass_tiles<<<dim3((unsigned)ceil_div(np, 256), (unsigned)ntiles), 256, 0, s>>>(g, tr, pv, pk);
        col_pass_reduce<<<(unsigned)ceil_div(np, 256), 256, 0, s>>>(g, ntiles, pv, pk);
      } else {
        col_pass_warp<<<(int)std::min<int64_t>(8192, ceil_div((int64_t)np * 32, 256)), 256, 0, s>>>(g);
      }
      match_pass<<<blocks, 256, 0, s>>>(g);
      int now = 0;
      A(cudaMemcpyAsync(&now, g.counters, sizeof(int), cudaMemcpyDeviceToHost, s));
      A(cudaStreamSynchronize(s));
      if (e != cudaSuccess) break;
      const int gained = now - matched;
      matched = now;
      if (matched < need && gained * 64 < need - matched + gained) break;   // stalled: finish on host
    }
    std::vector<int32_t> a(n);
    std::vector<uint8_t> rd(n), cd(np);
    A(cudaMemcpyAsync(a.data(), g.assign, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    A(cudaMemcpyAsync(rd.data(), g.row_dead, n, cudaMemcpyDeviceToHost, s));
    A(cudaMemcpyAsync(cd.data(), g.col_dead, np, cudaMemcpyDeviceToHost, s));
    A(cudaStreamSynchronize(s));
    if (e == cudaSuccess) {
      std::copy(a.begin(), a.end(), assign);
      if (matched < need) host_finish(X, ldX, n, np, rd, cd, assign, matched, s, msg, rc);
    }
  }
  for (void* p : {(void*)g.row_dead, (void*)g.col_dead, (void*)g.rbest, (void*)g.cbest,
                  (void*)g.assign, (void*)g.counters, (void*)pv, (void*)pk})
    if (p) cudaFree(p);
  if (e != cudaSuccess) {
    msg = std::string("discretize: ") + cudaGetErrorString(e);
    return FASTPFP_ECUDA;
  }
  return rc;
}
