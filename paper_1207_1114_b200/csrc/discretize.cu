// discretize.cu — greedy discretization (Algorithm 1 line 11), entirely on the GPU.
//
// The paper's greedy repeatedly takes the largest live X_ij and strikes row i and column j
// (Steps 1-3). Under a STRICT total order on entries — (value desc, row asc, col asc),
// reading A12 — that sequential result equals the result of repeatedly matching, in parallel, all
// "locally dominant" live entries: (i, j) such that j is the best live column of row i AND i is the
// best live row of column j. (The order's maximum live entry is always locally dominant, so every
// round makes progress, and a locally dominant entry is picked by the sequential greedy before any
// entry that competes with it.)
//
// Phase 1 — `rounds_kernel`, ONE cooperative launch: round 0 computes every row's and column's best
// live partner (full passes over X), later rounds recompute only the rows / columns whose partner
// died, and every round matches the mutually-best pairs. For FastPFP's near-permutation outputs a
// handful of rounds finish the job. Tie chains (e.g. a constant matrix needs min(n, n') rounds, each
// rescanning every live row) are detected on the device: a round that matches < 1/64 of the
// remaining pairs stops phase 1.
// Phase 2 (only after such a stall) — the literal Steps 1-3 on the live sub-matrix, on the device:
// compact the live rows and columns (ordered), build one 64-bit key per live entry
// (~order(value) << 32 | row-major rank among the live entries), sort the keys (cub radix sort, the
// one library primitive here), and scan them in order with one CTA: a window of 1024 keys is
// skipped when no entry in it is live; otherwise its live entries are taken one at a time in key
// order, each striking its row and column for the rest of the window.
// The host only launches, and reads the assignment back (one synchronisation in the common case).
#include <algorithm>
#include <cstdint>
#include <string>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "../../include/fastpfp.h"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace fpfp {
namespace {

constexpr int kThreads = 256;
constexpr int kColTile = 256;   // round 0 column pass: rows per partial

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

// counters: [0] pairs matched, [1] phase-1 stalled flag, [2] rounds run, [3] live rows,
// [4] live cols (phase 2 compaction cursors)
struct Greedy {
  const float* X; int64_t ld; int n, np;
  uint8_t* row_dead; uint8_t* col_dead;
  int* rbest; int* cbest;
  int* assign;
  int* ctr;
  float* pv; int* pk;      // round 0 column partials [ceil(n / kColTile)][np]
};

__device__ void row_best(const Greedy& g, int i, int lane) {
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

__device__ void col_best(const Greedy& g, int j, int lane) {
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

__global__ void __launch_bounds__(kThreads) rounds_kernel(Greedy g) {
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthr = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int gw = tid >> 5, nw = nthr >> 5;
  const int need = min(g.n, g.np);
  volatile int* vctr = g.ctr;
  for (int i = tid; i < max(g.n, g.np); i += nthr) {
    if (i < g.n) { g.row_dead[i] = 0; g.assign[i] = -1; }
    if (i < g.np) g.col_dead[i] = 0;
  }
  if (tid < 5) g.ctr[tid] = 0;
  grid.sync();
  // round 0: every row's best column (one warp per row) and every column's best row (coalesced
  // row tiles of partials, then a per-column reduction in tile order)
  for (int i = gw; i < g.n; i += nw) row_best(g, i, lane);
  const int ntiles = (int)ceil_div(g.n, kColTile);
  for (int64_t w = tid; w < (int64_t)ntiles * g.np; w += nthr) {
    const int rt = (int)(w / g.np), j = (int)(w - (int64_t)rt * g.np);
    float bv = -INFINITY;
    int bk = 0x7fffffff;
    const int i1 = min(g.n, (rt + 1) * kColTile);
    for (int i = rt * kColTile; i < i1; ++i) {
      const float v = g.X[(int64_t)i * g.ld + j];
      if (beats(v, i, bv, bk)) { bv = v; bk = i; }
    }
    g.pv[w] = bv;
    g.pk[w] = bk;
  }
  grid.sync();
  for (int j = tid; j < g.np; j += nthr) {
    float bv = -INFINITY;
    int bk = 0x7fffffff;
    for (int t = 0; t < ntiles; ++t) {
      const float v = g.pv[(int64_t)t * g.np + j];
      const int k = g.pk[(int64_t)t * g.np + j];
      if (beats(v, k, bv, bk)) { bv = v; bk = k; }
    }
    g.cbest[j] = bk == 0x7fffffff ? -1 : bk;
  }
  grid.sync();
  int before = 0;
  for (int round = 0;; ++round) {
    // match the mutually-best pairs (disjoint: cbest[j] names one row)
    int local = 0;
    for (int i = tid; i < g.n; i += nthr) {
      if (g.row_dead[i]) continue;
      const int j = g.rbest[i];
      if (j >= 0 && g.cbest[j] == i) {
        g.assign[i] = j;
        g.row_dead[i] = 1;
        g.col_dead[j] = 1;
        ++local;
      }
    }
    local = warp_sum(local);
    if (lane == 0 && local) atomicAdd(&g.ctr[0], local);
    grid.sync();
    const int now = vctr[0];
    const int gained = now - before;
    before = now;
    if (now >= need) break;
    if (gained * 64 < need - now + gained) {       // tie chain: finish with phase 2
      if (tid == 0) g.ctr[1] = 1;
      break;
    }
    for (int i = gw; i < g.n; i += nw) {
      if (g.row_dead[i]) continue;
      const int cur = g.rbest[i];
      if (cur < 0 || g.col_dead[cur]) row_best(g, i, lane);
    }
    for (int j = gw; j < g.np; j += nw) {
      if (g.col_dead[j]) continue;
      const int cur = g.cbest[j];
      if (cur < 0 || g.row_dead[cur]) col_best(g, j, lane);
    }
    grid.sync();
    if (tid == 0) g.ctr[2] = round + 1;
  }
}

// ---- phase 2 ------------------------------------------------------------------------------------

// ordered compaction of the live rows / columns (one CTA; n, n' are at most a few 10^4 here)
__global__ void __launch_bounds__(1024) compact_kernel(Greedy g, int* live_rows, int* live_cols) {
  __shared__ int base;
  for (int pass = 0; pass < 2; ++pass) {
    const int cnt = pass == 0 ? g.n : g.np;
    const uint8_t* dead = pass == 0 ? g.row_dead : g.col_dead;
    int* out = pass == 0 ? live_rows : live_cols;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int i0 = 0; i0 < cnt; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      const int live = (i < cnt && !dead[i]) ? 1 : 0;
      // block-wide exclusive scan of `live` (warp ballots + per-warp counts)
      __shared__ int wcnt[32];
      const unsigned b = __ballot_sync(0xffffffffu, live);
      const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (lane == 0) wcnt[wid] = __popc(b);
      __syncthreads();
      int off = 0;
      for (int w = 0; w < wid; ++w) off += wcnt[w];
      const int pos = base + off + __popc(b & ((1u << lane) - 1u));
      if (live) out[pos] = i;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wcnt[w];
        base += tot;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) g.ctr[3 + pass] = base;
    __syncthreads();
  }
}

// monotone map float -> uint32 (larger float -> larger key)
__device__ __forceinline__ uint32_t order_bits(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void keys_kernel(Greedy g, const int* live_rows, const int* live_cols, int nr, int nc,
                            uint64_t* keys) {
  const int64_t L = (int64_t)nr * nc;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L; k += (int64_t)gridDim.x * blockDim.x) {
    const int ri = (int)(k / nc), cj = (int)(k - (int64_t)ri * nc);
    const float v = g.X[(int64_t)live_rows[ri] * g.ld + live_cols[cj]];
    keys[k] = ((uint64_t)(~order_bits(v)) << 32) | (uint64_t)k;   // value desc, then (row, col) asc
  }
}

// Steps 1-3 over the sorted keys, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) scan_kernel(Greedy g, const int* live_rows,
                                                    const int* live_cols, int nc, int64_t L,
                                                    const uint64_t* keys) {
  __shared__ int s_i[1024], s_j[1024];
  __shared__ int matched;
  const int need = min(g.n, g.np);
  if (threadIdx.x == 0) matched = g.ctr[0];
  __syncthreads();
  for (int64_t w0 = 0; w0 < L; w0 += blockDim.x) {
    if (matched >= need) break;            // uniform: written before the last __syncthreads
    const int64_t k = w0 + threadIdx.x;
    int i = -1, j = -1;
    if (k < L) {
      const uint32_t idx = (uint32_t)(keys[k] & 0xffffffffu);
      i = live_rows[idx / nc];
      j = live_cols[idx % nc];
      if (g.row_dead[i] || g.col_dead[j]) i = -1;
    }
    s_i[threadIdx.x] = i;
    s_j[threadIdx.x] = j;
    if (!__syncthreads_or(i >= 0)) continue;
    if (threadIdx.x == 0) {                // the window's live entries, in key order
      const int lim = (int)(L - w0 < (int64_t)blockDim.x ? L - w0 : (int64_t)blockDim.x);
      for (int t = 0; t < lim && matched < need; ++t) {
        const int ii = s_i[t], jj = s_j[t];
        if (ii < 0 || g.row_dead[ii] || g.col_dead[jj]) continue;
        g.assign[ii] = jj;
        g.row_dead[ii] = 1;
        g.col_dead[jj] = 1;
        ++matched;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) g.ctr[0] = matched;
}

}  // namespace
}  // namespace fpfp

using namespace fpfp;

// Device scratch of the greedy, owned by a handle (grown on demand, freed with the handle).
struct GreedyScratch {
  uint8_t *row_dead = nullptr, *col_dead = nullptr;
  int *rbest = nullptr, *cbest = nullptr, *assign = nullptr, *ctr = nullptr;
  float* pv = nullptr;
  int* pk = nullptr;
  int *live_rows = nullptr, *live_cols = nullptr;
  int n = 0, np = 0;
  uint64_t *keys = nullptr, *keys_alt = nullptr;
  void* cub_tmp = nullptr;
  size_t keys_cap = 0, cub_cap = 0;
  int grid = 0;
  int* h_ctr = nullptr;   // pinned [5]
};

namespace {
template <typename T>
cudaError_t dalloc(T*& p, size_t count) { return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)); }

void free_base(GreedyScratch& s) {
  for (void* p : {(void*)s.row_dead, (void*)s.col_dead, (void*)s.rbest, (void*)s.cbest,
                  (void*)s.assign, (void*)s.ctr, (void*)s.pv, (void*)s.pk, (void*)s.live_rows,
                  (void*)s.live_cols})
    if (p) cudaFree(p);
  s.row_dead = s.col_dead = nullptr;
  s.rbest = s.cbest = s.assign = s.ctr = s.pk = s.live_rows = s.live_cols = nullptr;
  s.pv = nullptr;
  s.n = s.np = 0;
}
}  // namespace

void fpfp_greedy_free(GreedyScratch* s) {
  if (!s) return;
  free_base(*s);
  for (void* p : {(void*)s->keys, (void*)s->keys_alt, s->cub_tmp}) if (p) cudaFree(p);
  if (s->h_ctr) cudaFreeHost(s->h_ctr);
  delete s;
}

int fpfp_discretize_device(GreedyScratch** scratch, const float* X, int64_t ldX, int n, int np,
                           int32_t* assign, cudaStream_t s, std::string& msg) {
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  if (!*scratch) *scratch = new GreedyScratch();
  GreedyScratch& S = **scratch;
  if (S.n != n || S.np != np) {
    free_base(S);
    const int64_t ntiles = ceil_div(n, kColTile);
    A(dalloc(S.row_dead, n)); A(dalloc(S.col_dead, np)); A(dalloc(S.rbest, n)); A(dalloc(S.cbest, np));
    A(dalloc(S.assign, n)); A(dalloc(S.ctr, 8)); A(dalloc(S.pv, ntiles * np)); A(dalloc(S.pk, ntiles * np));
    A(dalloc(S.live_rows, n)); A(dalloc(S.live_cols, np));
    if (!S.h_ctr) A(cudaMallocHost(&S.h_ctr, 8 * sizeof(int)));
    if (e != cudaSuccess) { free_base(S); msg = cudaGetErrorString(e); return FASTPFP_ENOMEM; }
    S.n = n; S.np = np;
  }
  if (S.grid == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rounds_kernel, kThreads, 0);
    S.grid = sms * std::max(1, std::min(per, 4));
  }
  Greedy g{};
  g.X = X; g.ld = ldX; g.n = n; g.np = np;
  g.row_dead = S.row_dead; g.col_dead = S.col_dead; g.rbest = S.rbest; g.cbest = S.cbest;
  g.assign = S.assign; g.ctr = S.ctr; g.pv = S.pv; g.pk = S.pk;
  void* args[] = {&g};
  A(cudaLaunchCooperativeKernel((void*)rounds_kernel, dim3(S.grid), dim3(kThreads), args, 0, s));
  A(cudaMemcpyAsync(S.h_ctr, S.ctr, 5 * sizeof(int), cudaMemcpyDeviceToHost, s));
  A(cudaStreamSynchronize(s));
  if (e == cudaSuccess && S.h_ctr[1]) {
    // phase 2 on the live sub-matrix
    compact_kernel<<<1, 1024, 0, s>>>(g, S.live_rows, S.live_cols);
    A(cudaMemcpyAsync(S.h_ctr, S.ctr, 5 * sizeof(int), cudaMemcpyDeviceToHost, s));
    A(cudaStreamSynchronize(s));
    const int nr = S.h_ctr[3], nc = S.h_ctr[4];
    const int64_t L = (int64_t)nr * nc;
    if (e == cudaSuccess && L > 0) {
      if (L > 0xffffffffLL) { msg = "discretize: live sub-matrix exceeds 2^32 entries"; return FASTPFP_EUNSUPPORTED; }
      if ((size_t)L > S.keys_cap) {
        if (S.keys) cudaFree(S.keys);
        if (S.keys_alt) cudaFree(S.keys_alt);
        S.keys = S.keys_alt = nullptr;
        S.keys_cap = 0;
        A(dalloc(S.keys, (size_t)L)); A(dalloc(S.keys_alt, (size_t)L));
        if (e != cudaSuccess) { msg = cudaGetErrorString(e); return FASTPFP_ENOMEM; }
        S.keys_cap = (size_t)L;
      }
      cub::DoubleBuffer<uint64_t> db(S.keys, S.keys_alt);
      size_t need_tmp = 0;
      A(cub::DeviceRadixSort::SortKeys(nullptr, need_tmp, db, (int64_t)L, 0, 64, s));
      if (need_tmp > S.cub_cap) {
        if (S.cub_tmp) cudaFree(S.cub_tmp);
        S.cub_tmp = nullptr;
        S.cub_cap = 0;
        A(cudaMalloc(&S.cub_tmp, need_tmp));
        if (e != cudaSuccess) { msg = cudaGetErrorString(e); return FASTPFP_ENOMEM; }
        S.cub_cap = need_tmp;
      }
      const int kb = (int)std::min<int64_t>(8192, ceil_div(L, 256));
      keys_kernel<<<kb, 256, 0, s>>>(g, S.live_rows, S.live_cols, nr, nc, S.keys);
      A(cub::DeviceRadixSort::SortKeys(S.cub_tmp, need_tmp, db, (int64_t)L, 0, 64, s));
      scan_kernel<<<1, 1024, 0, s>>>(g, S.live_rows, S.live_cols, nc, L, db.Current());
      A(cudaGetLastError());
    }
  }
  A(cudaMemcpyAsync(assign, S.assign, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  A(cudaStreamSynchronize(s));
  if (e != cudaSuccess) {
    msg = std::string("discretize: ") + cudaGetErrorString(e);
    return FASTPFP_ECUDA;
  }
  return FASTPFP_OK;
}
