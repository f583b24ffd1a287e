// api.cu — the C-ABI of include/fastpfp.h: handle state, device memory layout and the host-side
// orchestration of Algorithm 1. All arithmetic of the path runs in the kernels of
// proj.cu / gemm_simt.cu / gemm_tc.cu / discretize.cu; this file only allocates, validates,
// launches and copies.
//
// Device layout: every matrix is fp32 row-major with its row stride rounded
// up to 32 floats (128 B) so rows are 16 B aligned for float4 / TMA access; padding is zero.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fastpfp.h"
#include "common.cuh"
#include "nccl_dyn.h"

using namespace fpfp;

struct GreedyScratch;   // discretize.cu

namespace {

constexpr int kMaxCheck = 64;  // max outer iterations per host convergence check
constexpr int kSweepChunk = 8; // sharded path: sweeps enqueued per host check of the inner stop

struct Buf {
  float* p = nullptr;
  int64_t ld = 0;
  int rows = 0, cols = 0;
};

// Ozaki int8 form of a rows x K matrix: 3 digit planes (row stride ld bytes) + row exponents
struct I8Buf {
  int8_t* d[3] = {nullptr, nullptr, nullptr};
  int64_t ld = 0;
  int* e = nullptr;
  int rows = 0, K = 0;
};

}  // namespace

struct fastpfp_handle {
  // n: rows of A/X/K held by this handle (= n_glob on one GPU, n_glob / world when row-sharded)
  int64_t n = 0, np = 0, d = 0, m = 0, n_glob = 0, yrows = 0;
  // row sharding (fastpfp_create_dist): rank r owns rows [r*n, (r+1)*n) of A, X, K, Y
  int rank = 0, world = 1;
  bool dist = false;
  ncclComm_t comm = nullptr;
  const NcclApi* nccl = nullptr;
  int64_t nccl_timeout_ms = 600000;   // FASTPFP_OPT_NCCL_TIMEOUT_MS
  int* inner = nullptr;               // [2] device inner-loop state of the sharded projection
  unsigned* tile_ctr = nullptr;       // projection tile counter (dynamic schedule)
  // collectives issued by the last iterate / objective / discretize call of a sharded handle, in
  // order: {kind (0 all-reduce, 1 all-gather), ncclDataType_t, ncclRedOp_t (-1), count}
  std::vector<std::array<int64_t, 4>> coll_log;
  Buf Uball, Usall;                 // gathered U blocks [world][n'][n]
  int device = 0, num_sms = 0, arch = 0;
  // graphs and their TF32 splits
  Buf A, Ab, As, Ap, Apb, Aps, B, Bp, K;
  // state
  Buf X, Xb, Xs, X0, U, Ub, Us, Y, G;  // G: objective scratch (lazy)
  // projection scratch
  double *rowpart = nullptr, *colpart = nullptr, *r = nullptr, *c = nullptr;
  double *sig_part = nullptr, *mu_part = nullptr;
  float *dlt_part = nullptr, *rho_part = nullptr;
  int TR = 8, RB = 1, CB = 1, RBx = 1, CBx = 1, grid = 1;
  // on-chip projection (proj_onchip.cu)
  bool oc_ok = false;
  int proj_kernel = 0;   // FASTPFP_OPT_PROJ_KERNEL
  int PR = 1, PC = 1, TRo = 1, TCo = 4;
  double *oc_rowp = nullptr, *oc_colp = nullptr, *oc_tot = nullptr;
  float* oc_dlt = nullptr;
  unsigned oc_epoch = 0;           // launch counter: the exchange records' tag epoch
  // Ozaki int8 operands (FASTPFP_OPT_PRECISION = 3, gemm_i8.cu), allocated on first use
  I8Buf Ai8, Api8, Xi8, Ui8, Ui8all;   // Ui8all: gathered U digit planes [world][n'][n/P] (sharded)
  unsigned* Urowmax = nullptr;
  bool i8_ready = false;
  // Xi8 holds the digits of the current X: set by a digit split of X or by the streaming finalize
  // that writes them (int8 path, one GPU); anything else that changes X clears it
  bool xdig_fresh = false;
  unsigned long long* xrowmax = nullptr;   // [n] max |X~| per row (bits), for the fused digits
  // FastGA workspace (ga.cu), allocated on first use of FASTPFP_METHOD_FASTGA
  double *ga_E = nullptr, *ga_u = nullptr, *ga_v = nullptr, *ga_dlt = nullptr, *ga_rho = nullptr;
  int64_t ga_ldE = 0;
  int ga_grid = 0, ga_W = 32;
  double ga_beta0 = 0.5, ga_rate = 1.075, ga_beta_max = 10.0;  // reading G5 defaults
  DevIter* iters = nullptr;       // [kMaxCheck] device
  DevIter* h_iters = nullptr;     // pinned mirror
  // pinned host scratch for small device->host reads on a sharded handle: a read into pageable
  // memory would block inside cudaMemcpyAsync until the stream drains, defeating stream_sync's
  // NCCL fault polling ([0..7] doubles, [8..9] as two ints)
  double* hpin = nullptr;
  int* done = nullptr;            // device flag
  int* flags = nullptr;           // validation flags (device)
  double* scal = nullptr;         // device scalars (objective)
  double* dot_part = nullptr;     // [kDotBlocks][2] objective partials (lazy)
  GreedyScratch* greedy = nullptr;  // discretization scratch (lazy, discretize.cu)
  Buf Xall;                       // gathered X of a sharded handle (lazy, discretize)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int slack_mode = 0, precision = 0, rescale = 1, check_every = 4, cta_group = 2, method = 0;
  bool graphs_set = false, x0_custom = false, poisoned = false;
  int64_t t = 0;
  std::string err;
  // stats / profiling
  fastpfp_stats stats{};
  int profile = 0;
  cudaEvent_t ev[3 * kMaxCheck] = {};
  bool ev_ready = false;
};

namespace {

// NVTX range for the duration of a C-ABI call (header-only NVTX 3: a no-op unless a profiler such as
// nsys is attached), so traces show set_graphs / iterate / discretize around their kernels
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int set_err(fastpfp_handle* h, int code, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
    if (code == FASTPFP_ECUDA || code == FASTPFP_ENCCL) h->poisoned = true;
  }
  return code;
}

#define CK(h, call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return set_err((h), e_ == cudaErrorMemoryAllocation ? FASTPFP_ENOMEM : FASTPFP_ECUDA, \
                     "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,       \
                     __LINE__);                                                              \
  } while (0)

#define GUARD(h)                                                             \
  do {                                                                       \
    if (!(h)) return FASTPFP_EINVAL;                                         \
    if ((h)->poisoned) return FASTPFP_EPOISONED;                             \
    cudaError_t e0_ = cudaSetDevice((h)->device);                            \
    if (e0_ != cudaSuccess) return set_err((h), FASTPFP_ECUDA, "cudaSetDevice: %s", \
                                           cudaGetErrorString(e0_));        \
  } while (0)

#define NK(h, call)                                                                            \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return set_err((h), FASTPFP_ENCCL, "%s failed: %s", #call, (h)->nccl->GetErrorString(r_)); \
  } while (0)

// The sharded path's collectives, logged in issue order (fastpfp_dist_collectives; the schedule the
// gloo decomposition test follows, paper_1207_1114_b200/dist.py collective_schedule).
ncclResult_t coll_allreduce(fastpfp_handle* h, void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op,
                            cudaStream_t s) {
  h->coll_log.push_back({0, (int64_t)t, (int64_t)op, (int64_t)count});
  return h->nccl->AllReduce(buf, buf, count, t, op, h->comm, s);
}
ncclResult_t coll_allgather(fastpfp_handle* h, const void* send, void* recv, size_t count, ncclDataType_t t,
                            cudaStream_t s) {
  h->coll_log.push_back({1, (int64_t)t, -1, (int64_t)count});
  return h->nccl->AllGather(send, recv, count, t, h->comm, s);
}

// Wait for the handle's stream. On a sharded handle the wait polls instead of blocking, so that a
// failed or vanished peer cannot hang the rank (SURVEY §5 failure detection): an asynchronous NCCL
// error, or no completion within nccl_timeout_ms, aborts the communicator (which releases the
// collectives stuck on the stream) and poisons the handle with ENCCL.
int stream_sync(fastpfp_handle* h) {
  if (!h->dist || !h->comm) {
    CK(h, cudaStreamSynchronize(h->stream));
    return FASTPFP_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(h->stream);
    if (q == cudaSuccess) return FASTPFP_OK;
    if (q != cudaErrorNotReady) {
      cudaGetLastError();
      return set_err(h, FASTPFP_ECUDA, "stream: %s", cudaGetErrorString(q));
    }
    ncclResult_t ae = ncclSuccess;
    const ncclResult_t r = h->nccl->CommGetAsyncError(h->comm, &ae);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (r != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress) || ms > (double)h->nccl_timeout_ms) {
      const bool timed_out = r == ncclSuccess && (ae == ncclSuccess || ae == ncclInProgress);
      h->nccl->CommAbort(h->comm);
      h->comm = nullptr;
      cudaStreamSynchronize(h->stream);   // the aborted collectives return
      cudaGetLastError();
      if (timed_out)
        return set_err(h, FASTPFP_ENCCL, "NCCL collectives did not complete within %lld ms (peer lost?); "
                       "communicator aborted", (long long)h->nccl_timeout_ms);
      return set_err(h, FASTPFP_ENCCL, "NCCL asynchronous error: %s; communicator aborted",
                     h->nccl->GetErrorString(r != ncclSuccess ? r : ae));
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

cudaError_t alloc_buf(Buf& b, int rows, int cols) {
  b.rows = rows;
  b.cols = cols;
  b.ld = round_up(std::max(cols, 1), 32);
  size_t bytes = (size_t)std::max(rows, 1) * b.ld * sizeof(float);
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) return e;
  return cudaMemset(b.p, 0, bytes);
}

void free_buf(Buf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
}

template <typename T>
cudaError_t alloc_arr(T*& p, size_t count) {
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T));
}

// dense (ld = cols) host/device matrix -> padded device buffer
cudaError_t upload(const Buf& b, const float* src, int is_device, cudaStream_t s) {
  return cudaMemcpy2DAsync(b.p, b.ld * sizeof(float), src, (size_t)b.cols * sizeof(float),
                           (size_t)b.cols * sizeof(float), b.rows,
                           is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
}

cudaError_t download(const Buf& b, float* dst, int is_device, cudaStream_t s) {
  return cudaMemcpy2DAsync(dst, (size_t)b.cols * sizeof(float), b.p, b.ld * sizeof(float),
                           (size_t)b.cols * sizeof(float), b.rows,
                           is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s);
}

// projection tiling: largest TR in {512, ..., 8} giving >= 2 tiles per SM, else 8
#ifndef FPFP_PROJ_MIN_TILES
#define FPFP_PROJ_MIN_TILES 2   // tiles per SM the row-block height TR must at least give
#endif
void plan_projection(fastpfp_handle* h) {
  const int64_t m = h->m, rows = h->yrows;
  const int CB = (int)ceil_div(m, kProjTC);
  int TR = 8;
  for (int tr : {512, 256, 128, 64, 32, 16, 8}) {
    if (ceil_div(rows, tr) * CB >= (int64_t)FPFP_PROJ_MIN_TILES * h->num_sms) { TR = tr; break; }
  }
  h->TR = TR;
  h->CB = CB;
  h->RB = (int)ceil_div(rows, TR);
  h->RBx = (int)ceil_div(h->n, TR);
  h->CBx = (int)ceil_div(h->np, kProjTC);
  const int64_t want = std::max<int64_t>((int64_t)h->RB * h->CB, (int64_t)h->RBx * h->CBx);
  const int maxg = proj_max_grid(h->device);
  h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, maxg));
}

int run_gemm(fastpfp_handle* h, GemmArgs& g) {
  cudaError_t e;
  h->stats.launches += 1;
  h->stats.gemm_launches += 1;
  g.cta_group = h->cta_group;
  if (h->precision == 2 || !gemm_tc_supported(g)) {
    if (h->precision != 2)
      return set_err(h, FASTPFP_EUNSUPPORTED, "tensor-core GEMM does not support M=%d N=%d K=%d",
                     g.M, g.N, g.K);
    e = launch_gemm_simt(g, h->stream);
  } else {
    e = launch_gemm_tc(g, h->precision == 1 ? 1 : 3, h->stream, h->device);
  }
  CK(h, e);
  return FASTPFP_OK;
}

// The TF32 GEMMs (precision 0, 1) read pre-split operands (A, A', X -> big + small parts); the
// int8 path reads digit planes instead and the SIMT path the plain fp32 matrices.
bool uses_tf32_split(const fastpfp_handle* h) { return h->precision == 0 || h->precision == 1; }

// TF32 splits of the graphs and of the current X (set_graphs, or a switch to a TF32 precision:
// while another precision ran, X changed without its split being refreshed)
int tf32_prepare(fastpfp_handle* h) {
  cudaStream_t s = h->stream;
  CK(h, launch_split(h->A.p, h->A.ld, h->Ab.p, h->As.p, h->A.ld, (int)h->n, (int)h->n_glob, s));
  CK(h, launch_split(h->Ap.p, h->Ap.ld, h->Apb.p, h->Aps.p, h->Ap.ld, (int)h->np, (int)h->np, s));
  CK(h, launch_split(h->X.p, h->X.ld, h->Xb.p, h->Xs.p, h->X.ld, (int)h->n, (int)h->np, s));
  CK(h, cudaStreamSynchronize(s));
  return FASTPFP_OK;
}

// X <- X0, split, Y <- 0, t <- 0
int reset_state(fastpfp_handle* h) {
  cudaStream_t s = h->stream;
  if (h->x0_custom) {
    CK(h, cudaMemcpy2DAsync(h->X.p, h->X.ld * 4, h->X0.p, h->X0.ld * 4, h->np * 4, h->n,
                            cudaMemcpyDeviceToDevice, s));
  } else {
    CK(h, launch_fill(h->X.p, h->X.ld, (int)h->n, (int)h->np,
                      (float)(1.0 / ((double)h->n_glob * (double)h->np)), s));  // 11^T/(nn')
  }
  if (uses_tf32_split(h))
    CK(h, launch_split(h->X.p, h->X.ld, h->Xb.p, h->Xs.p, h->X.ld, (int)h->n, (int)h->np, s));
  CK(h, cudaMemsetAsync(h->Y.p, 0, (size_t)h->yrows * h->Y.ld * sizeof(float), s));  // Y = 0
  CK(h, cudaMemsetAsync(h->done, 0, sizeof(int), s));
  CK(h, cudaStreamSynchronize(s));
  h->t = 0;
  h->xdig_fresh = false;
  return FASTPFP_OK;
}

int check_flags(fastpfp_handle* h, const char* what) {
  int f = 0;
  CK(h, cudaMemcpyAsync(&f, h->flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (f & 2) return set_err(h, FASTPFP_ENONFINITE, "%s contains NaN/Inf", what);
  if (f & 1) return set_err(h, FASTPFP_ESYM, "%s is not symmetric (undirected graphs, P:135-136)", what);
  return FASTPFP_OK;
}

cudaError_t alloc_i8(I8Buf& b, int rows, int K) {
  b.rows = rows; b.K = K;
  b.ld = round_up(std::max(K, 1), 128);
  for (auto& d : b.d) {
    cudaError_t e = alloc_arr(d, (size_t)std::max(rows, 1) * b.ld);
    if (e != cudaSuccess) return e;
  }
  return alloc_arr(b.e, (size_t)std::max(rows, 1));
}

cudaError_t split_i8(const Buf& src, I8Buf& dst, const unsigned* rowmax, const int* done,
                     cudaStream_t s) {
  return launch_split_i8(src.p, src.ld, dst.rows, dst.K, rowmax, dst.d, dst.ld, dst.e, done, s);
}

// Ozaki int8 operands: allocate on first use and digit-split the constant graphs (A, A') and X
int i8_prepare(fastpfp_handle* h) {
  if (!h->i8_ready) {
    if (!h->U.p) CK(h, alloc_buf(h->U, (int)h->np, (int)h->n));
    CK(h, alloc_i8(h->Ai8, (int)h->n, (int)h->n_glob));
    CK(h, alloc_i8(h->Api8, (int)h->np, (int)h->np));
    CK(h, alloc_i8(h->Xi8, (int)h->n, (int)h->np));
    CK(h, alloc_i8(h->Ui8, (int)h->np, (int)h->n));
    if (h->dist) CK(h, alloc_i8(h->Ui8all, (int)(h->world * h->np), (int)h->n));
    CK(h, alloc_arr(h->Urowmax, (size_t)h->np));
    CK(h, alloc_arr(h->xrowmax, (size_t)h->n));
    h->i8_ready = true;
  }
  if (h->graphs_set) {
    CK(h, split_i8(h->A, h->Ai8, nullptr, nullptr, h->stream));
    CK(h, split_i8(h->Ap, h->Api8, nullptr, nullptr, h->stream));
    CK(h, split_i8(h->X, h->Xi8, nullptr, nullptr, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->xdig_fresh = true;
  }
  return FASTPFP_OK;
}

// The two products of Algorithm 1 line 3 on one GPU, in the handle's precision:
// U = A' X^T (GEMM1), then out[0:n, 0:n'] = A U^T (+ lambda K when add_k; kEpiPG: X + alpha (...)).
int run_products(fastpfp_handle* h, double lambda, float* out, int64_t ldo, int epi2, bool add_k,
                 double alpha, const int* done) {
  cudaStream_t s = h->stream;
  const int N = (int)h->n, NP = (int)h->np;
  if (h->precision == 3) {
    const bool split_x = !h->xdig_fresh;
    if (split_x) CK(h, split_i8(h->X, h->Xi8, nullptr, done, s));   // digits of the current X
    h->xdig_fresh = false;   // the projection that follows changes X
    I8Gemm g1{};
    for (int k = 0; k < 3; ++k) { g1.P[k] = h->Api8.d[k]; g1.Q[k] = h->Xi8.d[k]; }
    g1.ldP = h->Api8.ld; g1.eP = h->Api8.e; g1.ldQ = h->Xi8.ld; g1.eQ = h->Xi8.e;
    g1.M = NP; g1.N = N; g1.K = NP;
    g1.epi = kEpiRowMax; g1.C = h->U.p; g1.ldC = h->U.ld; g1.rowmax = h->Urowmax; g1.done = done;
    if (!gemm_i8_supported(g1)) return set_err(h, FASTPFP_EUNSUPPORTED, "int8 GEMM1 unsupported shape");
    CK(h, cudaMemsetAsync(h->Urowmax, 0, (size_t)NP * sizeof(unsigned), s));
    CK(h, launch_gemm_i8(g1, s, h->device));
    CK(h, split_i8(h->U, h->Ui8, h->Urowmax, done, s));
    I8Gemm g2{};
    for (int k = 0; k < 3; ++k) { g2.P[k] = h->Ai8.d[k]; g2.Q[k] = h->Ui8.d[k]; }
    g2.ldP = h->Ai8.ld; g2.eP = h->Ai8.e; g2.ldQ = h->Ui8.ld; g2.eQ = h->Ui8.e;
    g2.M = N; g2.N = NP; g2.K = N;
    g2.epi = epi2; g2.C = out; g2.ldC = ldo;
    g2.D = (add_k && lambda != 0.0 && h->d > 0) ? h->K.p : nullptr; g2.ldD = h->K.ld;
    g2.lam = (float)lambda;
    g2.D2 = h->X.p; g2.ldD2 = h->X.ld; g2.scale = (float)alpha;
    g2.done = done;
    CK(h, launch_gemm_i8(g2, s, h->device));
    h->stats.launches += split_x ? 4 : 3;
    h->stats.gemm_launches += 2;
    return FASTPFP_OK;
  }
  // U = A' X^T (= (X A')^T, A' symmetric) ...
  GemmArgs g1{};
  g1.P = h->Ap.p; g1.ldP = h->Ap.ld; g1.Pb = h->Apb.p; g1.Ps = h->Aps.p;
  g1.Q = h->X.p; g1.ldQ = h->X.ld; g1.Qb = h->Xb.p; g1.Qs = h->Xs.p;
  g1.M = NP; g1.N = N; g1.K = NP;
  g1.epi = kEpiSplit; g1.C = h->Ub.p; g1.C2 = h->Us.p; g1.ldC = h->Ub.ld;
  g1.C3 = h->precision == 2 ? h->U.p : nullptr;   // plain U only feeds the SIMT GEMM2
  g1.done = done;
  int rc = run_gemm(h, g1);
  if (rc) return rc;
  // ... then out = A U^T (+ lambda K) = A X A' + lambda K
  GemmArgs g2{};
  g2.P = h->A.p; g2.ldP = h->A.ld; g2.Pb = h->Ab.p; g2.Ps = h->As.p;
  g2.Q = h->U.p; g2.ldQ = h->Ub.ld; g2.Qb = h->Ub.p; g2.Qs = h->Us.p;
  g2.M = N; g2.N = NP; g2.K = N;
  g2.epi = epi2; g2.C = out; g2.ldC = ldo;
  g2.D = (add_k && lambda != 0.0 && h->d > 0) ? h->K.p : nullptr; g2.ldD = h->K.ld;
  g2.lam = (float)lambda;
  g2.D2 = h->X.p; g2.ldD2 = h->X.ld; g2.scale = (float)alpha;   // PG: X + alpha grad f
  g2.done = done;
  return run_gemm(h, g2);
}

// FastGA workspace: E (m x m fp64), u, v ([2][m] each), per-block partials
int ga_alloc(fastpfp_handle* h) {
  if (h->ga_E) return FASTPFP_OK;
  h->ga_grid = ga_max_grid(h->device);
  if (h->ga_grid < 1) return set_err(h, FASTPFP_ECUDA, "FastGA kernel cannot be made resident");
  h->ga_W = ga_chunk_width((int)h->m, h->ga_grid);
  h->ga_ldE = round_up(h->m, 32);
  CK(h, alloc_arr(h->ga_E, (size_t)h->m * h->ga_ldE));
  CK(h, alloc_arr(h->ga_u, 2 * (size_t)h->ga_ldE));
  CK(h, alloc_arr(h->ga_v, 2 * (size_t)h->ga_ldE));
  CK(h, alloc_arr(h->ga_dlt, h->ga_grid));
  CK(h, alloc_arr(h->ga_rho, h->ga_grid));
  return FASTPFP_OK;
}

}  // namespace

struct GreedyScratch;
int fpfp_discretize_device(GreedyScratch**, const float*, int64_t, int, int, int32_t*, cudaStream_t,
                           std::string&);
void fpfp_greedy_free(GreedyScratch*);

extern "C" {

const char* fastpfp_status_string(int s) {
  switch (s) {
    case FASTPFP_OK: return "ok";
    case FASTPFP_EINVAL: return "invalid argument";
    case FASTPFP_ESYM: return "adjacency matrix not symmetric";
    case FASTPFP_ENONFINITE: return "non-finite input";
    case FASTPFP_ESTATE: return "call order (set_graphs first)";
    case FASTPFP_ENOMEM: return "device out of memory";
    case FASTPFP_ECUDA: return "CUDA error";
    case FASTPFP_ENCCL: return "NCCL error";
    case FASTPFP_ENODEV: return "no sm_100 device";
    case FASTPFP_EPOISONED: return "handle poisoned by an earlier CUDA/NCCL error";
    case FASTPFP_EUNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

int fastpfp_abi_version(void) { return FASTPFP_ABI_VERSION; }

int fastpfp_device_arch(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}

const char* fastpfp_last_error(const fastpfp_handle* h) { return h ? h->err.c_str() : ""; }

void fastpfp_destroy(fastpfp_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (Buf* b : {&h->A, &h->Ab, &h->As, &h->Ap, &h->Apb, &h->Aps, &h->B, &h->Bp, &h->K, &h->X,
                 &h->Xb, &h->Xs, &h->X0, &h->U, &h->Ub, &h->Us, &h->Y, &h->G, &h->Uball, &h->Usall,
                 &h->Xall})
    free_buf(*b);
  fpfp_greedy_free(h->greedy);
  for (I8Buf* b : {&h->Ai8, &h->Api8, &h->Xi8, &h->Ui8, &h->Ui8all}) {
    for (auto& d : b->d) if (d) cudaFree(d);
    if (b->e) cudaFree(b->e);
  }
  if (h->Urowmax) cudaFree(h->Urowmax);
  if (h->comm && h->nccl) h->nccl->CommDestroy(h->comm);   // (aborted communicators are nullptr)
  for (void* p : {(void*)h->rowpart, (void*)h->colpart, (void*)h->r, (void*)h->c,
                  (void*)h->sig_part, (void*)h->mu_part, (void*)h->dlt_part, (void*)h->rho_part,
                  (void*)h->iters, (void*)h->done, (void*)h->flags, (void*)h->scal, (void*)h->dot_part,
                  (void*)h->inner, (void*)h->tile_ctr,
                  (void*)h->oc_rowp, (void*)h->oc_colp, (void*)h->oc_tot, (void*)h->oc_dlt,
                  (void*)h->ga_E, (void*)h->ga_u, (void*)h->ga_v,
                  (void*)h->ga_dlt, (void*)h->ga_rho})
    if (p) cudaFree(p);
  if (h->h_iters) cudaFreeHost(h->h_iters);
  if (h->hpin) cudaFreeHost(h->hpin);
  if (h->ev_ready)
    for (auto& e : h->ev) cudaEventDestroy(e);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

static bool int8_default_ok(const fastpfp_handle* h) {
  return h->n_glob <= 32768 && h->np <= 32768 && (!h->dist || h->n % 128 == 0);
}

static int create_impl(int64_t n_glob, int64_t n_prime, int64_t d, int rank, int world,
                       const void* nccl_id, fastpfp_handle** out) {
  if (!out || n_glob < 1 || n_prime < 1 || d < 0 || n_glob > (1 << 20) || n_prime > (1 << 20) ||
      d > (1 << 20) || world < 1 || rank < 0 || rank >= world)
    return FASTPFP_EINVAL;
  *out = nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FASTPFP_ENODEV;
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return FASTPFP_ENODEV;
  const bool dist = nccl_id != nullptr;
  if (dist && (n_glob < n_prime || n_glob % world != 0 || (n_glob / world) % 32 != 0))
    return FASTPFP_EUNSUPPORTED;   // row sharding needs n >= n' and n/P a multiple of 32
  fastpfp_handle* h = new fastpfp_handle();
  h->n_glob = n_glob; h->n = n_glob / world; h->np = n_prime; h->d = d;
  h->m = std::max(n_glob, n_prime);
  h->yrows = dist ? h->n : h->m;
  h->rank = rank; h->world = world; h->dist = dist;
  h->device = dev;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
  h->arch = fastpfp_device_arch();
  int rc = FASTPFP_OK;
  auto A = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == FASTPFP_OK)
      rc = (e == cudaErrorMemoryAllocation) ? FASTPFP_ENOMEM : FASTPFP_ECUDA;
  };
  const int N = (int)h->n, NG = (int)n_glob, NP = (int)n_prime, M = (int)h->m, D = (int)d;
  A(alloc_buf(h->A, N, NG)); A(alloc_buf(h->Ab, N, NG)); A(alloc_buf(h->As, N, NG));
  A(alloc_buf(h->Ap, NP, NP)); A(alloc_buf(h->Apb, NP, NP)); A(alloc_buf(h->Aps, NP, NP));
  if (D > 0) { A(alloc_buf(h->B, N, D)); A(alloc_buf(h->Bp, NP, D)); }
  A(alloc_buf(h->K, N, NP));
  A(alloc_buf(h->X, N, NP)); A(alloc_buf(h->Xb, N, NP)); A(alloc_buf(h->Xs, N, NP));
  A(alloc_buf(h->Ub, NP, N)); A(alloc_buf(h->Us, NP, N));
  if (!dist) A(alloc_buf(h->U, NP, N));     // plain U: SIMT GEMM2 only
  if (dist) { A(alloc_buf(h->Uball, world * NP, N)); A(alloc_buf(h->Usall, world * NP, N)); }
  A(alloc_buf(h->Y, (int)h->yrows, M));
  plan_projection(h);
  A(alloc_arr(h->rowpart, (size_t)h->CB * h->yrows));
  A(alloc_arr(h->colpart, (size_t)h->RB * M));
  A(alloc_arr(h->r, kProjReplayC * h->yrows)); A(alloc_arr(h->c, kProjReplayC * ((size_t)M + 1)));   // replay generations
  A(alloc_arr(h->sig_part, h->grid)); A(alloc_arr(h->mu_part, h->grid));
  A(alloc_arr(h->dlt_part, h->grid)); A(alloc_arr(h->rho_part, h->grid));
  A(alloc_arr(h->iters, kMaxCheck)); A(alloc_arr(h->done, 1)); A(alloc_arr(h->flags, 1));
  A(alloc_arr(h->scal, 8)); A(alloc_arr(h->inner, 2)); A(alloc_arr(h->tile_ctr, 1));
  if (!dist && onchip_fits((int)h->m, h->num_sms, h->PR, h->PC, h->TRo, h->TCo)) {
    const int nb = h->PR * h->PC;
    h->oc_ok = true;
    // tagged 16-byte exchange records (proj_onchip.cu): 2 doubles / 4 floats of storage each
    A(alloc_arr(h->oc_rowp, 4 * (size_t)h->PC * M)); A(alloc_arr(h->oc_colp, 4 * (size_t)h->PR * M));
    A(alloc_arr(h->oc_tot, 4 * (size_t)nb)); A(alloc_arr(h->oc_dlt, 8 * (size_t)nb));
    if (nb > h->grid) {   // mu/rho partials are indexed by tile
      cudaFree(h->mu_part); cudaFree(h->rho_part);
      h->mu_part = nullptr; h->rho_part = nullptr;
      A(alloc_arr(h->mu_part, nb)); A(alloc_arr(h->rho_part, nb));
    }
  }
  A(cudaMallocHost(&h->h_iters, kMaxCheck * sizeof(DevIter)));
  A(cudaMallocHost(&h->hpin, 16 * sizeof(double)));
  A(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  if (rc == FASTPFP_OK && dist) {
    std::string msg;
    h->nccl = nccl_api(msg);
    if (!h->nccl) {
      h->err = msg;
      rc = FASTPFP_ENCCL;
    } else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      if (h->nccl->CommInitRank(&h->comm, world, id, rank) != ncclSuccess) rc = FASTPFP_ENCCL;
    }
  }
  if (rc == FASTPFP_OK && int8_default_ok(h)) {
    // default precision: the Ozaki int8 products (fp32-accurate) wherever they apply;
    // 3xTF32 otherwise (n or n' > 32768, or a row shard that is not a multiple of 128 rows)
    h->precision = 3;
    rc = i8_prepare(h);   // allocation only: the graphs are not set yet
  }
  if (rc != FASTPFP_OK) {
    cudaGetLastError();
    fastpfp_destroy(h);
    return rc;
  }
  *out = h;
  return FASTPFP_OK;
}

int fastpfp_create(int64_t n, int64_t n_prime, int64_t d, fastpfp_handle** out) {
  return create_impl(n, n_prime, d, 0, 1, nullptr, out);
}

int fastpfp_nccl_unique_id(void* out, int64_t size) {
  if (!out || size < (int64_t)sizeof(ncclUniqueId)) return FASTPFP_EINVAL;
  std::string msg;
  const NcclApi* api = nccl_api(msg);
  if (!api) return FASTPFP_ENCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return FASTPFP_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return FASTPFP_OK;
}

int fastpfp_create_dist(int64_t n, int64_t n_prime, int64_t d, int rank, int world,
                        const void* nccl_id, fastpfp_handle** out) {
  if (!nccl_id) return FASTPFP_EINVAL;
  return create_impl(n, n_prime, d, rank, world, nccl_id, out);
}

int fastpfp_set_option(fastpfp_handle* h, int key, int64_t value) {
  GUARD(h);
  switch (key) {
    case FASTPFP_OPT_SLACK_MODE:
      if (value != 0 && value != 1) return FASTPFP_EINVAL;
      h->slack_mode = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_PRECISION:
      if (value < 0 || value > 3) return FASTPFP_EINVAL;
      if (value == 3) {
        if (h->n_glob > 32768 || h->np > 32768)   // exact int32 digit sums need K <= 2^15
          return set_err(h, FASTPFP_EUNSUPPORTED, "int8 Ozaki GEMM needs n, n' <= 32768");
        if (h->dist && h->n % 128 != 0)
          return set_err(h, FASTPFP_EUNSUPPORTED, "sharded int8 GEMM needs (n/P) %% 128 == 0");
        h->precision = 3;
        return i8_prepare(h);
      }
      h->precision = (int)value;
      if (h->graphs_set && uses_tf32_split(h)) return tf32_prepare(h);
      return FASTPFP_OK;
    case FASTPFP_OPT_RESCALE:
      if (value != 0 && value != 1) return FASTPFP_EINVAL;
      h->rescale = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_STREAM:
      CK(h, cudaStreamSynchronize(h->stream));
      if (h->own_stream) cudaStreamDestroy(h->stream);
      h->own_stream = value == 0;
      if (value == 0) {
        CK(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      } else {
        h->stream = reinterpret_cast<cudaStream_t>(value);
      }
      return FASTPFP_OK;
    case FASTPFP_OPT_CHECK_EVERY:
      if (value < 1 || value > kMaxCheck) return FASTPFP_EINVAL;
      h->check_every = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_GEMM_CTA_GROUP:
      if (value != 1 && value != 2) return FASTPFP_EINVAL;
      h->cta_group = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_METHOD:
      if (value < 0 || value > 2) return FASTPFP_EINVAL;
      if (value == 2) {
        if (h->dist) return set_err(h, FASTPFP_EUNSUPPORTED, "FastGA is single-GPU only");
        int rc = ga_alloc(h);
        if (rc) return rc;
      }
      h->method = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_PROJ_KERNEL:
      if (value < 0 || value > 2) return FASTPFP_EINVAL;
      if (value == 2 && !h->oc_ok) return set_err(h, FASTPFP_EUNSUPPORTED, "Y does not fit on chip");
      h->proj_kernel = (int)value; return FASTPFP_OK;
    case FASTPFP_OPT_NCCL_TIMEOUT_MS:
      if (value < 0) return FASTPFP_EINVAL;
      h->nccl_timeout_ms = value; return FASTPFP_OK;
    case FASTPFP_OPT_PROFILE:
      if (value != 0 && value != 1) return FASTPFP_EINVAL;
      if (value && !h->ev_ready) {
        for (auto& e : h->ev) CK(h, cudaEventCreate(&e));
        h->ev_ready = true;
      }
      h->profile = (int)value; return FASTPFP_OK;
  }
  return set_err(h, FASTPFP_EINVAL, "unknown option key %d", key);
}

int fastpfp_get_option(fastpfp_handle* h, int key, int64_t* value) {
  GUARD(h);
  if (!value) return FASTPFP_EINVAL;
  switch (key) {
    case FASTPFP_OPT_SLACK_MODE: *value = h->slack_mode; return FASTPFP_OK;
    case FASTPFP_OPT_PRECISION: *value = h->precision; return FASTPFP_OK;
    case FASTPFP_OPT_RESCALE: *value = h->rescale; return FASTPFP_OK;
    case FASTPFP_OPT_STREAM: *value = reinterpret_cast<int64_t>(h->stream); return FASTPFP_OK;
    case FASTPFP_OPT_CHECK_EVERY: *value = h->check_every; return FASTPFP_OK;
    case FASTPFP_OPT_PROFILE: *value = h->profile; return FASTPFP_OK;
    case FASTPFP_OPT_GEMM_CTA_GROUP: *value = h->cta_group; return FASTPFP_OK;
    case FASTPFP_OPT_PROJ_KERNEL: *value = h->proj_kernel; return FASTPFP_OK;
    case FASTPFP_OPT_METHOD: *value = h->method; return FASTPFP_OK;
    case FASTPFP_OPT_NCCL_TIMEOUT_MS: *value = h->nccl_timeout_ms; return FASTPFP_OK;
  }
  return set_err(h, FASTPFP_EINVAL, "unknown option key %d", key);
}

int fastpfp_set_ga_schedule(fastpfp_handle* h, double beta0, double rate, double beta_max) {
  GUARD(h);
  if (!(beta0 > 0.0) || !std::isfinite(beta0) || !(rate >= 1.0) || !std::isfinite(rate) ||
      !(beta_max >= 0.0) || !std::isfinite(beta_max))
    return set_err(h, FASTPFP_EINVAL, "beta0 > 0, rate >= 1, beta_max >= 0 (finite)");
  h->ga_beta0 = beta0; h->ga_rate = rate; h->ga_beta_max = beta_max;
  return FASTPFP_OK;
}

int fastpfp_set_graphs(fastpfp_handle* h, const float* A, const float* A_prime, const float* B,
                       const float* B_prime, int is_device) {
  GUARD(h);
  NvtxRange nvtx_("fastpfp_set_graphs");
  if (!A || !A_prime) return set_err(h, FASTPFP_EINVAL, "A and A' are required");
  if (h->d > 0 && (!B || !B_prime)) return set_err(h, FASTPFP_EINVAL, "B and B' required (d > 0)");
  cudaStream_t s = h->stream;
  h->graphs_set = false;
  CK(h, upload(h->A, A, is_device, s));
  CK(h, upload(h->Ap, A_prime, is_device, s));
  CK(h, cudaMemsetAsync(h->flags, 0, sizeof(int), s));
  if (h->dist) {   // local row block: finiteness here, symmetry is the caller's contract
    CK(h, launch_check_finite(h->A.p, h->A.ld, (int)h->n, (int)h->n_glob, h->flags, s));
  } else {
    CK(h, launch_check_sym(h->A.p, h->A.ld, (int)h->n, h->flags, s));
  }
  int rc = check_flags(h, "A");
  if (rc) return rc;
  CK(h, launch_check_sym(h->Ap.p, h->Ap.ld, (int)h->np, h->flags, s));
  rc = check_flags(h, "A'");
  if (rc) return rc;
  if (uses_tf32_split(h)) {
    CK(h, launch_split(h->A.p, h->A.ld, h->Ab.p, h->As.p, h->A.ld, (int)h->n, (int)h->n_glob, s));
    CK(h, launch_split(h->Ap.p, h->Ap.ld, h->Apb.p, h->Aps.p, h->Ap.ld, (int)h->np, (int)h->np, s));
  }
  if (h->d > 0) {
    CK(h, upload(h->B, B, is_device, s));
    CK(h, upload(h->Bp, B_prime, is_device, s));
    CK(h, launch_check_finite(h->B.p, h->B.ld, (int)h->n, (int)h->d, h->flags, s));
    CK(h, launch_check_finite(h->Bp.p, h->Bp.ld, (int)h->np, (int)h->d, h->flags, s));
    rc = check_flags(h, "B/B'");
    if (rc) return rc;
    // K = B B'^T in fp32 (SIMT; d is small)
    GemmArgs g{};
    g.P = h->B.p; g.ldP = h->B.ld; g.Q = h->Bp.p; g.ldQ = h->Bp.ld;
    g.M = (int)h->n; g.N = (int)h->np; g.K = (int)h->d;
    g.epi = kEpiPlain; g.C = h->K.p; g.ldC = h->K.ld;
    CK(h, launch_gemm_simt(g, s));
  } else {
    CK(h, cudaMemsetAsync(h->K.p, 0, (size_t)h->n * h->K.ld * sizeof(float), s));
  }
  rc = reset_state(h);
  if (rc) return rc;
  h->graphs_set = true;
  if (h->precision == 3) return i8_prepare(h);   // digit planes of the new A, A'
  return FASTPFP_OK;
}

int fastpfp_set_x0(fastpfp_handle* h, const float* X0, int is_device) {
  GUARD(h);
  cudaStream_t s = h->stream;
  if (X0) {
    if (!h->X0.p) CK(h, alloc_buf(h->X0, (int)h->n, (int)h->np));
    CK(h, upload(h->X0, X0, is_device, s));
    CK(h, cudaMemsetAsync(h->flags, 0, sizeof(int), s));
    CK(h, launch_check_finite(h->X0.p, h->X0.ld, (int)h->n, (int)h->np, h->flags, s));
    int rc = check_flags(h, "X0");
    if (rc) return rc;
    h->x0_custom = true;
  } else {
    h->x0_custom = false;
  }
  return reset_state(h);
}

int fastpfp_reset(fastpfp_handle* h) {
  GUARD(h);
  return reset_state(h);
}

// ---- row-sharded outer iteration: every step is a local kernel; the three
// exchanges are NCCL collectives on the handle's stream: all-gather of U's TF32 parts after GEMM1,
// all-reduce SUM of [column sums | sigma] after every sweep, all-reduce MAX of mu and of rho.
static int dist_gemms(fastpfp_handle* h, double lambda, float* out, int64_t ldo, bool add_k,
                      double pg_alpha = 0.0) {
  cudaStream_t s = h->stream;
  const int N = (int)h->n, NP = (int)h->np;
  if (h->precision == 3) {
    // U_r = A' X_r^T (int8 digits, local rows) with its per-row |max| ...
    CK(h, split_i8(h->X, h->Xi8, nullptr, nullptr, s));
    I8Gemm g1{};
    for (int k = 0; k < 3; ++k) { g1.P[k] = h->Api8.d[k]; g1.Q[k] = h->Xi8.d[k]; }
    g1.ldP = h->Api8.ld; g1.eP = h->Api8.e; g1.ldQ = h->Xi8.ld; g1.eQ = h->Xi8.e;
    g1.M = NP; g1.N = N; g1.K = NP;
    g1.epi = kEpiRowMax; g1.C = h->U.p; g1.ldC = h->U.ld; g1.rowmax = h->Urowmax;
    if (!gemm_i8_supported(g1)) return set_err(h, FASTPFP_EUNSUPPORTED, "int8 GEMM1 unsupported shape");
    CK(h, cudaMemsetAsync(h->Urowmax, 0, (size_t)NP * sizeof(unsigned), s));
    CK(h, launch_gemm_i8(g1, s, h->device));
    // ... the row scales of U are global: MAX over ranks of the |max| bits (nonneg floats order
    // as unsigned), so every rank splits its block with the same exponents ...
    NK(h, coll_allreduce(h, h->Urowmax, (size_t)NP, ncclUint32, ncclMax, s));
    CK(h, split_i8(h->U, h->Ui8, h->Urowmax, nullptr, s));
    // ... all-gather of the 3 digit planes (3 bytes per element instead of 8 for the TF32 parts)
    const size_t cnt = (size_t)NP * h->Ui8.ld;
    NK(h, h->nccl->GroupStart());
    for (int k = 0; k < 3; ++k)
      NK(h, coll_allgather(h, h->Ui8.d[k], h->Ui8all.d[k], cnt, ncclInt8, s));
    NK(h, h->nccl->GroupEnd());
    // Y_r[:, 0:n'] = A_r U^T + lambda K_r, K-loop over the gathered rank blocks (3-D TMA)
    I8Gemm g2{};
    for (int k = 0; k < 3; ++k) { g2.P[k] = h->Ai8.d[k]; g2.Q[k] = h->Ui8all.d[k]; }
    g2.ldP = h->Ai8.ld; g2.eP = h->Ai8.e; g2.ldQ = h->Ui8.ld; g2.eQ = h->Ui8.e;
    g2.M = N; g2.N = NP; g2.K = (int)h->n_glob;
    g2.q_blocks = h->world; g2.q_block_k = N; g2.q_block_stride = (int64_t)NP * h->Ui8.ld;
    g2.epi = (add_k && h->method == 1) ? kEpiPG : kEpiAxpy; g2.C = out; g2.ldC = ldo;
    g2.D = (add_k && lambda != 0.0 && h->d > 0) ? h->K.p : nullptr; g2.ldD = h->K.ld;
    g2.lam = (float)lambda;
    g2.D2 = h->X.p; g2.ldD2 = h->X.ld; g2.scale = (float)pg_alpha;
    if (!gemm_i8_supported(g2)) return set_err(h, FASTPFP_EUNSUPPORTED, "int8 GEMM2 unsupported shape");
    CK(h, launch_gemm_i8(g2, s, h->device));
    h->stats.launches += 4;
    h->stats.gemm_launches += 2;
    return FASTPFP_OK;
  }
  // U_r = A' X_r^T for the local rows r
  GemmArgs g1{};
  g1.P = h->Ap.p; g1.ldP = h->Ap.ld; g1.Pb = h->Apb.p; g1.Ps = h->Aps.p;
  g1.Q = h->X.p; g1.ldQ = h->X.ld; g1.Qb = h->Xb.p; g1.Qs = h->Xs.p;
  g1.M = NP; g1.N = N; g1.K = NP;
  g1.epi = kEpiSplit; g1.C = h->Ub.p; g1.C2 = h->Us.p; g1.ldC = h->Ub.ld;
  int rc = run_gemm(h, g1);
  if (rc) return rc;
  const size_t cnt = (size_t)NP * h->Ub.ld;
  NK(h, h->nccl->GroupStart());
  NK(h, coll_allgather(h, h->Ub.p, h->Uball.p, cnt, ncclFloat32, s));
  NK(h, coll_allgather(h, h->Us.p, h->Usall.p, cnt, ncclFloat32, s));
  NK(h, h->nccl->GroupEnd());
  // Y_r[:, 0:n'] = A_r U^T + lambda K_r, K-loop over the gathered rank blocks
  GemmArgs g2{};
  g2.P = h->A.p; g2.ldP = h->A.ld; g2.Pb = h->Ab.p; g2.Ps = h->As.p;
  g2.Qb = h->Uball.p; g2.Qs = h->Usall.p; g2.ldQ = h->Uball.ld;
  g2.M = N; g2.N = NP; g2.K = (int)h->n_glob;
  g2.q_blocks = h->world; g2.q_block_k = N; g2.q_block_stride = (int64_t)NP * h->Uball.ld;
  g2.epi = (add_k && h->method == 1) ? kEpiPG : kEpiAxpy; g2.C = out; g2.ldC = ldo;
  g2.D = (add_k && lambda != 0.0 && h->d > 0) ? h->K.p : nullptr; g2.ldD = h->K.ld;
  g2.lam = (float)lambda;
  g2.D2 = h->X.p; g2.ldD2 = h->X.ld; g2.scale = (float)pg_alpha;
  return run_gemm(h, g2);
}

static ProjArgs dist_proj_args(fastpfp_handle* h, int mode, double alpha, double eps1, double eps2) {
  ProjArgs pa{};
  pa.mode = mode; pa.rows = (int)h->yrows;
  pa.Y = h->Y.p; pa.ldY = h->Y.ld; pa.m = (int)h->m;
  pa.X = h->X.p; pa.Xb = h->Xb.p; pa.Xs = h->Xs.p; pa.ldX = h->X.ld; pa.n = (int)h->n;
  pa.np = (int)h->np;
  pa.alpha = alpha; pa.eps1 = eps1; pa.eps2 = eps2; pa.max_iter2 = 1;
  pa.rescale = h->rescale; pa.split = h->precision == 3 ? 0 : 1;
  pa.TR = h->TR; pa.RB = h->RB; pa.CB = h->CB; pa.RBx = h->RBx; pa.CBx = h->CBx;
  pa.rowpart = h->rowpart; pa.colpart = h->colpart; pa.r = h->r; pa.c = h->c; pa.scal = h->scal;
  pa.sig_part = h->sig_part; pa.dlt_part = h->dlt_part; pa.mu_part = h->mu_part;
  pa.rho_part = h->rho_part; pa.iter_out = h->iters; pa.done = h->done;
  return pa;
}

static int dist_outer(fastpfp_handle* h, double alpha, double lambda, double eps1, double eps2,
                      int32_t max_iter2, DevIter& out) {
  cudaStream_t s = h->stream;
  if (h->profile) CK(h, cudaEventRecord(h->ev[0], s));
  int rc = dist_gemms(h, lambda, h->Y.p, h->Y.ld, true, alpha);
  if (rc) return rc;
  if (h->profile) CK(h, cudaEventRecord(h->ev[1], s));
  if (h->slack_mode == 1 && h->m > h->np) {
    CK(h, launch_zero_slack(h->Y.p, h->Y.ld, (int)h->yrows, (int)h->m, (int)h->n, (int)h->np,
                            h->done, s));
    h->stats.launches += 1;
  }
  const size_t mc = (size_t)h->m + 1;
  ProjArgs pa = dist_proj_args(h, kProjSums, h->method == 1 ? 1.0 : alpha, eps1, eps2);
  if (h->method == 1) pa.rescale = 0;
  pa.tile_ctr = h->tile_ctr;   // dynamic tile schedule: the counter is reset before each pass launch
  CK(h, cudaMemsetAsync(h->tile_ctr, 0, sizeof(unsigned), s));
  CK(h, launch_proj(pa, h->grid, s));
  NK(h, coll_allreduce(h, h->c, mc, ncclFloat64, ncclSum, s));
  h->stats.launches += 1;
  // inner loop: sweep launches enqueued in chunks; each launch first applies the stop
  // test of the previous sweep on the device (global delta after its MAX all-reduce), so the host
  // synchronises once per chunk, not per sweep. With eps2 = 0 the whole fixed schedule is enqueued
  // at once and the delta all-reduce runs for the reported last sweep only.
  CK(h, cudaMemsetAsync(h->inner, 0, 2 * sizeof(int), s));
  pa.mode = kProjOneSweep;
  pa.inner = eps2 > 0.0 ? h->inner : nullptr;
  int enq = 0;
  while (enq < max_iter2) {
    const int chunk = eps2 > 0.0 ? std::min(kSweepChunk, max_iter2 - enq) : max_iter2 - enq;
    for (int k = 0; k < chunk; ++k, ++enq) {
      CK(h, cudaMemsetAsync(h->tile_ctr, 0, sizeof(unsigned), s));
      CK(h, launch_proj(pa, h->grid, s));
      NK(h, coll_allreduce(h, h->c, mc, ncclFloat64, ncclSum, s));
      if (eps2 > 0.0 || enq + 1 >= max_iter2)
        NK(h, coll_allreduce(h, h->scal, 1, ncclFloat64, ncclMax, s));
      h->stats.launches += 1;
    }
    if (eps2 > 0.0 && enq < max_iter2) {
      int* st = reinterpret_cast<int*>(h->hpin + 8);
      CK(h, cudaMemcpyAsync(st, h->inner, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
      int rc2 = stream_sync(h);
      if (rc2) return rc2;
      if (st[1]) break;
    }
  }
  pa.inner = nullptr;
  pa.tile_ctr = nullptr;       // the finalize phases tile by rows of X (static)
  pa.mode = kProjFinMu;
  CK(h, launch_proj(pa, h->grid, s));
  NK(h, coll_allreduce(h, h->scal + 1, 1, ncclFloat64, ncclMax, s));
  pa.mode = kProjFinApply;
  CK(h, launch_proj(pa, h->grid, s));
  NK(h, coll_allreduce(h, h->scal + 2, 1, ncclFloat64, ncclMax, s));
  h->stats.launches += 2;
  h->stats.proj_launches += 1;
  if (h->profile) CK(h, cudaEventRecord(h->ev[2], s));
  double* sc = h->hpin;
  int* st = reinterpret_cast<int*>(h->hpin + 8);
  CK(h, cudaMemcpyAsync(sc, h->scal, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(h, cudaMemcpyAsync(st, h->inner, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  rc = stream_sync(h);
  if (rc) return rc;
  out = DevIter{};
  out.valid = 1; out.sweeps = eps2 > 0.0 ? st[0] : max_iter2; out.delta = sc[0]; out.mu = sc[1];
  if (sc[2] < 0.0) {
    out.degenerate = 1;
  } else {
    out.rho = sc[2];
    out.converged = sc[2] < eps1;
  }
  if (h->profile) {
    float g_ms = 0.f, p_ms = 0.f;
    CK(h, cudaEventElapsedTime(&g_ms, h->ev[0], h->ev[1]));
    CK(h, cudaEventElapsedTime(&p_ms, h->ev[1], h->ev[2]));
    h->stats.gemm_ms += g_ms;
    h->stats.proj_ms += p_ms;
    h->stats.gemm_flops += 2.0 * (double)h->n * h->np * ((double)h->n_glob + h->np);
  }
  return FASTPFP_OK;
}

int fastpfp_iterate(fastpfp_handle* h, double alpha, double lambda, double eps1, double eps2,
                    int32_t max_iter1, int32_t max_iter2, float* X_out, fastpfp_report* rep) {
  GUARD(h);
  NvtxRange nvtx_("fastpfp_iterate");
  if (h->dist && h->graphs_set && (alpha >= 0.0 && alpha <= 1.0) && lambda >= 0.0 &&
      std::isfinite(lambda) && eps1 >= 0.0 && eps2 >= 0.0 && max_iter1 >= 1 && max_iter2 >= 1) {
    if (h->precision == 2) return set_err(h, FASTPFP_EUNSUPPORTED, "row sharding needs the tensor-core GEMM");
    fastpfp_report R{};
    if (rep) {
      R.trace_capacity = rep->trace_capacity;
      R.rho_trace = rep->rho_trace; R.sweeps_trace = rep->sweeps_trace;
      R.delta_trace = rep->delta_trace; R.mu_trace = rep->mu_trace;
    }
    CK(h, cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    h->coll_log.clear();
    for (int32_t k = 0; k < max_iter1; ++k) {
      DevIter it{};
      int rc = dist_outer(h, alpha, lambda, eps1, eps2, max_iter2, it);
      if (rc) return rc;
      h->stats.outer_iterations += 1;
      h->stats.sweeps += it.sweeps;
      R.total_sweeps += it.sweeps;
      R.last_delta = it.delta;
      R.last_mu = it.mu;
      if (it.degenerate) { R.degenerate = 1; break; }
      if (R.trace_capacity > R.iterations) {
        const int q = R.iterations;
        if (R.rho_trace) R.rho_trace[q] = it.rho;
        if (R.sweeps_trace) R.sweeps_trace[q] = it.sweeps;
        if (R.delta_trace) R.delta_trace[q] = it.delta;
        if (R.mu_trace) R.mu_trace[q] = it.mu;
      }
      R.iterations += 1;
      R.last_rho = it.rho;
      h->t += 1;
      if (it.converged) { R.converged = 1; break; }
    }
    if (X_out) {   // wait with fault polling first: a copy into pageable memory would block
      int rc = stream_sync(h);
      if (rc) return rc;
      CK(h, download(h->X, X_out, 0, h->stream));
      CK(h, cudaStreamSynchronize(h->stream));
    }
    if (rep) *rep = R;
    return FASTPFP_OK;
  }
  if (!h->graphs_set) return set_err(h, FASTPFP_ESTATE, "fastpfp_set_graphs must come first");
  if (!(alpha >= 0.0 && alpha <= 1.0) || !(lambda >= 0.0) || !std::isfinite(lambda) ||
      !(eps1 >= 0.0) || !(eps2 >= 0.0) || max_iter1 < 1 || max_iter2 < 1)
    return set_err(h, FASTPFP_EINVAL, "alpha in [0,1], lambda >= 0, eps >= 0, maxIter >= 1");
  cudaStream_t s = h->stream;
  fastpfp_report R{};
  if (rep) {
    R.trace_capacity = rep->trace_capacity;
    R.rho_trace = rep->rho_trace; R.sweeps_trace = rep->sweeps_trace;
    R.delta_trace = rep->delta_trace; R.mu_trace = rep->mu_trace;
  }
  CK(h, cudaMemsetAsync(h->done, 0, sizeof(int), s));
  const int N = (int)h->n, NP = (int)h->np;
  // PG: the projection output is the new X (blend weight 1, no rescale)
  const double blend = h->method == 1 ? 1.0 : alpha;
  const int rescale = h->method == 1 ? 0 : h->rescale;
  int32_t left = max_iter1;
  if (h->method == 2) {   // FastGA anneals while beta_t = beta0 rate^t <= beta_max (reading G5)
    int32_t allowed = 0;
    while (allowed < left && h->ga_beta0 * std::pow(h->ga_rate, (double)(h->t + allowed)) <= h->ga_beta_max)
      ++allowed;
    left = allowed;
  }
  bool stop = false;
  while (left > 0 && !stop) {
    const int chunk = std::min<int32_t>(left, h->check_every);
    CK(h, cudaMemsetAsync(h->iters, 0, chunk * sizeof(DevIter), s));
    for (int k = 0; k < chunk; ++k) {
      if (h->profile) CK(h, cudaEventRecord(h->ev[3 * k], s));
      // Algorithm 1 line 3: Y[0:n, 0:n'] = A X A' + lambda K (PG: X + alpha grad f)
      int rc = run_products(h, lambda, h->Y.p, h->Y.ld, h->method == 1 ? kEpiPG : kEpiAxpy, true,
                            alpha, h->done);
      if (rc) return rc;
      if (h->profile) CK(h, cudaEventRecord(h->ev[3 * k + 1], s));
      if (h->method != 2 && h->slack_mode == 1 && h->m > std::min(h->n, h->np)) {
        CK(h, launch_zero_slack(h->Y.p, h->Y.ld, (int)h->m, (int)h->m, N, NP, h->done, s));
        h->stats.launches += 1;
      }
      if (h->method == 2) {   // FastGA: exp + slack-padded Sinkhorn + X update (ga.cu)
        GaArgs ga{};
        ga.Q = h->Y.p; ga.ldQ = h->Y.ld; ga.m = (int)h->m; ga.n = N; ga.np = NP;
        ga.beta = h->ga_beta0 * std::pow(h->ga_rate, (double)(h->t + k));   // reading G5
        ga.eps1 = eps1; ga.eps2 = eps2; ga.max_iter2 = max_iter2; ga.W = h->ga_W;
        ga.E = h->ga_E; ga.ldE = h->ga_ldE; ga.u = h->ga_u; ga.v = h->ga_v;
        ga.dlt_part = h->ga_dlt; ga.rho_part = h->ga_rho;
        ga.X = h->X.p; ga.Xb = h->Xb.p; ga.Xs = h->Xs.p; ga.ldX = h->X.ld;
        ga.iter_out = h->iters + k; ga.done = h->done;
        CK(h, launch_ga(ga, h->ga_grid, s));
        h->stats.launches += 1;
        h->stats.proj_launches += 1;
        if (h->profile) CK(h, cudaEventRecord(h->ev[3 * k + 2], s));
        continue;
      }
      // lines 4-9: projection loop, blend, rescale (one persistent kernel)
      if (h->oc_ok && h->proj_kernel != 1) {
        OnchipArgs oa{};
        oa.Y = h->Y.p; oa.ldY = h->Y.ld; oa.m = (int)h->m;
        oa.X = h->X.p; oa.Xb = h->Xb.p; oa.Xs = h->Xs.p; oa.ldX = h->X.ld; oa.n = N; oa.np = NP;
        oa.alpha = blend; oa.eps1 = eps1; oa.eps2 = eps2; oa.max_iter2 = max_iter2;
        oa.rescale = rescale; oa.do_finalize = 1;
        oa.PR = h->PR; oa.PC = h->PC; oa.TRo = h->TRo; oa.TCo = h->TCo;
        oa.rowp = h->oc_rowp; oa.colp = h->oc_colp; oa.tot = h->oc_tot; oa.dlt = h->oc_dlt;
        oa.mu_part = h->mu_part; oa.rho_part = h->rho_part; oa.iter_out = h->iters + k;
        oa.done = h->done;
        if (((++h->oc_epoch) & 0xffffu) == 0) ++h->oc_epoch;   // tags of the exchange records
        oa.epoch = h->oc_epoch;
        CK(h, launch_proj_onchip(oa, s));
        h->stats.launches += 1;
        h->stats.proj_launches += 1;
        h->stats.onchip_launches += 1;
        if (h->profile) CK(h, cudaEventRecord(h->ev[3 * k + 2], s));
        continue;
      }
      ProjArgs pa{};
      pa.mode = kProjFull; pa.rows = (int)h->yrows;
      pa.Y = h->Y.p; pa.ldY = h->Y.ld; pa.m = (int)h->m;
      pa.X = h->X.p; pa.Xb = h->Xb.p; pa.Xs = h->Xs.p; pa.ldX = h->X.ld; pa.n = N; pa.np = NP;
      pa.alpha = blend; pa.eps1 = eps1; pa.eps2 = eps2; pa.max_iter2 = max_iter2;
      // the TF32 split of X feeds only the TF32 GEMMs (the int8 path splits X into digits itself)
      pa.rescale = rescale; pa.split = h->precision == 3 ? 0 : 1; pa.do_finalize = 1; pa.do_sums = 1;
      pa.TR = h->TR; pa.RB = h->RB; pa.CB = h->CB; pa.RBx = h->RBx; pa.CBx = h->CBx;
      pa.rowpart = h->rowpart; pa.colpart = h->colpart; pa.r = h->r; pa.c = h->c;
      pa.sig_part = h->sig_part; pa.dlt_part = h->dlt_part; pa.mu_part = h->mu_part;
      pa.rho_part = h->rho_part; pa.iter_out = h->iters + k; pa.done = h->done;
      const bool fuse_digits = h->precision == 3 && h->i8_ready;
      if (fuse_digits) {   // the finalize writes the new X's digit planes (no split_i8 of X next)
        for (int q = 0; q < 3; ++q) pa.xd[q] = h->Xi8.d[q];
        pa.ldxd = h->Xi8.ld; pa.xe = h->Xi8.e; pa.xrowmax = h->xrowmax;
        CK(h, cudaMemsetAsync(h->xrowmax, 0, (size_t)N * sizeof(unsigned long long), s));
      }
      pa.tile_ctr = h->tile_ctr;
      pa.replay = proj_replay_default();
      CK(h, cudaMemsetAsync(h->tile_ctr, 0, sizeof(unsigned), s));
      CK(h, launch_proj(pa, h->grid, s));
      h->stats.launches += 1;
      h->stats.proj_launches += 1;
      if (fuse_digits) h->xdig_fresh = true;
      if (h->profile) CK(h, cudaEventRecord(h->ev[3 * k + 2], s));
    }
    CK(h, cudaMemcpyAsync(h->h_iters, h->iters, chunk * sizeof(DevIter), cudaMemcpyDeviceToHost, s));
    CK(h, cudaStreamSynchronize(s));
    for (int k = 0; k < chunk; ++k) {
      const DevIter& it = h->h_iters[k];
      if (!it.valid) { stop = true; break; }
      if (h->profile) {
        float g_ms = 0.f, p_ms = 0.f;
        CK(h, cudaEventElapsedTime(&g_ms, h->ev[3 * k], h->ev[3 * k + 1]));
        CK(h, cudaEventElapsedTime(&p_ms, h->ev[3 * k + 1], h->ev[3 * k + 2]));
        h->stats.gemm_ms += g_ms;
        h->stats.proj_ms += p_ms;
        h->stats.gemm_flops += 2.0 * (double)N * NP * ((double)N + NP);
      }
      h->stats.outer_iterations += 1;
      h->stats.sweeps += it.sweeps;
      R.total_sweeps += it.sweeps;
      R.last_delta = it.delta;
      R.last_mu = it.mu;
      if (it.degenerate) { R.degenerate = 1; stop = true; break; }
      if (R.trace_capacity > R.iterations) {
        const int q = R.iterations;
        if (R.rho_trace) R.rho_trace[q] = it.rho;
        if (R.sweeps_trace) R.sweeps_trace[q] = it.sweeps;
        if (R.delta_trace) R.delta_trace[q] = it.delta;
        if (R.mu_trace) R.mu_trace[q] = it.mu;
      }
      R.iterations += 1;
      R.last_rho = it.rho;
      h->t += 1;
      if (it.converged) { R.converged = 1; stop = true; break; }
    }
    left -= chunk;
  }
  if (X_out) {
    CK(h, download(h->X, X_out, 0, s));
    CK(h, cudaStreamSynchronize(s));
  }
  if (rep) *rep = R;
  return FASTPFP_OK;
}

int fastpfp_dist_collectives(fastpfp_handle* h, int64_t* out, int64_t capacity, int64_t* count) {
  GUARD(h);
  if (!count || (capacity > 0 && !out)) return FASTPFP_EINVAL;
  *count = (int64_t)h->coll_log.size();
  for (int64_t k = 0; k < std::min<int64_t>(capacity, *count); ++k)
    for (int q = 0; q < 4; ++q) out[4 * k + q] = h->coll_log[k][q];
  return FASTPFP_OK;
}

int fastpfp_get_stats(fastpfp_handle* h, fastpfp_stats* out) {
  GUARD(h);
  if (!out) return FASTPFP_EINVAL;
  *out = h->stats;
  out->onchip_tiles = h->oc_ok ? h->PR * h->PC : 0;
  return FASTPFP_OK;
}

int fastpfp_reset_stats(fastpfp_handle* h) {
  GUARD(h);
  h->stats = fastpfp_stats{};
  return FASTPFP_OK;
}

int fastpfp_copy_x(fastpfp_handle* h, float* dst, int dst_is_device) {
  GUARD(h);
  if (!dst) return FASTPFP_EINVAL;
  CK(h, download(h->X, dst, dst_is_device, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return FASTPFP_OK;
}

int fastpfp_copy_y(fastpfp_handle* h, float* dst, int dst_is_device) {
  GUARD(h);
  if (!dst) return FASTPFP_EINVAL;
  CK(h, download(h->Y, dst, dst_is_device, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return FASTPFP_OK;
}

int fastpfp_set_y(fastpfp_handle* h, const float* Y, int is_device) {
  GUARD(h);
  if (!Y) return FASTPFP_EINVAL;
  if (!h->graphs_set) return set_err(h, FASTPFP_ESTATE, "fastpfp_set_graphs must come first");
  cudaStream_t s = h->stream;
  CK(h, upload(h->Y, Y, is_device, s));
  CK(h, cudaMemsetAsync(h->flags, 0, sizeof(int), s));
  CK(h, launch_check_finite(h->Y.p, h->Y.ld, (int)h->yrows, (int)h->m, h->flags, s));
  return check_flags(h, "Y");
}

int fastpfp_objective(fastpfp_handle* h, double lambda, double* f) {
  GUARD(h);
  NvtxRange nvtx_("fastpfp_objective");
  if (!f) return FASTPFP_EINVAL;
  if (!h->graphs_set) return set_err(h, FASTPFP_ESTATE, "fastpfp_set_graphs must come first");
  if (!h->G.p) CK(h, alloc_buf(h->G, (int)h->n, (int)h->np));
  if (!h->dot_part) CK(h, alloc_arr(h->dot_part, 2 * (size_t)kDotBlocks));
  cudaStream_t s = h->stream;
  if (h->dist) {
    h->coll_log.clear();
    int rc = dist_gemms(h, lambda, h->G.p, h->G.ld, false);
    if (rc) return rc;
    CK(h, launch_dot2(h->X.p, h->G.p, h->d > 0 ? h->K.p : nullptr, h->X.ld, (int)h->n, (int)h->np,
                      h->dot_part, h->scal + 4, s));
    NK(h, coll_allreduce(h, h->scal + 4, 2, ncclFloat64, ncclSum, s));
    double* v = h->hpin + 4;
    CK(h, cudaMemcpyAsync(v, h->scal + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    rc = stream_sync(h);
    if (rc) return rc;
    *f = 0.5 * v[0] + lambda * v[1];
    return FASTPFP_OK;
  }
  const int N = (int)h->n, NP = (int)h->np;
  int rc = run_products(h, 0.0, h->G.p, h->G.ld, kEpiAxpy, false, 0.0, nullptr);
  if (rc) return rc;
  CK(h, launch_dot2(h->X.p, h->G.p, h->d > 0 ? h->K.p : nullptr, h->X.ld, N, NP, h->dot_part, h->scal, s));
  double v[2];
  CK(h, cudaMemcpyAsync(v, h->scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  *f = 0.5 * v[0] + lambda * v[1];  // 1/2 tr(X^T A X A') + lambda tr(X^T K)
  return FASTPFP_OK;
}

int fastpfp_discretize(fastpfp_handle* h, int32_t* assign) {
  GUARD(h);
  NvtxRange nvtx_("fastpfp_discretize");
  if (!assign) return FASTPFP_EINVAL;
  if (!h->graphs_set) return set_err(h, FASTPFP_ESTATE, "fastpfp_set_graphs must come first");
  std::string msg;
  if (h->dist) {   // gather the full X (every rank gets the same greedy result)
    h->coll_log.clear();
    if (!h->Xall.p) CK(h, alloc_buf(h->Xall, (int)h->n_glob, (int)h->np));
    const size_t cnt = (size_t)h->n * h->X.ld;
    NK(h, coll_allgather(h, h->X.p, h->Xall.p, cnt, ncclFloat32, h->stream));
    int rc = stream_sync(h);
    if (rc) return rc;
    rc = fpfp_discretize_device(&h->greedy, h->Xall.p, h->Xall.ld, (int)h->n_glob, (int)h->np, assign,
                                    h->stream, msg);
    if (rc) return set_err(h, rc, "%s", msg.c_str());
    return FASTPFP_OK;
  }
  int rc = fpfp_discretize_device(&h->greedy, h->X.p, h->X.ld, (int)h->n, (int)h->np, assign, h->stream, msg);
  if (rc) return set_err(h, rc, "%s", msg.c_str());
  return FASTPFP_OK;
}

int fastpfp_project(float* Y, int64_t m, double eps2, int32_t max_iter2, int32_t* sweeps_out,
                    double* delta_out, int64_t stream) {
  if (!Y || m < 1 || max_iter2 < 1 || !(eps2 >= 0.0)) return FASTPFP_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FASTPFP_ENODEV;
  fastpfp_handle tmp;
  tmp.n = m; tmp.np = m; tmp.m = m; tmp.n_glob = m; tmp.yrows = m; tmp.device = dev;
  cudaDeviceGetAttribute(&tmp.num_sms, cudaDevAttrMultiProcessorCount, dev);
  plan_projection(&tmp);
  Buf Yp;
  int rc = FASTPFP_OK;
  DevIter it{};
  auto A = [&](cudaError_t e) { if (e != cudaSuccess && rc == FASTPFP_OK) rc = FASTPFP_ECUDA; };
  A(alloc_buf(Yp, (int)m, (int)m));
  A(alloc_arr(tmp.rowpart, (size_t)tmp.CB * m)); A(alloc_arr(tmp.colpart, (size_t)tmp.RB * m));
  A(alloc_arr(tmp.r, kProjReplayC * m)); A(alloc_arr(tmp.c, kProjReplayC * (m + 1)));
  A(alloc_arr(tmp.sig_part, tmp.grid)); A(alloc_arr(tmp.mu_part, tmp.grid));
  A(alloc_arr(tmp.dlt_part, tmp.grid)); A(alloc_arr(tmp.rho_part, tmp.grid));
  A(alloc_arr(tmp.iters, 1)); A(alloc_arr(tmp.done, 1));
  if (rc == FASTPFP_OK) {
    A(upload(Yp, Y, 1, s));
    ProjArgs pa{};
    pa.mode = kProjFull; pa.rows = (int)m;
    pa.Y = Yp.p; pa.ldY = Yp.ld; pa.m = (int)m; pa.n = (int)m; pa.np = (int)m;
    pa.eps2 = eps2; pa.max_iter2 = max_iter2; pa.do_finalize = 0; pa.do_sums = 1;
    pa.TR = tmp.TR; pa.RB = tmp.RB; pa.CB = tmp.CB; pa.RBx = tmp.RBx; pa.CBx = tmp.CBx;
    pa.rowpart = tmp.rowpart; pa.colpart = tmp.colpart; pa.r = tmp.r; pa.c = tmp.c;
    pa.sig_part = tmp.sig_part; pa.dlt_part = tmp.dlt_part; pa.mu_part = tmp.mu_part;
    pa.rho_part = tmp.rho_part; pa.iter_out = tmp.iters; pa.done = tmp.done;
    pa.replay = proj_replay_default();
    A(launch_proj(pa, tmp.grid, s));
    A(download(Yp, Y, 1, s));
    A(cudaMemcpyAsync(&it, tmp.iters, sizeof(DevIter), cudaMemcpyDeviceToHost, s));
    A(cudaStreamSynchronize(s));
  }
  free_buf(Yp);
  for (void* p : {(void*)tmp.rowpart, (void*)tmp.colpart, (void*)tmp.r, (void*)tmp.c,
                  (void*)tmp.sig_part, (void*)tmp.mu_part, (void*)tmp.dlt_part,
                  (void*)tmp.rho_part, (void*)tmp.iters, (void*)tmp.done})
    if (p) cudaFree(p);
  tmp.rowpart = tmp.colpart = tmp.r = tmp.c = tmp.sig_part = tmp.mu_part = nullptr;
  tmp.dlt_part = tmp.rho_part = nullptr; tmp.iters = nullptr; tmp.done = nullptr;
  if (rc == FASTPFP_OK) {
    if (sweeps_out) *sweeps_out = it.sweeps;
    if (delta_out) *delta_out = it.delta;
  }
  return rc;
}

int fastpfp_gemm_nt(const float* P, const float* Q, float* C, int64_t M, int64_t N, int64_t K,
                    int precision, int cta_group, int64_t stream) {
  if (!P || !Q || !C || M < 1 || N < 1 || K < 1 || precision < 0 || precision > 3 ||
      (cta_group != 1 && cta_group != 2))
    return FASTPFP_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FASTPFP_ENODEV;
  Buf Pp, Pb, Ps, Qp, Qb, Qs, Cp;
  int rc = FASTPFP_OK;
  auto A = [&](cudaError_t e) { if (e != cudaSuccess && rc == FASTPFP_OK) rc = FASTPFP_ECUDA; };
  A(alloc_buf(Pp, (int)M, (int)K)); A(alloc_buf(Pb, (int)M, (int)K)); A(alloc_buf(Ps, (int)M, (int)K));
  A(alloc_buf(Qp, (int)N, (int)K)); A(alloc_buf(Qb, (int)N, (int)K)); A(alloc_buf(Qs, (int)N, (int)K));
  A(alloc_buf(Cp, (int)M, (int)N));
  if (rc == FASTPFP_OK) {
    A(upload(Pp, P, 1, s)); A(upload(Qp, Q, 1, s));
    A(launch_split(Pp.p, Pp.ld, Pb.p, Ps.p, Pp.ld, (int)M, (int)K, s));
    A(launch_split(Qp.p, Qp.ld, Qb.p, Qs.p, Qp.ld, (int)N, (int)K, s));
    GemmArgs g{};
    g.P = Pp.p; g.ldP = Pp.ld; g.Pb = Pb.p; g.Ps = Ps.p;
    g.Q = Qp.p; g.ldQ = Qp.ld; g.Qb = Qb.p; g.Qs = Qs.p;
    g.M = (int)M; g.N = (int)N; g.K = (int)K; g.epi = kEpiPlain; g.C = Cp.p; g.ldC = Cp.ld;
    g.cta_group = cta_group;
    if (precision == 3) {
      I8Buf Pi, Qi;
      A(alloc_i8(Pi, (int)M, (int)K)); A(alloc_i8(Qi, (int)N, (int)K));
      if (rc == FASTPFP_OK) {
        A(split_i8(Pp, Pi, nullptr, nullptr, s)); A(split_i8(Qp, Qi, nullptr, nullptr, s));
        I8Gemm gi{};
        for (int k = 0; k < 3; ++k) { gi.P[k] = Pi.d[k]; gi.Q[k] = Qi.d[k]; }
        gi.ldP = Pi.ld; gi.eP = Pi.e; gi.ldQ = Qi.ld; gi.eQ = Qi.e;
        gi.M = (int)M; gi.N = (int)N; gi.K = (int)K; gi.epi = kEpiPlain; gi.C = Cp.p; gi.ldC = Cp.ld;
        if (!gemm_i8_supported(gi)) rc = FASTPFP_EUNSUPPORTED;
        else A(launch_gemm_i8(gi, s, dev));
      }
      A(cudaStreamSynchronize(s));
      for (I8Buf* b : {&Pi, &Qi}) {
        for (auto& d : b->d) if (d) cudaFree(d);
        if (b->e) cudaFree(b->e);
      }
    } else if (precision == 2) {
      A(launch_gemm_simt(g, s));
    } else if (!gemm_tc_supported(g)) {
      rc = FASTPFP_EUNSUPPORTED;
    } else {
      A(launch_gemm_tc(g, precision == 1 ? 1 : 3, s, dev));
    }
    if (rc == FASTPFP_OK) A(download(Cp, C, 1, s));
    A(cudaStreamSynchronize(s));
  }
  for (Buf* b : {&Pp, &Pb, &Ps, &Qp, &Qb, &Qs, &Cp}) free_buf(*b);
  return rc;
}


int fastpfp_gemm_nt_blocked(const float* P, const float* Q, float* C, int64_t M, int64_t N,
                            int64_t K, int32_t q_blocks, int precision, int64_t stream) {
  // the row-sharded GEMM2 operand layout: Q re-laid as [q_blocks][N][K / q_blocks] (the NCCL
  // all-gather output), read by the 3-D TMA K-loop of the tensor-core GEMMs
  if (!P || !Q || !C || M < 1 || N < 1 || K < 1 || q_blocks < 2 || K % q_blocks != 0 ||
      (precision != 0 && precision != 1 && precision != 3))
    return FASTPFP_EINVAL;
  const int64_t kb = K / q_blocks;
  if (kb % (precision == 3 ? 128 : 32) != 0) return FASTPFP_EUNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FASTPFP_ENODEV;
  Buf Pp, Pb, Ps, Qp, Qb, Qs, Cp, Qbb, Qsb;
  I8Buf Pi, Qi, Qib;
  int rc = FASTPFP_OK;
  auto A = [&](cudaError_t e) { if (e != cudaSuccess && rc == FASTPFP_OK) rc = FASTPFP_ECUDA; };
  A(alloc_buf(Pp, (int)M, (int)K)); A(alloc_buf(Qp, (int)N, (int)K)); A(alloc_buf(Cp, (int)M, (int)N));
  if (rc == FASTPFP_OK) {
    A(upload(Pp, P, 1, s)); A(upload(Qp, Q, 1, s));
    if (precision == 3) {
      A(alloc_i8(Pi, (int)M, (int)K)); A(alloc_i8(Qi, (int)N, (int)K));
      A(alloc_i8(Qib, (int)(q_blocks * N), (int)kb));
      if (rc == FASTPFP_OK) {
        A(split_i8(Pp, Pi, nullptr, nullptr, s)); A(split_i8(Qp, Qi, nullptr, nullptr, s));
        for (int k = 0; k < 3; ++k)
          for (int b = 0; b < q_blocks; ++b)
            A(cudaMemcpy2DAsync(Qib.d[k] + (size_t)b * N * Qib.ld, Qib.ld, Qi.d[k] + b * kb, Qi.ld,
                                kb, N, cudaMemcpyDeviceToDevice, s));
        I8Gemm gi{};
        for (int k = 0; k < 3; ++k) { gi.P[k] = Pi.d[k]; gi.Q[k] = Qib.d[k]; }
        gi.ldP = Pi.ld; gi.eP = Pi.e; gi.ldQ = Qib.ld; gi.eQ = Qi.e;
        gi.M = (int)M; gi.N = (int)N; gi.K = (int)K; gi.epi = kEpiPlain; gi.C = Cp.p; gi.ldC = Cp.ld;
        gi.q_blocks = q_blocks; gi.q_block_k = (int)kb; gi.q_block_stride = (int64_t)N * Qib.ld;
        if (!gemm_i8_supported(gi)) rc = FASTPFP_EUNSUPPORTED;
        else A(launch_gemm_i8(gi, s, dev));
      }
    } else {
      A(alloc_buf(Pb, (int)M, (int)K)); A(alloc_buf(Ps, (int)M, (int)K));
      A(alloc_buf(Qb, (int)N, (int)K)); A(alloc_buf(Qs, (int)N, (int)K));
      A(alloc_buf(Qbb, (int)(q_blocks * N), (int)kb)); A(alloc_buf(Qsb, (int)(q_blocks * N), (int)kb));
      if (rc == FASTPFP_OK) {
        A(launch_split(Pp.p, Pp.ld, Pb.p, Ps.p, Pp.ld, (int)M, (int)K, s));
        A(launch_split(Qp.p, Qp.ld, Qb.p, Qs.p, Qp.ld, (int)N, (int)K, s));
        for (int b = 0; b < q_blocks; ++b) {
          A(cudaMemcpy2DAsync(Qbb.p + (size_t)b * N * Qbb.ld, Qbb.ld * 4, Qb.p + b * kb, Qb.ld * 4,
                              kb * 4, N, cudaMemcpyDeviceToDevice, s));
          A(cudaMemcpy2DAsync(Qsb.p + (size_t)b * N * Qsb.ld, Qsb.ld * 4, Qs.p + b * kb, Qs.ld * 4,
                              kb * 4, N, cudaMemcpyDeviceToDevice, s));
        }
        GemmArgs g{};
        g.P = Pp.p; g.ldP = Pp.ld; g.Pb = Pb.p; g.Ps = Ps.p;
        g.Qb = Qbb.p; g.Qs = Qsb.p; g.ldQ = Qbb.ld;
        g.M = (int)M; g.N = (int)N; g.K = (int)K; g.epi = kEpiPlain; g.C = Cp.p; g.ldC = Cp.ld;
        g.cta_group = 2;
        g.q_blocks = q_blocks; g.q_block_k = (int)kb; g.q_block_stride = (int64_t)N * Qbb.ld;
        if (!gemm_tc_supported(g)) rc = FASTPFP_EUNSUPPORTED;
        else A(launch_gemm_tc(g, precision == 1 ? 1 : 3, s, dev));
      }
    }
    if (rc == FASTPFP_OK) A(download(Cp, C, 1, s));
    A(cudaStreamSynchronize(s));
  }
  for (Buf* b : {&Pp, &Pb, &Ps, &Qp, &Qb, &Qs, &Cp, &Qbb, &Qsb}) free_buf(*b);
  for (I8Buf* b : {&Pi, &Qi, &Qib}) {
    for (auto& d : b->d) if (d) cudaFree(d);
    if (b->e) cudaFree(b->e);
  }
  return rc;
}

}  // extern "C"
