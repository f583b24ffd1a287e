/*
 * fastpfp.h — C-ABI of the B200-native FastPFP hot path (arXiv 1207.1114, "A Fast Projected
 * Fixed-Point Algorithm for Large Graph Matching", Lu, Huang & Liu).
 *
 * Citations "P:123" are PAPER.md line numbers (the paper's LaTeX source); readings of ambiguous
 * passages are listed in DESIGN.md §Readings (A1-A20).
 *
 * The problem: two undirected graphs with symmetric adjacency A (n x n) and A'
 * (n' x n'), node attributes B (n x d) and B' (n' x d), affinity K = B B'^T. The relaxed
 * problem maximises f(X) = 1/2 tr(X^T A X A') + lambda tr(X^T K) over partial doubly stochastic X
 * (P:167-200). FastPFP iterates (Algorithm 1):
 *     Y[0:n, 0:n'] = A X A' + lambda K                              (line 3)
 *     repeat  Y = P2(P1(Y))  until max|dY| < eps2 or I_1 sweeps     (lines 4-7)
 *     X = (1 - alpha) X + alpha Y[0:n, 0:n']                        (line 8)
 *     X = X / max(X)                                                (line 9)
 * until max|dX| < eps1 or I_0 iterations; then greedy discretization.
 * Y is the m x m slacked matrix, m = max(n, n'); the smaller side is fully assigned
 * (slack columns when n > n', slack rows when n < n', reading A1).
 *
 * Conventions
 *  - All matrices crossing the boundary are dense, row-major, float32, with the exact shapes given
 *    (no padding). Host pointers unless an `is_device` flag says the pointer is CUDA device memory
 *    of the current device. Inputs are COPIED; the caller keeps ownership of every buffer it
 *    passes. Outputs are written into caller-owned buffers.
 *  - Every call returns a fastpfp_status. On FASTPFP_ECUDA / FASTPFP_ENCCL the handle is poisoned:
 *    every later call except fastpfp_destroy / fastpfp_last_error returns FASTPFP_EPOISONED.
 *  - A handle is not thread-safe; distinct handles are independent. All device work of a handle is
 *    issued on its stream (FASTPFP_OPT_STREAM, default: a private non-blocking stream); calls
 *    return after that work has completed unless documented otherwise.
 *  - There is no CPU fallback: every step of the path runs in the library's sm_100a kernels. If no
 *    sm_100a device is present fastpfp_create returns FASTPFP_ENODEV.
 */
#ifndef FASTPFP_H_
#define FASTPFP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FASTPFP_ABI_VERSION 1

typedef enum fastpfp_status {
  FASTPFP_OK = 0,
  FASTPFP_EINVAL = 1,       /* bad argument (sizes, NULL, ranges of alpha/lambda/eps/maxIter)   */
  FASTPFP_ESYM = 2,         /* A or A' not exactly symmetric (undirected graphs)     */
  FASTPFP_ENONFINITE = 3,   /* NaN/Inf in an input matrix                                       */
  FASTPFP_ESTATE = 4,       /* call order: iterate/discretize before set_graphs                 */
  FASTPFP_ENOMEM = 5,       /* device allocation failed                                         */
  FASTPFP_ECUDA = 6,        /* CUDA runtime/driver error (handle poisoned)                      */
  FASTPFP_ENCCL = 7,        /* NCCL error (handle poisoned)                                     */
  FASTPFP_ENODEV = 8,       /* no sm_100 device / library built for another architecture       */
  FASTPFP_EPOISONED = 9,    /* handle poisoned by an earlier ECUDA/ENCCL                        */
  FASTPFP_EUNSUPPORTED = 10 /* option/shape combination not implemented                         */
} fastpfp_status;

typedef struct fastpfp_handle fastpfp_handle;

/* Per-call iteration report (SURVEY §5 "Tracing": the paper's only instrumentation is the
 * eps1 trace). Trace arrays are caller-owned and optional (trace_capacity = 0 or NULL
 * pointers disable them); entry k describes outer iteration k of THIS call. */
typedef struct fastpfp_report {
  int32_t iterations;    /* outer iterations completed by this call (X updated that many times)  */
  int32_t converged;     /* 1 iff the loop stopped because rho < eps1                */
  int32_t degenerate;    /* 1 iff max(X~) <= 1e-300 stopped the loop; X is left unchanged         */
  int32_t total_sweeps;  /* projection sweeps (P1+P2 pairs) summed over the call                  */
  double last_rho;       /* max|X^(t+1) - X^(t)| of the last iteration, after the rescale (A6)   */
  double last_delta;     /* max|Y^(s+1) - Y^(s)| of the last sweep (A5)                          */
  double last_mu;        /* max(X~) used by the last rescale                             */
  int32_t trace_capacity;
  int32_t reserved;
  double* rho_trace;     /* [trace_capacity] or NULL                                            */
  int32_t* sweeps_trace; /* [trace_capacity] or NULL                                            */
  double* delta_trace;   /* [trace_capacity] or NULL                                            */
  double* mu_trace;      /* [trace_capacity] or NULL                                            */
} fastpfp_report;

/* Options (fastpfp_set_option keys). */
typedef enum fastpfp_option {
  /* 0 = persist (default): slack entries of Y keep their values across outer iterations, as
   *     Algorithm 1 initialises Y once and only overwrites Y[0:n,0:n'], reading A3.
   * 1 = reset: slack set to 0 before every projection (SPEC's variant). */
  FASTPFP_OPT_SLACK_MODE = 1,
  /* Default: 3 where it applies (n, n' <= 32768; sharded: (n/P) % 128 == 0), else 0.
   * 0 = 3xTF32 tensor-core GEMMs (tcgen05; fp32-accurate)
   * 1 = 1xTF32 tensor-core GEMMs (reported separately; NOT parity-accurate)
   * 2 = fp32 SIMT GEMMs (FFMA; the scaffold the tensor-core path is checked against)
   * 3 = Ozaki int8 tensor-core GEMMs (tcgen05 kind::i8; every operand row = a power-of-two scale
   *     and three signed 7-bit digit planes, six exact int32 digit products in three weight
   *     classes; fp32-accurate). Needs n, n' <= 32768 (exact int32 class sums);
   *     sharded handles need (n/P) % 128 == 0 (else
   *     EUNSUPPORTED); allocates 3 bytes per element of A, A', X, U (+ U in fp32) on first
   *     selection. Switching precision after set_graphs re-derives the operand form the new
   *     precision reads (digit planes or TF32 parts of A, A' and the current X). Sharded: the row scales of U are all-reduced (MAX) and U's digit planes, not its
   *     TF32 parts, are all-gathered (3 instead of 8 bytes per element). */
  FASTPFP_OPT_PRECISION = 2,
  /* 1 (default) = X <- X/max(X) each iteration; 0 = off (Theorem 1 test, reading A11). */
  FASTPFP_OPT_RESCALE = 3,
  /* cudaStream_t (as int64) on which all work of the handle is issued; 0 = private stream. */
  FASTPFP_OPT_STREAM = 4,
  /* outer iterations launched between host convergence checks (>= 1, default 4). Extra launched
   * iterations after convergence are no-ops on the device, so the result is identical. */
  FASTPFP_OPT_CHECK_EVERY = 5,
  /* 1 = record CUDA events around every GEMM and projection launch on the handle's stream and
   * accumulate their device time into fastpfp_stats (bench.py's per-kernel roofline); 0 = off. */
  FASTPFP_OPT_PROFILE = 6,
  /* tensor-core GEMM tiling: 2 (default) = 256 x 256 tiles per CTA pair (tcgen05 cta_group::2),
   * 1 = 128 x 128 tiles per CTA (cta_group::1). Same arithmetic, same results up to ordering. */
  FASTPFP_OPT_GEMM_CTA_GROUP = 7,
  /* projection kernel: 0 = auto (on-chip tiles exchanging tagged partial-sum records once per sweep
   * when Y fits in the aggregate shared memory, m <~ 2.2k; one CTA for m <= 128; else streaming),
   * 1 = streaming, 2 = on-chip (EUNSUPPORTED if Y does not fit). Same arithmetic; sums are reduced
   * in a different fixed order. */
  FASTPFP_OPT_PROJ_KERNEL = 8,
  /* 0 = FastPFP (Algorithm 1; default). 1 = Projected Gradient {pg}:
   * X <- P_d(X + alpha (A X A' + lambda K)), same projection, initialisation and stopping rules,
   * no blend and no rescale (alpha is the gradient step). SURVEY §8(f2).
   * 2 = FastGA (Appendix "FastGA", `{GAO3}`): per outer iteration
   * X <- Sinkhorn(exp(beta_t (A X A' + lambda K))) on the slack-padded m x m matrix,
   * beta_t = beta0 rate^t (fastpfp_set_ga_schedule); alpha is ignored; readings G1-G8 in DESIGN.md
   * §3b. Single-GPU handles only (EUNSUPPORTED on a sharded handle). Allocates an m x m fp64
   * workspace on first selection (ENOMEM if it does not fit). In the report, a FastGA iteration's
   * "mu" entries carry beta_t and delta = +inf when only one Sinkhorn sweep ran. */
  FASTPFP_OPT_METHOD = 9,
  /* Sharded handles (SURVEY §5 failure detection): every host wait on the handle's stream polls
   * the stream and ncclCommGetAsyncError; an asynchronous NCCL error, or collectives not complete
   * after this many milliseconds (default 600000; a peer that died or hung), aborts the
   * communicator and returns ENCCL (the handle is poisoned). Ignored on single-GPU handles. */
  FASTPFP_OPT_NCCL_TIMEOUT_MS = 10
} fastpfp_option;

/* Counters of a handle (since creation or the last fastpfp_reset_stats). */
typedef struct fastpfp_stats {
  int64_t launches;          /* kernels launched by iterate (GEMMs, projection, slack reset)    */
  int64_t gemm_launches;     /* of which GEMM launches (the two products of P:387)             */
  int64_t proj_launches;     /* of which persistent projection/finalize launches   */
  int64_t outer_iterations;  /* completed outer iterations                                     */
  int64_t sweeps;            /* projection sweeps                                              */
  double gemm_ms;            /* device time of GEMM launches (FASTPFP_OPT_PROFILE = 1)         */
  double proj_ms;            /* device time of projection launches (FASTPFP_OPT_PROFILE = 1)   */
  double gemm_flops;         /* algorithmic flops of the timed GEMM launches (2 M N K each)     */
  int64_t onchip_launches;   /* of proj_launches, how many used the on-chip projection kernel  */
  int32_t onchip_tiles;      /* PR * PC tiles of the on-chip kernel (0 if Y does not fit)      */
  int32_t reserved;
} fastpfp_stats;

/* ---------------------------------------------------------------------------------------------
 * Single pair
 * ------------------------------------------------------------------------------------------- */

/* Create a handle for graphs of n and n' nodes with d attributes per node (d = 0: no attributes,
 * K = 0). Either orientation is accepted (reading A1). Allocates all device state (A, A' and their
 * TF32 splits, K, X, Y (m x m), U, reduction scratch). *out is owned by the caller and released
 * with fastpfp_destroy. Errors: EINVAL (n, n' < 1, d < 0, out NULL), ENODEV, ENOMEM. */
int fastpfp_create(int64_t n, int64_t n_prime, int64_t d, fastpfp_handle** out);

/* FastGA annealing schedule (reading G5; the paper publishes none): outer iteration t
 * uses beta_t = beta0 * rate^t, and fastpfp_iterate stops once beta_t > beta_max (t counts the
 * handle's completed iterations since the last reset). Defaults 0.5, 1.075, 10. Errors: EINVAL
 * unless beta0 > 0, rate >= 1, beta_max >= 0, all finite. */
int fastpfp_set_ga_schedule(fastpfp_handle* h, double beta0, double rate, double beta_max);

/* Load the graphs: A n x n, A_prime n' x n', B n x d, B_prime n' x d (B, B_prime may be
 * NULL iff d = 0). A and A' must be exactly symmetric (ESYM; not symmetrised) and finite
 * (ENONFINITE). Computes K = B B'^T on the device and resets X <- X0, slack <- 0, t <- 0. */
int fastpfp_set_graphs(fastpfp_handle* h, const float* A, const float* A_prime, const float* B,
                       const float* B_prime, int is_device);

/* Store the initial X0 (n x n', finite) and reset (X <- X0, Y <- 0, t <- 0). X0 == NULL selects
 * the paper's X0 = 1 1^T / (n n'). BASELINE configs[0] uses 1/n * ones (reading A4). */
int fastpfp_set_x0(fastpfp_handle* h, const float* X0, int is_device);

/* Re-initialise from the stored X0: X <- X0, Y <- 0, t <- 0. */
int fastpfp_reset(fastpfp_handle* h);

/* Run up to max_iter1 outer iterations of Algorithm 1 CONTINUING from the handle's
 * state, so k calls with max_iter1 = 1 equal one call with max_iter1 = k. alpha in [0,1]
 * (P:207-211), lambda >= 0, eps1/eps2 >= 0 (0 => run exactly max_iter; strict '<' tests, readings
 * A5/A6), max_iter1 >= 1 (I_0), max_iter2 >= 1 (I_1, sweeps per projection, at least one).
 * X_out (nullable, host, n x n') receives X after the last rescale. rep (nullable) is filled.
 * Non-convergence is not an error. Errors: EINVAL, ESTATE, ECUDA. */
int fastpfp_iterate(fastpfp_handle* h, double alpha, double lambda, double eps1, double eps2,
                    int32_t max_iter1, int32_t max_iter2, float* X_out, fastpfp_report* rep);

/* Copy the current X (n x n') to dst (host if dst_is_device == 0, else device memory). */
int fastpfp_copy_x(fastpfp_handle* h, float* dst, int dst_is_device);

/* Copy the current slacked matrix Y to dst (diagnostics, tests, checkpoints): m x m with
 * m = max(n, n') on a single-GPU handle; on a row-sharded handle the LOCAL rows, n/P x m. After an
 * outer iteration Y holds the last projection output; its slack part (columns n'..m-1 when n > n',
 * rows n..m-1 when n < n') is the state Algorithm 1 carries into the next iteration. */
int fastpfp_copy_y(fastpfp_handle* h, float* dst, int dst_is_device);

/* Checkpoint/resume of the slack: load Y (same shape as fastpfp_copy_y writes, finite,
 * else ENONFINITE) into the handle without touching X. Algorithm 1 initialises Y once and
 * overwrites only Y[0:n, 0:n'] each iteration, so a run resumed with
 * fastpfp_set_x0(X_saved) followed by fastpfp_set_y(Y_saved) continues exactly as the original
 * (set_x0 zeroes Y, so set_y must come after it). Errors: EINVAL, ESTATE (before set_graphs). */
int fastpfp_set_y(fastpfp_handle* h, const float* Y, int is_device);

/* Greedy discretization of the current X (Algorithm 1 line 11): repeatedly take the
 * largest remaining X_ij (ties: smaller i, then smaller j, reading A12) and strike row i and
 * column j, until min(n, n') pairs are taken. assign (host, length n): assign[i] = matched column
 * j, or -1 for an unmatched row (n > n'). */
int fastpfp_discretize(fastpfp_handle* h, int32_t* assign);

/* f(X) = 1/2 tr(X^T A X A') + lambda tr(X^T K) at the current X, accumulated in
 * fp64 over fp32 products. */
int fastpfp_objective(fastpfp_handle* h, double lambda, double* f);

/* ---------------------------------------------------------------------------------------------
 * Row-sharded single pair over P GPUs of one node (BASELINE configs[4], one process per GPU)
 *
 * Rank r owns rows [r n/P, (r+1) n/P) of A, X, K, B and Y; A' and B' are replicated. Per outer
 * iteration: GEMM1 U_r = A' X_r^T locally; NCCL all-gather of U's TF32 parts over NVLink;
 * GEMM2 Y_r = A_r U^T + lambda K_r with a K-loop over the gathered rank blocks; per sweep an NCCL
 * all-reduce (SUM) of the m column sums and sigma (row sums are local); all-reduce (MAX) of mu
 * and rho. With eps2 > 0 the inner stop test runs on the device (sweeps
 * are enqueued 8 at a time, launches past the stop are no-ops; one host check per 8 sweeps). Requirements: n >= n', n % P == 0, (n/P) % 32 == 0 (else
 * EUNSUPPORTED); tensor-core precision (0, 1 or 3).
 * On a sharded handle: fastpfp_set_graphs takes the LOCAL rows of A (n/P x n, row-major) and of B
 * (n/P x d) and the full A' and B' (A's symmetry is the caller's contract; finiteness is checked);
 * set_x0 / iterate's X_out / copy_x use the local rows of X (n/P x n'); fastpfp_discretize gathers
 * X and returns the full assignment (length n) on every rank; fastpfp_objective returns the global
 * f on every rank. All ranks must make the same calls in the same order (collectives).
 * ------------------------------------------------------------------------------------------- */

/* Write a fresh NCCL unique id (128 bytes) to out (call on rank 0; broadcast it to all ranks,
 * e.g. over the torch process group). Errors: EINVAL (size < 128), ENCCL (NCCL not loadable). */
int fastpfp_nccl_unique_id(void* out, int64_t size);

/* Collective: every rank calls it with the same n, n', d, world and id. */
int fastpfp_create_dist(int64_t n, int64_t n_prime, int64_t d, int rank, int world,
                        const void* nccl_id, fastpfp_handle** out);

/* The collectives the last fastpfp_iterate / fastpfp_objective / fastpfp_discretize call of a
 * sharded handle issued, in order (empty on single-GPU handles): out[4k .. 4k+3] = {kind (0
 * all-reduce, 1 all-gather), ncclDataType_t, ncclRedOp_t (-1 for all-gather), element count}; at
 * most `capacity` entries are written, *count receives the total. The per-outer-iteration sequence
 * is the one paper_1207_1114_b200/dist.py collective_schedule describes.
 * Errors: EINVAL. */
int fastpfp_dist_collectives(fastpfp_handle* h, int64_t* out, int64_t capacity, int64_t* count);

/* Set an option (fastpfp_option). Errors: EINVAL for unknown keys or values. */
int fastpfp_set_option(fastpfp_handle* h, int key, int64_t value);

/* Read the current value of an option (e.g. the precision the handle chose by default).
 * Errors: EINVAL for unknown keys or a NULL value pointer. */
int fastpfp_get_option(fastpfp_handle* h, int key, int64_t* value);

/* Read / clear the handle's counters. */
int fastpfp_get_stats(fastpfp_handle* h, fastpfp_stats* out);
int fastpfp_reset_stats(fastpfp_handle* h);

/* Release every resource of the handle (NULL is a no-op). */
void fastpfp_destroy(fastpfp_handle* h);

/* Last error message of the handle (never NULL; "" if none). Valid until the next call on h. */
const char* fastpfp_last_error(const fastpfp_handle* h);

/* Static description of a status code. */
const char* fastpfp_status_string(int status);

/* ABI version (FASTPFP_ABI_VERSION) and the compiled device architecture (e.g. 100). */
int fastpfp_abi_version(void);
int fastpfp_device_arch(void);

/* ---------------------------------------------------------------------------------------------
 * Batches of small pairs (BASELINE configs[3]: 8192 independent pairs of n = n' = 128)
 *
 * Every pair runs the whole of Algorithm 1 inside one CTA, on chip, with its own
 * convergence; the same scalars (alpha, lambda, eps, maxIter) apply to all pairs.
 * Arrays are pair-major and dense: A [batch][n][n], A' [batch][n'][n'], B [batch][n][d],
 * B' [batch][n'][d], X [batch][n][n']. Limits: 1 <= n, n' <= 128. Projection arithmetic is fp32
 * here; products are int8 Ozaki tcgen05 MMAs (default) or fp32 FFMA. Multi-GPU: pairs are split across ranks by the
 * caller (one handle per GPU, no communication, BASELINE configs[3] "pairs split evenly").
 * ------------------------------------------------------------------------------------------- */
typedef struct fastpfp_batched fastpfp_batched;

/* Errors: EINVAL (batch < 1, sizes outside [1,128], d < 0), ENODEV, ENOMEM. */
int fastpfp_batched_create(int64_t batch, int64_t n, int64_t n_prime, int64_t d,
                           fastpfp_batched** out);
/* Load all pairs (copied; ESYM / ENONFINITE as fastpfp_set_graphs); K = B B'^T per pair;
 * resets every pair to X0 (default 1 1^T/(n n')) and zero slack. */
int fastpfp_batched_set_graphs(fastpfp_batched* h, const float* A, const float* A_prime,
                               const float* B, const float* B_prime, int is_device);
/* X0 [batch][n][n'] (NULL: 1 1^T/(n n') for every pair); resets all pairs. */
int fastpfp_batched_set_x0(fastpfp_batched* h, const float* X0, int is_device);
/* Up to max_iter1 outer iterations per pair, continuing from each pair's state. Per-pair outputs
 * (host arrays of length batch, each nullable): iterations done, converged flag, sweeps made. */
int fastpfp_batched_iterate(fastpfp_batched* h, double alpha, double lambda, double eps1,
                            double eps2, int32_t max_iter1, int32_t max_iter2, float* X_out,
                            int32_t* iterations, int32_t* converged, int32_t* sweeps);
/* Current X of all pairs to dst ([batch][n][n'], host or device). */
int fastpfp_batched_copy_x(fastpfp_batched* h, float* dst, int dst_is_device);
/* Greedy discretization (ties: smaller row, then column) of every pair on the device:
 * assign [batch][n] (host), assign[p*n + i] = column or -1. */
int fastpfp_batched_discretize(fastpfp_batched* h, int32_t* assign);
/* Options: STREAM, RESCALE, PRECISION (3 = the two products on the int8 tensor cores with the Ozaki
 * digit decomposition, fp32-accurate, default; 2 = fp32 SIMT FFMA). */
int fastpfp_batched_set_option(fastpfp_batched* h, int key, int64_t value);
int fastpfp_batched_get_stats(fastpfp_batched* h, fastpfp_stats* out);
void fastpfp_batched_destroy(fastpfp_batched* h);
const char* fastpfp_batched_last_error(const fastpfp_batched* h);

/* ---------------------------------------------------------------------------------------------
 * Building blocks (exposed for unit parity tests; same kernels the iterate path launches).
 * All pointers are DEVICE pointers, dense row-major float32 unless stated; stream 0 = default.
 * ------------------------------------------------------------------------------------------- */

/* One projection sweep (Algorithm 1 lines 5-6) applied k times in place to the m x m
 * matrix Y (device, dense, ld = m), stopping early when max|dY| < eps2. *sweeps_out,
 * *delta_out (host) receive the count and the last delta. Row/column sums are combined in fp64;
 * the first sweep's P1 correction is fp64, the later sweeps' fp32 (checkpointed sweeps: Y stored
 * every other sweep). */
int fastpfp_project(float* Y, int64_t m, double eps2, int32_t max_iter2, int32_t* sweeps_out,
                    double* delta_out, int64_t stream);

/* C[M x N] = P[M x K] * Q[N x K]^T (both operands K-major, i.e. row-major with K contiguous) in
 * the given precision (FASTPFP_OPT_PRECISION values 0-3; 3 needs K <= 32768) and tensor-core tiling cta_group (1 or 2,
 * FASTPFP_OPT_GEMM_CTA_GROUP); the product behind A X A'. */
int fastpfp_gemm_nt(const float* P, const float* Q, float* C, int64_t M, int64_t N, int64_t K,
                    int precision, int cta_group, int64_t stream);

/* The same product with Q re-laid internally as [q_blocks][N][K / q_blocks] — the layout the
 * row-sharded path's all-gather produces — so the 3-D TMA K-loop of the GEMM2 of a P-rank run is
 * exercised on one GPU. precision 0, 1 (TF32, (K/q_blocks) % 32 == 0) or 3 (int8 Ozaki,
 * (K/q_blocks) % 128 == 0; Q's row scales span the whole K as in the sharded run). q_blocks >= 2,
 * K % q_blocks == 0. Errors: EINVAL, EUNSUPPORTED, ECUDA. */
int fastpfp_gemm_nt_blocked(const float* P, const float* Q, float* C, int64_t M, int64_t N,
                            int64_t K, int32_t q_blocks, int precision, int64_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTPFP_H_ */
