// common.cuh — shared device helpers and internal declarations of the FastPFP B200 library.
// Everything here is product code (no oracle); see include/fastpfp.h for the public contract.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fpfp {

constexpr int kWarp = 32;

__host__ __device__ inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t q) { return (x + q - 1) / q; }

// TF32 round-to-nearest (ties away), the split used by the 3xTF32 GEMM: a = big + small with
// big = rna_tf32(a), small = rna_tf32(a - big) (a - big is exact in fp32).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Ozaki digit helpers (no XU-pipe conversions): round-to-nearest-even via the 1.5 * 2^23 magic
// constant (exact for |x| < 2^22), exponents from the float bits.
__device__ __forceinline__ int frexp_exp(float mx) {   // e with mx = f 2^e, f in [0.5, 1); 0 for mx = 0
  const int bits = __float_as_int(mx);
  const int E = (bits >> 23) & 0xFF;
  if (E != 0) return E - 126;
  int e = 0;
  if (mx != 0.0f) frexpf(mx, &e);                      // subnormal: rare
  return e;
}
__device__ __forceinline__ float exp2i(int e) {         // exact 2^e
  return (e > -127 && e < 128) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e);
}
// the three signed 7-bit digits of r0 = x 2^-e (given as x * inv, |r0| < 1), d = clamp(rint(128 r), +-127)
__device__ __forceinline__ void ozaki_digits3(float x, float inv, int& a, int& b, int& c) {
  constexpr float kMagic = 12582912.0f;                 // 1.5 * 2^23
  const float r0 = x * inv * 128.0f;                    // exact (power-of-two scaling)
  const float fa = fminf(fmaxf((r0 + kMagic) - kMagic, -127.0f), 127.0f);
  const float r1 = (r0 - fa) * 128.0f;                  // exact remainder
  const float fb = fminf(fmaxf((r1 + kMagic) - kMagic, -127.0f), 127.0f);
  const float r2 = (r1 - fb) * 128.0f;
  const float fc = fminf(fmaxf((r2 + kMagic) - kMagic, -127.0f), 127.0f);
  a = __float_as_int(fa + kMagic) - 0x4B400000;
  b = __float_as_int(fb + kMagic) - 0x4B400000;
  c = __float_as_int(fc + kMagic) - 0x4B400000;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// fp32: one warp-wide reduction instruction on sm_100a (CREDUX.MAX.F32) instead of 5 shuffle +
// max steps; same value as the butterfly (max is exact and order-free; NaN-ignoring like fmaxf)
#ifndef FPFP_NO_REDUX
template <>
__device__ __forceinline__ float warp_max<float>(float v) {
  float r;
  asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
#endif

// Per-outer-iteration record written by the projection/finalize kernel (device memory).
struct DevIter {
  int32_t valid;       // 1 if this outer iteration ran (X updated or degenerate detected)
  int32_t sweeps;      // projection sweeps made
  int32_t degenerate;  // max(X~) <= 1e-300
  int32_t converged;   // rho < eps1
  double delta;        // last sweep's max|dY|
  double mu;           // max(X~)
  double rho;          // max|X_new - X_old|
};

// Arguments of the persistent projection + finalize kernel (proj.cu).
enum ProjMode { kProjFull = 0, kProjSums = 1, kProjOneSweep = 2, kProjFinMu = 3, kProjFinApply = 4 };

// On-chip projection (proj_onchip_kernel): the m x m Y is split into PR x PC tiles, one per CTA,
// each resident in shared memory for the whole inner loop; one grid barrier per sweep.
struct OnchipArgs {
  float* Y; int64_t ldY; int m;
  float* X; float* Xb; float* Xs; int64_t ldX; int n, np;
  double alpha, eps1, eps2;
  int max_iter2, rescale, do_finalize;
  int PR, PC, TRo, TCo;          // tile grid and tile extent
  // exchange buffers, each value a 16-byte tagged record {lo32, tag, hi32, tag} (tag = the
  // launch epoch and sweep: the reader polls until both tags match, no barrier)
  double* rowp;                  // [2][PC][m] row partials (2 doubles of storage per record)
  double* colp;                  // [2][PR][m] column partials
  double* tot;                   // [2][PR*PC] tile totals
  float* dlt;                    // [2][PR*PC] tile deltas (4 floats of storage per record)
  unsigned epoch;                // launch epoch (host counter, never 0 mod 2^16)
  double* mu_part;               // [PR*PC]
  float* rho_part;               // [PR*PC]
  DevIter* iter_out;
  int* done;
};
constexpr int kOnchipMaxTC = 256;
cudaError_t launch_proj_onchip(const OnchipArgs& a, cudaStream_t s);
bool onchip_fits(int m, int num_sms, int& PR, int& PC, int& TRo, int& TCo);

struct ProjArgs {
  int mode;                                    // ProjMode (kProjFull: whole inner loop + finalize)
  float* Y; int64_t ldY; int m;                // slacked matrix, rows x m (row stride ldY, 16B rows)
  int rows;                                    // rows of Y held here (m on one GPU, n/P when sharded)
  float* X; float* Xb; float* Xs; int64_t ldX; // soft assignment n x n' and its TF32 split
  int n, np;
  double alpha, eps1, eps2;
  int max_iter2;
  int rescale, split, do_finalize, do_sums;
  // optional (int8 path): the finalize also writes the new X's Ozaki digit planes and row exponents
  // (what split_i8_kernel would compute from it), using per-row max |X~| gathered in the mu pass
  int8_t* xd[3]; int64_t ldxd; int* xe; unsigned long long* xrowmax;
  int TR, RB, CB;        // sweep tiles: TR rows x 512 cols over m x m
  int RBx, CBx;          // finalize tiles over n x n'
  double* rowpart;       // [CB][rows]
  double* colpart;       // [RB][m]
  double* r;             // [rows]
  double* c;             // [m + 1]: column sums, c[m] = sigma (dist all-reduce buffer)
  double* scal;          // dist scalars: [0] delta_local, [1] mu, [2] rho (or -1: degenerate)
  double* sig_part;      // [grid]
  float* dlt_part;       // [grid]
  double* mu_part;       // [grid]
  float* rho_part;       // [grid]
  DevIter* iter_out;     // this iteration's record
  int* done;             // early-exit flag (converged / degenerate)
  // kProjOneSweep (sharded path): [0] sweeps made in this projection, [1] inner loop stopped. A
  // sweep launch first applies the stop test of the previous sweep (global delta in scal[0] < eps2)
  // on the device, so launches enqueued past the stop are no-ops (nullptr: no test).
  int* inner;
  // kProjFull: tile counter (zeroed before the launch). Tiles of each pass are handed out by an
  // atomic counter instead of a static round robin, so fast blocks take more tiles and the wait at
  // the pass's grid barrier shrinks; results do not depend on which block ran a tile (partials are
  // indexed by tile). nullptr: static schedule.
  unsigned* tile_ctr;
  // kProjFull, single GPU: checkpointed sweeps (proj.cu replay_pass): Y stored every other sweep,
  // the sweeps after the first re-applied from the last stored Y in fp32. r and c then hold two
  // kProjReplayC generations ([kProjReplayC][rows] and [kProjReplayC][m + 1]).
  int replay;
};
#ifndef FPFP_PROJ_REPLAY_C
#define FPFP_PROJ_REPLAY_C 2
#endif
constexpr int kProjReplayC = FPFP_PROJ_REPLAY_C;   // replay: Y stored every kProjReplayC sweeps
// default of ProjArgs::replay (environment FPFP_PROJ_REPLAY=0 turns it off: experiments / A-B)
int proj_replay_default();

constexpr int kProjThreads = 256;
#ifndef FPFP_PROJ_TC
#define FPFP_PROJ_TC 256
#endif
constexpr int kProjTC = FPFP_PROJ_TC;  // columns per projection tile (32 lanes x float4 x TC/128 chunks)

// host-side launchers (return cudaError_t)
cudaError_t launch_proj(const ProjArgs& a, int grid, cudaStream_t s);
int proj_max_grid(int device);
cudaError_t launch_split(const float* src, int64_t lds, float* big, float* small, int64_t ldd,
                         int rows, int cols, cudaStream_t s);
cudaError_t launch_check_sym(const float* A, int64_t lda, int n, int* flags, cudaStream_t s);
cudaError_t launch_check_finite(const float* A, int64_t lda, int rows, int cols, int* flags,
                                cudaStream_t s);
cudaError_t launch_fill(float* A, int64_t lda, int rows, int cols, float v, cudaStream_t s);
cudaError_t launch_zero_slack(float* Y, int64_t ldY, int rows, int m, int n, int np,
                              const int* done, cudaStream_t s);
// objective sums over X∘G and X∘K; part: kDotBlocks x 2 fp64 scratch
constexpr int kDotBlocks = 592;
cudaError_t launch_dot2(const float* X, const float* G, const float* K, int64_t ld, int rows,
                        int cols, double* part, double* out2, cudaStream_t s);

// GEMM: C[M x N] = P[M x K] * Q[N x K]^T (+ epilogue). Both operands K-major.
enum GemmEpi { kEpiPlain = 0, kEpiAxpy = 1, kEpiSplit = 2, kEpiPG = 3, kEpiRowMax = 4 };
struct GemmArgs {
  const float* P; int64_t ldP;     // plain fp32 operands (SIMT path)
  const float* Q; int64_t ldQ;
  const float* Pb; const float* Ps; // TF32 splits (tensor-core path), same ld as P
  const float* Qb; const float* Qs; // same ld as Q
  int M, N, K;
  int epi;
  float* C; int64_t ldC;           // plain output (or big part in kEpiSplit)
  float* C2;                       // small part (kEpiSplit), ld = ldC
  float* C3;                       // optional plain copy in kEpiSplit (nullable), ld = ldC
  const float* D; int64_t ldD; float lam;  // kEpiAxpy: C = acc + lam * D
  const float* D2; int64_t ldD2; float scale;  // kEpiPG: C = scale * (acc + lam * D) + D2
  const int* done;                 // nullable early-exit flag
  int cta_group = 2;               // tensor-core path: 1 = 128x128 tiles per CTA, 2 = 256x256 per CTA pair
  // row-sharded GEMM2: Q = [q_blocks][N][q_block_k] (one block per rank, block stride in floats)
  int q_blocks = 1, q_block_k = 0;
  int64_t q_block_stride = 0;
};
// Batched small-pair whole solve (small_solve.cu), n, n' <= 128, one pair per CTA.
struct SmallArgs {
  int batch, n, np, m;
  const float* A;   // [batch][n][n]
  const float* Ap;  // [batch][np][np]
  const float* K;   // [batch][n][np] or null
  float* X;         // [batch][n][np] state
  float* Y;         // [batch][m][m] slack state (null when n == np)
  float alpha, lam, eps1, eps2;
  int max_iter1, max_iter2, rescale;
  int32_t* iters;   // [batch] outer iterations done by this call
  int32_t* conv;    // [batch]
  int32_t* sweeps;  // [batch] total sweeps
  float* rho;       // [batch] last rho
  int32_t* degen;   // [batch]
  // int8 tensor-core kernel (small_solve_tc.cu): per pair the swizzled digit-plane images of A', A
  // and the current X ([batch][3][3][128 x 128] int8) and the row exponents of A', A ([batch][2][128])
  int8_t* dig;
  int* dexp;
};
size_t small_smem_bytes();
cudaError_t launch_small_solve(const SmallArgs& a, int grid, cudaStream_t s);
// the same whole solve with the products on the int8 tensor cores (small_solve_tc.cu)
size_t small_tc_smem_bytes();
size_t small_tc_digit_bytes_per_pair();
size_t small_tc_exp_ints_per_pair();
cudaError_t launch_small_digits_prep(const SmallArgs& a, int grid, cudaStream_t s);
cudaError_t launch_small_solve_tc(const SmallArgs& a, int grid, cudaStream_t s);
cudaError_t launch_small_greedy(const float* X, int batch, int n, int np, int32_t* assign, int grid,
                                cudaStream_t s);

// FastGA normalisation (ga.cu): stabilised exp of the GEMM output + slack-padded Sinkhorn + X
// update, one cooperative kernel per outer iteration.
struct GaArgs {
  const float* Q; int64_t ldQ;   // exponent A X A' + lambda K on the n x n' block (Y buffer)
  int m, n, np;
  double beta, eps1, eps2;
  int max_iter2;
  int W;                         // pass-C column chunk width (8, 16 or 32)
  double* E; int64_t ldE;        // m x m fp64 workspace
  double* u; double* v;          // [2][ldE] each (sweep-parity double buffers)
  double* dlt_part; double* rho_part;  // [grid]
  float* X; float* Xb; float* Xs; int64_t ldX;
  DevIter* iter_out;
  int* done;
};
cudaError_t launch_ga(const GaArgs& a, int grid, cudaStream_t s);
int ga_max_grid(int device);
int ga_chunk_width(int m, int grid);

// Ozaki int8 GEMM (gemm_i8.cu): C[M x N] = P Q^T with P, Q given as 3 int8 digit planes (row
// stride ldP / ldQ bytes, K contiguous) and per-row power-of-two exponents eP / eQ.
struct I8Gemm {
  const int8_t* P[3]; int64_t ldP; const int* eP;
  const int8_t* Q[3]; int64_t ldQ; const int* eQ;
  int M, N, K;
  int epi;                          // kEpiPlain, kEpiAxpy, kEpiPG or kEpiRowMax
  float* C; int64_t ldC;
  const float* D; int64_t ldD; float lam;
  const float* D2; int64_t ldD2; float scale;
  unsigned* rowmax;                 // kEpiRowMax: [M] |max| bits (zeroed by the caller)
  const int* done;
  // row-sharded GEMM2: Q planes = [q_blocks][N][q_block_k] (block stride in bytes)
  int q_blocks = 1, q_block_k = 0;
  int64_t q_block_stride = 0;
};
bool gemm_i8_supported(const I8Gemm& g);
cudaError_t launch_gemm_i8(const I8Gemm& g, cudaStream_t s, int device);
// fp32 rows x K (stride lds floats) -> 3 digit planes (stride ldd bytes) + exponents; rowmax
// (nullable) supplies max|row| bits, else it is computed.
cudaError_t launch_split_i8(const float* src, int64_t lds, int rows, int K, const unsigned* rowmax,
                            int8_t* const d[3], int64_t ldd, int* ex, const int* done, cudaStream_t s);

cudaError_t launch_gemm_simt(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_gemm_tc(const GemmArgs& g, int passes, cudaStream_t s, int device);
bool gemm_tc_supported(const GemmArgs& g);

}  // namespace fpfp
