// proj_onchip.cu — the projection loop (Algorithm 1 lines 4-7) plus blend/rescale
// (lines 8-9) for m small enough that Y fits in the GPU's aggregate shared memory (m <~ 2.2k:
// BASELINE configs[1] and [2], n ~ 1000). Y is split into PR x PC tiles, one per CTA, read from
// HBM/L2 once, kept in shared memory (fp32, Y's storage precision) across all sweeps and written back
// once. Sums are fp64 beyond short fp32 chains; the first sweep after the product (which cancels its
// large values) is fp64 arithmetic, the later ones fp32 (see the note in the kernel).
//
// Each sweep: update the own tile with the row sums r_i (own rows), column sums c_j (own columns)
// and sigma of the previous Y; emit fp64 partial row/column sums of the new tile, its total and its
// delta to a double-buffered global exchange; every CTA then re-reduces just the partials of its
// own rows / columns (PC and PR values each) and the PR*PC totals in a fixed order, so every CTA
// holds bit-identical r, c, sigma and delta (deterministic, no float atomics). At n ~ 1000 the
// exchange is the cost, so it has no grid barrier: every exchanged value travels as a tagged
// 16-byte record {lo32 | tag << 32, hi32 | tag << 32} (two single-copy-atomic 64-bit words, tag =
// launch epoch and sweep), and a reader polls the records it needs until both tags match, so the
// synchronisation and the data share one L2 round trip.
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>
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
  union {                     // per-warp column partials: fp64 (sums pass, first sweep) or fp32
    double d[kWarps][kOnchipMaxTC];
    float f[kWarps][kOnchipMaxTC];
  } colsum;
  double r[kOnchipMaxTC];     // own rows' sums
  double c[kOnchipMaxTC];     // own columns' sums
  float uf[kOnchipMaxTC];     // fl32(c_j / m) for the fp32 sweeps (padding columns: 3e38)
  double red[kWarps];
  float dred[kWarps];
  double bc[4];
};

// tagged exchange records (see the header): written and polled with .relaxed.gpu 64-bit words
__device__ __forceinline__ void st_tagged(void* dst, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(dst), "l"((u & 0xffffffffull) | t),
               "l"((u >> 32) | t) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_tagged(const void* src) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src) : "memory");
  return v;
}
__device__ __forceinline__ bool has_tag(const ulonglong2& v, unsigned tag) {
  return (unsigned)(v.x >> 32) == tag && (unsigned)(v.y >> 32) == tag;
}
__device__ __forceinline__ double tagged_value(const ulonglong2& v) {
  return __longlong_as_double((long long)((v.x & 0xffffffffull) | (v.y << 32)));
}

// 8-byte records {fp32 value | tag << 32} (one single-copy-atomic word) for the partial sums of the
// fp32 sweeps (FPFP_OC_REC32): half the bytes every CTA polls per sweep
__device__ __forceinline__ void st_tagged32(void* dst, float v, unsigned tag) {
  const unsigned long long w = (unsigned long long)__float_as_uint(v) | ((unsigned long long)tag << 32);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
}
struct Rec16 {   // the fp64 record
  using T = ulonglong2;
  static __device__ __forceinline__ T ld(const T* p) { return ld_tagged(p); }
  static __device__ __forceinline__ bool ok(const T& v, unsigned tag) { return has_tag(v, tag); }
  static __device__ __forceinline__ double val(const T& v) { return tagged_value(v); }
  static __device__ __forceinline__ T zero(unsigned tag) {
    const unsigned long long z = (unsigned long long)tag << 32;
    return make_ulonglong2(z, z);
  }
};
struct Rec8 {    // the fp32 record
  using T = unsigned long long;
  static __device__ __forceinline__ T ld(const T* p) {
    T v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
  }
  static __device__ __forceinline__ bool ok(const T& v, unsigned tag) { return (unsigned)(v >> 32) == tag; }
  static __device__ __forceinline__ double val(const T& v) { return (double)__uint_as_float((unsigned)v); }
  static __device__ __forceinline__ T zero(unsigned tag) { return (unsigned long long)tag << 32; }
};
template <class R, int N>
__device__ __forceinline__ void issue_rec(typename R::T (&v)[N], const typename R::T* src, int64_t stride, int count,
                                          unsigned tag) {
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = q < count ? R::ld(src + q * stride) : R::zero(tag);
}
template <class R, int N>
__device__ __forceinline__ bool repoll_rec(typename R::T (&v)[N], const typename R::T* src, int64_t stride, unsigned tag) {
  bool ready = true;
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (!R::ok(v[q], tag)) { ready = false; v[q] = R::ld(src + q * stride); }
  return ready;
}
template <class R, int N>
__device__ __forceinline__ double sum_rec(const typename R::T (&v)[N]) {   // in q order
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < N; ++q) s += R::val(v[q]);
  return s;
}
#ifndef FPFP_OC_REC32
#define FPFP_OC_REC32 1
#endif
#ifndef FPFP_OC_TOT32   // the fp32 sweeps' tile totals and deltas as 8-byte records too
#define FPFP_OC_TOT32 0
#endif

#ifndef FPFP_OC_POLL_NS
#define FPFP_OC_POLL_NS 0
#endif
__device__ __forceinline__ void poll_backoff() {   // between re-polls of stale records
  if (FPFP_OC_POLL_NS > 0) __nanosleep(FPFP_OC_POLL_NS);
}

// the first `count` records src[q * stride] into v (the rest: a tagged zero, never re-polled)
template <int N>
__device__ __forceinline__ void issue_tagged(ulonglong2 (&v)[N], const ulonglong2* src, int64_t stride, int count,
                                             unsigned tag) {
  const unsigned long long z = (unsigned long long)tag << 32;
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = q < count ? ld_tagged(src + q * stride) : make_ulonglong2(z, z);
}
// re-load the records whose tags are stale; true when none was
template <int N>
__device__ __forceinline__ bool repoll_tagged(ulonglong2 (&v)[N], const ulonglong2* src, int64_t stride, unsigned tag) {
  bool ready = true;
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (!has_tag(v[q], tag)) { ready = false; v[q] = ld_tagged(src + q * stride); }
  return ready;
}
template <int N>
__device__ __forceinline__ double sum_tagged(const ulonglong2 (&v)[N]) {   // in q order
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < N; ++q) s += tagged_value(v[q]);
  return s;
}

template <int NQ>   // column chunks of 32 per lane: TCo <= 32 * NQ
__global__ void __launch_bounds__(kThreads, 1) proj_onchip_kernel(OnchipArgs p) {
  if (*p.done) return;
  cg::grid_group grid = cg::this_grid();
  // Storage and arithmetic. The tile is fp32, Y's storage precision. The sums pass after the GEMM
  // and the launch's first sweep (which cancels the GEMM's large values down to the projection's
  // scale) run in fp64: fp64 correction and sums, one rounding of z to fp32. The
  // later sweeps operate on the projection's own output and run in fp32 (P1, P2, delta), with fp32
  // partial sums over short chains (<= NQ values per lane then 4 lanes per chain for a row; the
  // warp's rows for a column) combined in fp64 — the streaming kernel's precision class.
  // Rows of the shared tile are padded to kLdt = 32 NQ columns: padded entries are 0 and their
  // column correction is huge (1e300 / 3e38), so P2 keeps them at 0 with no bounds test.
  constexpr int kLdt = 32 * NQ;
  extern __shared__ __align__(16) float tile[];   // [TRo][kLdt]
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
      tile[i * kLdt + j] = j < nc ? p.Y[(int64_t)(r0 + i) * p.ldY + c0 + j] : 0.0f;
  for (int j = nc + threadIdx.x; j < kLdt; j += kThreads) sh.uf[j] = 3.0e38f;
  __syncthreads();

  // One fused pass over the tile: the sums of the incoming Y (kSums) or one sweep (P1 then P2;
  // kSweep64 in fp64, kSweep32 in fp32), and the row / column partial sums, the tile total and the
  // tile delta of the resulting values to exchange buffer `buf`. Latency, not bandwidth, bounds this
  // kernel at n ~ 1000, so the element loop carries no cross-lane reduction: warp w
  // walks rows w, w+8, ...; lane l keeps its columns' partial sums in registers and writes its
  // per-row partial to shared memory (rowacc[i][l]); the 32 lane partials of a row and the 8 warp
  // partials of a column are then summed by one thread each, in a fixed order. P2 is a sign test /
  // max with 0; the delta is tracked in fp32: rounding is monotonic, so max_ij fl32(|dz|) =
  // fl32(max_ij |dz|).
  enum { kSums = 0, kSweep64 = 1, kSweep32 = 2 };
  double* rowacc = reinterpret_cast<double*>(tile + (size_t)p.TRo * kLdt);   // [TRo][33] fp64
  float* rowacc_f = reinterpret_cast<float*>(rowacc);                        // [TRo][33] fp32 (same space)
#ifdef FPFP_OC_PROF
  long long pc_rows = 0, pc_cols = 0;
#endif
  ulonglong2* const rowq = reinterpret_cast<ulonglong2*>(p.rowp);   // [2][PC][m] records
  ulonglong2* const colq = reinterpret_cast<ulonglong2*>(p.colp);   // [2][PR][m]
  // the fp32 sweeps' 8-byte records [2][PC][m] / [2][PR][m] live in the first half of the fp64
  // records' storage, inside buffer 0, which only exchange 0 (the sums pass) uses as fp64: exchange
  // x >= 2 can be written only after every CTA has absorbed exchange x - 1 >= 1, so after exchange 0;
  // stale words there carry other tags
  unsigned long long* const rowq8 = reinterpret_cast<unsigned long long*>(p.rowp);
  unsigned long long* const colq8 = reinterpret_cast<unsigned long long*>(p.colp);
  unsigned long long* const totq8 = reinterpret_cast<unsigned long long*>(p.tot);   // (FPFP_OC_TOT32)
  unsigned long long* const dltq8 = reinterpret_cast<unsigned long long*>(p.dlt);
  ulonglong2* const totq = reinterpret_cast<ulonglong2*>(p.tot);    // [2][nb]
  ulonglong2* const dltq = reinterpret_cast<ulonglong2*>(p.dlt);    // [2][nb]
  const unsigned tag0 = p.epoch << 16;                               // tag = tag0 ^ exchange index
  auto pass = [&](int mode, int buf, unsigned tag, double tconst) {
#ifdef FPFP_OC_PROF
    const long long c0_ = clock64();
#endif
    float dmax = 0.0f;
    double tacc = 0.0;   // this lane's share of the tile total (published first, below)
    if (mode == kSweep32) {
      float uf[NQ], cacc[NQ], dq[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) { uf[q] = sh.uf[lane + 32 * q]; cacc[q] = 0.0f; dq[q] = 0.0f; }
      // t_i of the warp's rows: lane k rounds row warp + kWarps k's (fp64 -> fp32 once per row)
      const int myrow = warp + kWarps * lane;
      const float tmine = myrow < nr ? (float)(tconst - sh.r[myrow] * inv_m) : 0.0f;
      float taccf = 0.0f;
      int k = 0;
#pragma unroll kRowUnroll
      for (int i = warp; i < nr; i += kWarps, ++k) {
        const float ti = __shfl_sync(0xffffffffu, tmine, k);
        float* row = &tile[i * kLdt + lane];
        float y[NQ], z[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) y[q] = row[32 * q];
        float racc = 0.0f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          z[q] = fmaxf((y[q] + ti) - uf[q], 0.0f);                 // P1 then P2 (fp32)
          dq[q] = fmaxf(dq[q], fabsf(z[q] - y[q]));
          racc += z[q];
          cacc[q] += z[q];
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) row[32 * q] = z[q];
        rowacc_f[i * 33 + lane] = racc;
        taccf += racc;
      }
      tacc = (double)taccf;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        dmax = fmaxf(dmax, dq[q]);
        sh.colsum.f[warp][lane + 32 * q] = cacc[q];
      }
    } else {
      double cacc[NQ], cj[NQ];
      float dq[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        cacc[q] = 0.0;
        dq[q] = 0.0f;
        const int j = lane + 32 * q;
        cj[q] = j < nc ? sh.c[j] * inv_m : 1e300;
      }
      if (mode == kSweep64) {
#pragma unroll kRowUnroll
        for (int i = warp; i < nr; i += kWarps) {
          const double ti = tconst - sh.r[i] * inv_m;
          float* row = &tile[i * kLdt + lane];
          double y[NQ];
          float z[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) y[q] = (double)row[32 * q];
          double racc = 0.0;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const double v = (y[q] + ti) - cj[q];                  // P1 (fp64)
            z[q] = __double2hiint(v) < 0 ? 0.0f : (float)v;        // P2, one rounding to fp32
            dq[q] = fmaxf(dq[q], (float)fabs((double)z[q] - y[q]));
            racc += (double)z[q];                                  // sums of the stored values
            cacc[q] += (double)z[q];
          }
#pragma unroll
          for (int q = 0; q < NQ; ++q) row[32 * q] = z[q];
          rowacc[i * 33 + lane] = racc;
          tacc += racc;
        }
      } else {
#pragma unroll 2
        for (int i = warp; i < nr; i += kWarps) {
          const float* row = &tile[i * kLdt + lane];
          double racc = 0.0;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const double y = (double)row[32 * q];
            racc += y;
            cacc[q] += y;
          }
          rowacc[i * 33 + lane] = racc;
          tacc += racc;
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        dmax = fmaxf(dmax, dq[q]);
        sh.colsum.d[warp][lane + 32 * q] = cacc[q];
      }
    }
    dmax = warp_max(dmax);
    tacc = warp_sum(tacc);
    if (lane == 0) { sh.dred[warp] = dmax; sh.red[warp] = tacc; }
    __syncthreads();
    // the tile total and delta go out first: every CTA needs all of them, so they are the last
    // records a reader waits for (the last thread rarely has a row or column of its own)
    if (threadIdx.x == kThreads - 1) {
      double t = 0.0;
      float d = 0.0f;
      for (int w = 0; w < kWarps; ++w) { t += sh.red[w]; d = fmaxf(d, sh.dred[w]); }
      if (nb == 1) {
        sh.bc[0] = t;
        sh.bc[1] = (double)d;
      } else {
        if (FPFP_OC_TOT32 && mode == kSweep32) {
          st_tagged32(totq8 + buf * nb + b, (float)t, tag);
          st_tagged32(dltq8 + buf * nb + b, d, tag);
        } else {
          st_tagged(totq + buf * nb + b, t, tag);
          st_tagged(dltq + buf * nb + b, (double)d, tag);
        }
      }
    }
#ifdef FPFP_OC_PROF
    const long long c1_ = clock64();
    pc_rows += c1_ - c0_;
#endif
    // row partials (own rows) and column partials (own columns), fixed order
    for (int t = threadIdx.x; t < nr; t += kThreads) {
      double rs;
      if (mode == kSweep32) {   // 8 fp32 chains of 4 lane partials, combined in fp64
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < 32; l += 4) {
          const float* v = &rowacc_f[t * 33 + l];
          acc += (double)((v[0] + v[1]) + (v[2] + v[3]));
        }
        rs = acc;
      } else {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < 32; l += 4) {
          s0 += rowacc[t * 33 + l]; s1 += rowacc[t * 33 + l + 1];
          s2 += rowacc[t * 33 + l + 2]; s3 += rowacc[t * 33 + l + 3];
        }
        rs = (s0 + s1) + (s2 + s3);
      }
      if (nb == 1) sh.r[t] = rs;   // one tile: the sums stay on chip (the element loop is done)
      else if (FPFP_OC_REC32 && mode == kSweep32)
        st_tagged32(rowq8 + ((int64_t)buf * p.PC + pc) * p.m + r0 + t, (float)rs, tag);
      else st_tagged(rowq + ((int64_t)buf * p.PC + pc) * p.m + r0 + t, rs, tag);
    }
    for (int j = threadIdx.x; j < nc; j += kThreads) {
      double s = 0.0;
      if (mode == kSweep32) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += (double)sh.colsum.f[w][j];
      } else {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += sh.colsum.d[w][j];
      }
      if (nb == 1) { sh.c[j] = s; sh.uf[j] = (float)(s * inv_m); }
      else if (FPFP_OC_REC32 && mode == kSweep32)
        st_tagged32(colq8 + ((int64_t)buf * p.PR + pr) * p.m + c0 + j, (float)s, tag);
      else st_tagged(colq + ((int64_t)buf * p.PR + pr) * p.m + c0 + j, s, tag);
    }
#ifdef FPFP_OC_PROF
    pc_cols += clock64() - c1_;
#endif
    __syncwarp();   // reconverge after the per-thread branches (see the note in absorb)
  };

  // r (own rows), c (own columns), sigma, delta from exchange buffer `buf`, in a fixed order.
  // Every record is loaded before any is consumed (one L2 round trip when the writers are done);
  // a record whose tags are stale is re-polled. Row t's PC partials, column t's PR partials and
  // (one warp) the PR*PC tile totals and deltas; with 512 threads rows and columns are polled by
  // different halves of the block (register budget), with 256 by the same threads.
  constexpr int kMaxTilesPerLane = 5;   // PR * PC <= 160
  constexpr int kMaxP = 12;             // PR, PC <= 12
  constexpr bool kSplit = kThreads >= 512;
  // R: the record type of the row / column partials (Rec16, or Rec8 for the fp32 sweeps)
  auto absorb = [&](auto rec, int buf, unsigned tag, double& sigma, float& delta) {
    using R = decltype(rec);
    using RT = typename R::T;
    const int t = threadIdx.x;
    const RT* rbase = std::is_same<R, Rec8>::value ? reinterpret_cast<const RT*>(rowq8) : reinterpret_cast<const RT*>(rowq);
    const RT* cbase = std::is_same<R, Rec8>::value ? reinterpret_cast<const RT*>(colq8) : reinterpret_cast<const RT*>(colq);
    const RT* rsrc = rbase + (int64_t)buf * p.PC * p.m + r0 + t;
    const RT* csrc = cbase + (int64_t)buf * p.PR * p.m + c0 + (kSplit ? t - kThreads / 2 : t);
    using TR = typename std::conditional<FPFP_OC_TOT32 && std::is_same<R, Rec8>::value, Rec8, Rec16>::type;
    using TT = typename TR::T;
    const TT* tsrc = (std::is_same<TR, Rec8>::value ? reinterpret_cast<const TT*>(totq8)
                                                     : reinterpret_cast<const TT*>(totq)) + buf * nb + lane;
    const TT* dsrc = (std::is_same<TR, Rec8>::value ? reinterpret_cast<const TT*>(dltq8)
                                                     : reinterpret_cast<const TT*>(dltq)) + buf * nb + lane;
    const int tw = kSplit ? kWarps / 2 - 1 : kWarps - 1;   // the warp that sums the tile totals
    if (kSplit && t >= kThreads / 2) {
      RT cv[kMaxP];
      const int nq = t - kThreads / 2 < nc ? p.PR : 0;
      issue_rec<R>(cv, csrc, p.m, nq, tag);
      while (!repoll_rec<R>(cv, csrc, p.m, tag)) poll_backoff();
      __syncwarp();
      if (nq) {
        const double cs = sum_rec<R>(cv);
        sh.c[t - kThreads / 2] = cs;
        sh.uf[t - kThreads / 2] = (float)(cs * inv_m);
      }
    } else {
      RT rv[kMaxP], cv[kSplit ? 1 : kMaxP];
      TT tv[kMaxTilesPerLane], dv[kMaxTilesPerLane];
      const int nr_q = t < nr ? p.PC : 0, nc_q = (!kSplit && t < nc) ? p.PR : 0;
      const int nt_q = warp == tw ? (nb - lane + 31) / 32 : 0;   // tiles lane, lane + 32, ...
      issue_rec<R>(rv, rsrc, p.m, nr_q, tag);
      issue_rec<R>(cv, csrc, p.m, nc_q, tag);
      issue_rec<TR>(tv, tsrc, 32, nt_q, tag);
      issue_rec<TR>(dv, dsrc, 32, nt_q, tag);
      for (;;) {
        bool ready = repoll_rec<R>(rv, rsrc, p.m, tag);
        ready &= repoll_rec<R>(cv, csrc, p.m, tag);
        ready &= repoll_rec<TR>(tv, tsrc, 32, tag);
        ready &= repoll_rec<TR>(dv, dsrc, 32, tag);
        if (ready) break;
        poll_backoff();
      }
      // the lanes of a warp leave the poll loop in different iterations: reconverge them here
      // (with the __syncwarp at the end of pass, which follows thread-dependent branches) or the
      // next element loop can run with its warps split (measured at c2: 5.2 us per sweep with
      // neither, 4.6 with this one only, 3.5 with both)
      __syncwarp();
      if (nr_q) sh.r[t] = sum_rec<R>(rv);
      if (nc_q) {
        const double cs = sum_rec<R>(cv);
        sh.c[t] = cs;
        sh.uf[t] = (float)(cs * inv_m);
      }
      if (warp == tw) {   // (converged: __syncwarp above)
        double sv = sum_rec<TR>(tv);
        float d = 0.0f;
#pragma unroll
        for (int u = 0; u < kMaxTilesPerLane; ++u) d = fmaxf(d, (float)TR::val(dv[u]));
        sv = warp_sum(sv);
        d = warp_max(d);
        if (lane == 0) { sh.bc[0] = sv; sh.bc[1] = (double)d; }
      }
    }
    __syncthreads();
    sigma = sh.bc[0];
    delta = (float)sh.bc[1];
  };

  // a single tile (m <= FPFP_OC_SINGLE_TILE) needs no exchange: its sums are already in shared memory
  auto exchange = [&](int bufx, unsigned tag, double& sigma_, float& delta_, bool rec32) {
    if (nb == 1) {
      __syncthreads();
      sigma_ = sh.bc[0];
      delta_ = (float)sh.bc[1];
      return;
    }
    if (FPFP_OC_REC32 && rec32) absorb(Rec8{}, bufx, tag, sigma_, delta_);
    else absorb(Rec16{}, bufx, tag, sigma_, delta_);
  };
  double sigma;
  float delta;
  pass(kSums, 0, tag0, 0.0);               // exchange 0: the sums of the incoming Y
  exchange(0, tag0, sigma, delta, false);

  int sweeps = 0;
#ifdef FPFP_OC_PROF
  long long pc_abs = 0;
  pc_rows = pc_cols = 0;
#endif
  for (;;) {
    const unsigned x = (unsigned)sweeps + 1;   // exchange index of this sweep (buffer x & 1)
    pass(sweeps == 0 ? kSweep64 : kSweep32, (int)(x & 1), tag0 ^ (x & 0xffffu), (1.0 + sigma * inv_m) * inv_m);
#ifdef FPFP_OC_PROF
    const long long b0_ = clock64();
#endif
    exchange((int)(x & 1), tag0 ^ (x & 0xffffu), sigma, delta, sweeps > 0);
#ifdef FPFP_OC_PROF
    pc_abs += clock64() - b0_;
#endif
    ++sweeps;
    if ((double)delta < p.eps2 || sweeps >= p.max_iter2) break;
  }
#if defined(FPFP_OC_PROF) && !defined(FPFP_OC_PROF_NOPRINT)
  if ((b == 0 || b == nb - 1) && threadIdx.x == 0)
    printf("oc-prof block %d: %d sweeps, clk/sweep: element loop %lld, partials %lld, exchange wait + absorb %lld\n",
           b, sweeps, pc_rows / sweeps, pc_cols / sweeps, pc_abs / sweeps);
#endif

  // write the tile back in fp32 (slack persists across outer iterations, reading A3)
  for (int i = warp; i < nr; i += kWarps)
    for (int j = lane; j < nc; j += 32) p.Y[(int64_t)(r0 + i) * p.ldY + c0 + j] = tile[i * kLdt + j];
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
  return (size_t)TRo * ldt * sizeof(float) + (size_t)TRo * 33 * sizeof(double);   // tile + lane row partials
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
