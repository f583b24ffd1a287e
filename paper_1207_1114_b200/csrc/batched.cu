// batched.cu — C-ABI of the batched small-pair path (include/fastpfp.h "Batches of small pairs"):
// validation, device buffers, and launches of small_solve.cu's kernels (one CTA per pair).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/fastpfp.h"
#include "common.cuh"


using namespace fpfp;

struct fastpfp_batched {
  int64_t batch = 0, n = 0, np = 0, d = 0, m = 0;
  int device = 0, num_sms = 0;
  float *A = nullptr, *Ap = nullptr, *B = nullptr, *Bp = nullptr, *K = nullptr;
  float *X = nullptr, *X0 = nullptr, *Y = nullptr;
  int32_t *iters = nullptr, *conv = nullptr, *sweeps = nullptr, *degen = nullptr, *assign = nullptr;
  float* rho = nullptr;
  int* flags = nullptr;
  int8_t* dig = nullptr;   // digit-plane images of A', A, X per pair (int8 path, small_solve_tc.cu)
  int* dexp = nullptr;     // row exponents of A', A per pair
  bool dig_ready = false;
  cudaStream_t stream = nullptr;
  bool own_stream = false, graphs_set = false, x0_custom = false, poisoned = false;
  int rescale = 1;
  int precision = 3;   // 3 = int8 Ozaki tensor-core products (small_solve_tc.cu), 2 = SIMT fp32
  fastpfp_stats stats{};
  std::string err;
};

namespace {

int berr(fastpfp_batched* h, int code, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
    if (code == FASTPFP_ECUDA) h->poisoned = true;
  }
  return code;
}

#define BCK(h, call)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return berr((h), e_ == cudaErrorMemoryAllocation ? FASTPFP_ENOMEM : FASTPFP_ECUDA,     \
                  "%s failed: %s", #call, cudaGetErrorString(e_));                            \
  } while (0)

#define BGUARD(h)                                   \
  do {                                              \
    if (!(h)) return FASTPFP_EINVAL;                \
    if ((h)->poisoned) return FASTPFP_EPOISONED;    \
    BCK((h), cudaSetDevice((h)->device));           \
  } while (0)

template <typename T>
cudaError_t balloc(T*& p, size_t count) {
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T));
}

__global__ void batched_check_kernel(const float* A, int64_t batch, int n, int* flags) {
  const int64_t total = batch * n * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = k / ((int64_t)n * n);
    const int64_t r = k - p * n * n;
    const int i = (int)(r / n), j = (int)(r % n);
    const float a = A[k];
    if (!isfinite(a)) atomicOr(flags, 2);
    if (j > i && a != A[p * n * n + (int64_t)j * n + i]) atomicOr(flags, 1);
  }
}

__global__ void batched_finite_kernel(const float* A, int64_t total, int* flags) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(A[k])) atomicOr(flags, 2);
}

// K[p][i][j] = sum_t B[p][i][t] B'[p][j][t], fp32 with a sequential t loop
__global__ void batched_affinity_kernel(const float* B, const float* Bp, float* K, int64_t batch,
                                        int n, int np, int d) {
  const int64_t total = batch * n * np;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = k / ((int64_t)n * np);
    const int64_t r = k - p * n * np;
    const int i = (int)(r / np), j = (int)(r % np);
    const float* b = B + (p * n + i) * d;
    const float* bp = Bp + (p * np + j) * d;
    float s = 0.f;
    for (int t = 0; t < d; ++t) s = fmaf(b[t], bp[t], s);
    K[k] = s;
  }
}

__global__ void batched_fill_kernel(float* X, int64_t total, float v) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x)
    X[k] = v;
}

int grid_for(int64_t total) { return (int)std::min<int64_t>(8192, std::max<int64_t>(1, (total + 255) / 256)); }

int breset(fastpfp_batched* h) {
  const int64_t xs = h->batch * h->n * h->np;
  if (h->x0_custom) {
    BCK(h, cudaMemcpyAsync(h->X, h->X0, xs * 4, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    batched_fill_kernel<<<grid_for(xs), 256, 0, h->stream>>>(h->X, xs, (float)(1.0 / ((double)h->n * h->np)));
    BCK(h, cudaGetLastError());
  }
  if (h->Y) BCK(h, cudaMemsetAsync(h->Y, 0, h->batch * h->m * h->m * 4, h->stream));
  BCK(h, cudaStreamSynchronize(h->stream));
  return FASTPFP_OK;
}

int bflags(fastpfp_batched* h, const char* what) {
  int f = 0;
  BCK(h, cudaMemcpyAsync(&f, h->flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  BCK(h, cudaStreamSynchronize(h->stream));
  if (f & 2) return berr(h, FASTPFP_ENONFINITE, "%s contains NaN/Inf", what);
  if (f & 1) return berr(h, FASTPFP_ESYM, "%s is not symmetric (P:135-136)", what);
  return FASTPFP_OK;
}

// digit-plane images of the constant graphs for the tensor-core kernel (allocated on first use)
int bdigits(fastpfp_batched* h) {
  if (!h->dig) {
    BCK(h, balloc(h->dig, (size_t)h->batch * small_tc_digit_bytes_per_pair()));
    BCK(h, balloc(h->dexp, (size_t)h->batch * small_tc_exp_ints_per_pair()));
  }
  SmallArgs a{};
  a.batch = (int)h->batch; a.n = (int)h->n; a.np = (int)h->np; a.A = h->A; a.Ap = h->Ap;
  a.dig = h->dig; a.dexp = h->dexp;
  BCK(h, launch_small_digits_prep(a, (int)std::min<int64_t>(h->batch, 8 * h->num_sms), h->stream));
  h->dig_ready = true;
  return FASTPFP_OK;
}

}  // namespace

extern "C" {

void fastpfp_batched_destroy(fastpfp_batched* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : {(void*)h->A, (void*)h->Ap, (void*)h->B, (void*)h->Bp, (void*)h->K, (void*)h->X,
                  (void*)h->X0, (void*)h->Y, (void*)h->iters, (void*)h->conv, (void*)h->sweeps,
                  (void*)h->degen, (void*)h->assign, (void*)h->rho, (void*)h->flags,
                  (void*)h->dig, (void*)h->dexp})
    if (p) cudaFree(p);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

const char* fastpfp_batched_last_error(const fastpfp_batched* h) { return h ? h->err.c_str() : ""; }

int fastpfp_batched_create(int64_t batch, int64_t n, int64_t n_prime, int64_t d,
                           fastpfp_batched** out) {
  if (!out || batch < 1 || n < 1 || n_prime < 1 || n > 128 || n_prime > 128 || d < 0 || d > 4096)
    return FASTPFP_EINVAL;
  *out = nullptr;
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FASTPFP_ENODEV;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return FASTPFP_ENODEV;
  auto* h = new fastpfp_batched();
  h->batch = batch; h->n = n; h->np = n_prime; h->d = d; h->m = std::max(n, n_prime); h->device = dev;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  A(balloc(h->A, batch * n * n)); A(balloc(h->Ap, batch * n_prime * n_prime));
  if (d > 0) { A(balloc(h->B, batch * n * d)); A(balloc(h->Bp, batch * n_prime * d)); A(balloc(h->K, batch * n * n_prime)); }
  A(balloc(h->X, batch * n * n_prime));
  if (n != n_prime) A(balloc(h->Y, batch * h->m * h->m));
  A(balloc(h->iters, batch)); A(balloc(h->conv, batch)); A(balloc(h->sweeps, batch));
  A(balloc(h->degen, batch)); A(balloc(h->assign, batch * n)); A(balloc(h->rho, batch));
  A(balloc(h->flags, 1));
  A(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  if (e != cudaSuccess) {
    cudaGetLastError();
    fastpfp_batched_destroy(h);
    return e == cudaErrorMemoryAllocation ? FASTPFP_ENOMEM : FASTPFP_ECUDA;
  }
  *out = h;
  return FASTPFP_OK;
}

int fastpfp_batched_set_option(fastpfp_batched* h, int key, int64_t value) {
  BGUARD(h);
  if (key == FASTPFP_OPT_STREAM) {
    BCK(h, cudaStreamSynchronize(h->stream));
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->own_stream = value == 0;
    if (value == 0) BCK(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    else h->stream = reinterpret_cast<cudaStream_t>(value);
    return FASTPFP_OK;
  }
  if (key == FASTPFP_OPT_RESCALE) {
    if (value != 0 && value != 1) return FASTPFP_EINVAL;
    h->rescale = (int)value;
    return FASTPFP_OK;
  }
  if (key == FASTPFP_OPT_PRECISION) {
    if (value != 2 && value != 3) return berr(h, FASTPFP_EINVAL, "batched precision: 2 (fp32 SIMT) or 3 (int8 Ozaki)");
    h->precision = (int)value;
    if (value == 3 && h->graphs_set && !h->dig_ready) return bdigits(h);
    return FASTPFP_OK;
  }
  return berr(h, FASTPFP_EINVAL, "option %d not supported by the batched path", key);
}

int fastpfp_batched_set_graphs(fastpfp_batched* h, const float* A, const float* A_prime,
                               const float* B, const float* B_prime, int is_device) {
  BGUARD(h);
  if (!A || !A_prime || (h->d > 0 && (!B || !B_prime))) return berr(h, FASTPFP_EINVAL, "missing input");
  const cudaMemcpyKind kind = is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaStream_t s = h->stream;
  h->graphs_set = false;
  BCK(h, cudaMemcpyAsync(h->A, A, h->batch * h->n * h->n * 4, kind, s));
  BCK(h, cudaMemcpyAsync(h->Ap, A_prime, h->batch * h->np * h->np * 4, kind, s));
  BCK(h, cudaMemsetAsync(h->flags, 0, sizeof(int), s));
  batched_check_kernel<<<grid_for(h->batch * h->n * h->n), 256, 0, s>>>(h->A, h->batch, (int)h->n, h->flags);
  BCK(h, cudaGetLastError());
  int rc = bflags(h, "A");
  if (rc) return rc;
  batched_check_kernel<<<grid_for(h->batch * h->np * h->np), 256, 0, s>>>(h->Ap, h->batch, (int)h->np, h->flags);
  BCK(h, cudaGetLastError());
  rc = bflags(h, "A'");
  if (rc) return rc;
  if (h->d > 0) {
    BCK(h, cudaMemcpyAsync(h->B, B, h->batch * h->n * h->d * 4, kind, s));
    BCK(h, cudaMemcpyAsync(h->Bp, B_prime, h->batch * h->np * h->d * 4, kind, s));
    batched_finite_kernel<<<grid_for(h->batch * h->n * h->d), 256, 0, s>>>(h->B, h->batch * h->n * h->d, h->flags);
    batched_finite_kernel<<<grid_for(h->batch * h->np * h->d), 256, 0, s>>>(h->Bp, h->batch * h->np * h->d, h->flags);
    BCK(h, cudaGetLastError());
    rc = bflags(h, "B/B'");
    if (rc) return rc;
    batched_affinity_kernel<<<grid_for(h->batch * h->n * h->np), 256, 0, s>>>(h->B, h->Bp, h->K, h->batch,
                                                                              (int)h->n, (int)h->np, (int)h->d);
    BCK(h, cudaGetLastError());
  }
  h->dig_ready = false;
  if (h->precision == 3) {
    rc = bdigits(h);
    if (rc) return rc;
  }
  rc = breset(h);
  if (rc) return rc;
  h->graphs_set = true;
  return FASTPFP_OK;
}

int fastpfp_batched_set_x0(fastpfp_batched* h, const float* X0, int is_device) {
  BGUARD(h);
  if (X0) {
    if (!h->X0) BCK(h, balloc(h->X0, h->batch * h->n * h->np));
    BCK(h, cudaMemcpyAsync(h->X0, X0, h->batch * h->n * h->np * 4,
                           is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    BCK(h, cudaMemsetAsync(h->flags, 0, sizeof(int), h->stream));
    batched_finite_kernel<<<grid_for(h->batch * h->n * h->np), 256, 0, h->stream>>>(h->X0, h->batch * h->n * h->np, h->flags);
    BCK(h, cudaGetLastError());
    int rc = bflags(h, "X0");
    if (rc) return rc;
    h->x0_custom = true;
  } else {
    h->x0_custom = false;
  }
  return breset(h);
}

int fastpfp_batched_iterate(fastpfp_batched* h, double alpha, double lambda, double eps1,
                            double eps2, int32_t max_iter1, int32_t max_iter2, float* X_out,
                            int32_t* iterations, int32_t* converged, int32_t* sweeps) {
  BGUARD(h);
  if (!h->graphs_set) return berr(h, FASTPFP_ESTATE, "fastpfp_batched_set_graphs must come first");
  if (!(alpha >= 0.0 && alpha <= 1.0) || !(lambda >= 0.0) || !std::isfinite(lambda) ||
      !(eps1 >= 0.0) || !(eps2 >= 0.0) || max_iter1 < 1 || max_iter2 < 1)
    return berr(h, FASTPFP_EINVAL, "alpha in [0,1], lambda >= 0, eps >= 0, maxIter >= 1");
  SmallArgs a{};
  a.batch = (int)h->batch; a.n = (int)h->n; a.np = (int)h->np; a.m = (int)h->m;
  a.A = h->A; a.Ap = h->Ap; a.K = (h->d > 0 && lambda != 0.0) ? h->K : nullptr;
  a.X = h->X; a.Y = h->Y;
  a.alpha = (float)alpha; a.lam = (float)lambda; a.eps1 = (float)eps1; a.eps2 = (float)eps2;
  a.max_iter1 = max_iter1; a.max_iter2 = max_iter2; a.rescale = h->rescale;
  a.iters = h->iters; a.conv = h->conv; a.sweeps = h->sweeps; a.rho = h->rho; a.degen = h->degen;
  a.dig = h->dig; a.dexp = h->dexp;
  if (h->precision == 3) {   // two pairs per CTA (small_solve_tc.cu)
    const int grid = (int)std::min<int64_t>((h->batch + 1) / 2, h->num_sms);
    BCK(h, launch_small_solve_tc(a, grid, h->stream));
  } else {
    const int grid = (int)std::min<int64_t>(h->batch, h->num_sms);
    BCK(h, launch_small_solve(a, grid, h->stream));
  }
  h->stats.launches += 1;
  cudaStream_t s = h->stream;
  if (iterations) BCK(h, cudaMemcpyAsync(iterations, h->iters, h->batch * 4, cudaMemcpyDeviceToHost, s));
  if (converged) BCK(h, cudaMemcpyAsync(converged, h->conv, h->batch * 4, cudaMemcpyDeviceToHost, s));
  if (sweeps) BCK(h, cudaMemcpyAsync(sweeps, h->sweeps, h->batch * 4, cudaMemcpyDeviceToHost, s));
  if (X_out) BCK(h, cudaMemcpyAsync(X_out, h->X, h->batch * h->n * h->np * 4, cudaMemcpyDeviceToHost, s));
  BCK(h, cudaStreamSynchronize(s));
  return FASTPFP_OK;
}

int fastpfp_batched_copy_x(fastpfp_batched* h, float* dst, int dst_is_device) {
  BGUARD(h);
  if (!dst) return FASTPFP_EINVAL;
  BCK(h, cudaMemcpyAsync(dst, h->X, h->batch * h->n * h->np * 4,
                         dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  BCK(h, cudaStreamSynchronize(h->stream));
  return FASTPFP_OK;
}

int fastpfp_batched_discretize(fastpfp_batched* h, int32_t* assign) {
  BGUARD(h);
  if (!assign) return FASTPFP_EINVAL;
  if (!h->graphs_set) return berr(h, FASTPFP_ESTATE, "fastpfp_batched_set_graphs must come first");
  const int grid = (int)std::min<int64_t>(h->batch, 4 * h->num_sms);
  BCK(h, launch_small_greedy(h->X, (int)h->batch, (int)h->n, (int)h->np, h->assign, grid, h->stream));
  h->stats.launches += 1;
  BCK(h, cudaMemcpyAsync(assign, h->assign, h->batch * h->n * 4, cudaMemcpyDeviceToHost, h->stream));
  BCK(h, cudaStreamSynchronize(h->stream));
  return FASTPFP_OK;
}

int fastpfp_batched_get_stats(fastpfp_batched* h, fastpfp_stats* out) {
  BGUARD(h);
  if (!out) return FASTPFP_EINVAL;
  *out = h->stats;
  return FASTPFP_OK;
}

}  // extern "C"
