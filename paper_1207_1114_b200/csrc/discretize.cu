// discretize.cu — greedy discretization (Algorithm 1 line 11).
//
// v1 (this file): the scan is done on the host after one D2H copy of X: sort the n*n' entries by
// (value desc, row asc, col asc) (reading A12) and take (i, j) whenever row i and column j are
// both free, until min(n, n') pairs are taken. The GPU rounds version (mutually-maximal pairs,
// identical result under the strict order) is SURVEY §8(f1) NEXT-1.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fastpfp.h"
#include "common.cuh"

int fpfp_discretize_device(fastpfp_handle* /*h*/, const float* X, int64_t ldX, int n, int np,
                           int32_t* assign, cudaStream_t s, std::string& msg) {
  std::vector<float> hx((size_t)n * np);
  cudaError_t e = cudaMemcpy2DAsync(hx.data(), (size_t)np * sizeof(float), X, ldX * sizeof(float),
                                    (size_t)np * sizeof(float), n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    msg = std::string("discretize copy: ") + cudaGetErrorString(e);
    return FASTPFP_ECUDA;
  }
  const int64_t total = (int64_t)n * np;
  std::vector<int64_t> order(total);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    const float va = hx[a], vb = hx[b];
    if (va != vb) return va > vb;
    return a < b;  // row-major flat index: smaller row, then smaller column
  });
  std::vector<char> row_free(n, 1), col_free(np, 1);
  for (int i = 0; i < n; ++i) assign[i] = -1;
  const int need = std::min(n, np);
  int taken = 0;
  for (int64_t k = 0; k < total && taken < need; ++k) {
    const int i = (int)(order[k] / np), j = (int)(order[k] % np);
    if (row_free[i] && col_free[j]) {
      assign[i] = j;
      row_free[i] = 0;
      col_free[j] = 0;
      ++taken;
    }
  }
  return FASTPFP_OK;
}
