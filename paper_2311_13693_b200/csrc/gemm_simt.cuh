// Batched strided SIMT GEMM (fp64 / fp32) for the compatibility paths:
// the mode products of comp (compression.cpp:202-209), comp_from_factors
// (:215-220), two-stage materialisation (:187-195), CP-ALS sweeps and the
// stacked least-squares updates. Column-major like xts::Matrix
// (tensor.hpp:10-20); deterministic (fixed k order per output element).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xtsg {

template <class T>
struct GemmArgs {
  int64_t m = 0, n = 0, k = 0, batch = 1;
  const T* a = nullptr;
  int64_t lda = 0, stride_a = 0;
  bool trans_a = false;
  const T* b = nullptr;
  int64_t ldb = 0, stride_b = 0;
  bool trans_b = false;
  T* c = nullptr;
  int64_t ldc = 0, stride_c = 0;
  T alpha = T(1), beta = T(0);
  bool lower_only = false;  // skip output tiles strictly above the diagonal (m == n, batch 1)
};

// C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b]
template <class T>
void gemm_simt(const GemmArgs<T>& g, cudaStream_t st);

}  // namespace xtsg
