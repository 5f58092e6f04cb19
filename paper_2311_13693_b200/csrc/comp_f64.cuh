#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xtsg {

// y = beta*y + (t x1 u x2 v x3 w), all device pointers; u is l x n1 with
// leading dimension ldu (a column slice of a wider matrix when ldu == its
// row count and the pointer is offset), likewise v, w.
void comp_f64_dev(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                  int64_t ldu, int64_t l, const double* v, int64_t ldv, int64_t m,
                  const double* w, int64_t ldw, int64_t n, double* y, double beta,
                  cudaStream_t st);

void reconstruct_dev(const double* a, const double* b, const double* c, int64_t ni, int64_t nj,
                     int64_t nk, int64_t rank, double* out, cudaStream_t st);

void comp_from_factors_dev(const double* a, const double* b, const double* c, int64_t ni,
                           int64_t nj, int64_t nk, int64_t rank, const double* u, int64_t l,
                           const double* v, int64_t m, const double* w, int64_t n, double* y,
                           cudaStream_t st);

}  // namespace xtsg
