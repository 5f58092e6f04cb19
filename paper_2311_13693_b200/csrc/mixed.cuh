#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xtsg {

// mode: 0 round_to_half (res unused), 1 fp16_split, 2 fp16_split_stored.
// Throws XTSG_E_HALFRANGE like double_to_half_bits (half.cpp:10-47).
void split_dev(const double* x, int64_t n, int mode, double* half, double* res, cudaStream_t st);
// half_gemm (mixed.cpp:63-76), bit-exact.
void half_gemm_dev(const double* a, int64_t rows, int64_t inner, const double* b, int64_t cols,
                   double* out, cudaStream_t st);
// comp_with(t, u, v, w, &half_gemm) (mixed.cpp:84-86), bit-exact.
void comp_half_dev(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                   const double* v, int64_t m, const double* w, int64_t n, double* y, cudaStream_t st);
// comp_mixed (mixed.cpp:88-98), bit-exact.
void comp_mixed_dev(const double* th, const double* tr, int64_t n1, int64_t n2, int64_t n3,
                    const double* uh, const double* ur, int64_t l, const double* vh, const double* vr,
                    int64_t m, const double* wh, const double* wr, int64_t n, double* y,
                    cudaStream_t st);

}  // namespace xtsg
