// TEST INFRASTRUCTURE ONLY (oracle build). Not part of the product.
//
// Stand-in for the reference's Eigen-backed src/linalg.cpp (Eigen3 is not
// installed in this image). Implements the four entry points declared in
// /root/reference/proj/include/xts/linalg.hpp:8-24 on top of the OpenBLAS
// ILP64 build bundled with numpy (cblas dgemm + LAPACKE), so that the
// reference's own compression/cp_als/alignment/pipeline sources can be
// compiled unchanged and used as the parity oracle.
//
// Behaviour mirrored from the reference (src/linalg.cpp):
//   gemm                 :24-43  plain C = op(A) op(B), shape check -> UsageError
//   pseudo_inverse       :52-61  SVD, sigma <= rcond*sigma_max -> 0
//   leading_left_sv      :63-74  eigenvectors of m m^T, descending order
//   solve_least_squares  :76-92  column-pivoted QR, rank threshold like
//                                Eigen::ColPivHouseholderQR (eps * diagSize
//                                relative to the largest pivot)
// Bit-level Eigen rounding is NOT reproduced (parity unpinned at that layer);
// the reference's own tests pin these at tolerance level only.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "xts/errors.hpp"
#include "xts/linalg.hpp"

extern "C" {
void scipy_cblas_dgemm64_(int layout, int ta, int tb, int64_t m, int64_t n, int64_t k,
                          double alpha, const double* a, int64_t lda, const double* b,
                          int64_t ldb, double beta, double* c, int64_t ldc);
int64_t scipy_LAPACKE_dgesvd64_(int layout, char jobu, char jobvt, int64_t m, int64_t n,
                                double* a, int64_t lda, double* s, double* u, int64_t ldu,
                                double* vt, int64_t ldvt, double* superb);
int64_t scipy_LAPACKE_dsyevd64_(int layout, char jobz, char uplo, int64_t n, double* a,
                                int64_t lda, double* w);
int64_t scipy_LAPACKE_dgeqp364_(int layout, int64_t m, int64_t n, double* a, int64_t lda,
                                int64_t* jpvt, double* tau);
int64_t scipy_LAPACKE_dormqr64_(int layout, char side, char trans, int64_t m, int64_t n,
                                int64_t k, const double* a, int64_t lda, const double* tau,
                                double* c, int64_t ldc);
int64_t scipy_LAPACKE_dtrtrs64_(int layout, char uplo, char trans, char diag, int64_t n,
                                int64_t nrhs, const double* a, int64_t lda, double* b,
                                int64_t ldb);
}

namespace xts {

namespace {
constexpr int kColMajor = 102;
constexpr int kNoTrans = 111;
constexpr int kTrans = 112;
}  // namespace

Matrix gemm(const Matrix& a, const Matrix& b, bool transpose_a, bool transpose_b) {
  const index_t ar = transpose_a ? a.cols : a.rows;
  const index_t ac = transpose_a ? a.rows : a.cols;
  const index_t br = transpose_b ? b.cols : b.rows;
  const index_t bc = transpose_b ? b.rows : b.cols;
  if (ac != br)
    throw UsageError("gemm: inner dimensions differ (" + std::to_string(ac) + " vs " +
                     std::to_string(br) + ")");
  Matrix out(ar, bc);
  if (ar == 0 || bc == 0 || ac == 0) return out;
  scipy_cblas_dgemm64_(kColMajor, transpose_a ? kTrans : kNoTrans,
                       transpose_b ? kTrans : kNoTrans, ar, bc, ac, 1.0, a.values.data(),
                       std::max<index_t>(1, a.rows), b.values.data(),
                       std::max<index_t>(1, b.rows), 0.0, out.values.data(),
                       std::max<index_t>(1, ar));
  return out;
}

Matrix transpose(const Matrix& m) {
  Matrix out(m.cols, m.rows);
  for (index_t j = 0; j < m.cols; ++j)
    for (index_t i = 0; i < m.rows; ++i) out(j, i) = m(i, j);
  return out;
}

Matrix pseudo_inverse(const Matrix& m, double rcond) {
  const index_t r = m.rows, c = m.cols, k = std::min(r, c);
  std::vector<double> a = m.values, s(k), u(r * k), vt(k * c), superb(std::max<index_t>(1, k));
  if (k > 0)
    scipy_LAPACKE_dgesvd64_(kColMajor, 'S', 'S', r, c, a.data(), std::max<index_t>(1, r),
                            s.data(), u.data(), std::max<index_t>(1, r), vt.data(),
                            std::max<index_t>(1, k), superb.data());
  const double cutoff = k > 0 ? rcond * s[0] : 0.0;
  Matrix out(c, r);
  for (index_t q = 0; q < k; ++q) {
    if (!(s[q] > cutoff)) continue;
    const double inv = 1.0 / s[q];
    for (index_t j = 0; j < r; ++j) {
      const double uj = u[j + r * q] * inv;
      for (index_t i = 0; i < c; ++i) out(i, j) += vt[q + k * i] * uj;
    }
  }
  return out;
}

Matrix leading_left_singular_vectors(const Matrix& m, index_t count) {
  if (count < 1 || count > m.rows)
    throw UsageError("leading_left_singular_vectors: count out of range");
  Matrix g = gemm(m, m, false, true);
  std::vector<double> w(m.rows);
  scipy_LAPACKE_dsyevd64_(kColMajor, 'V', 'L', m.rows, g.values.data(), m.rows, w.data());
  Matrix out(m.rows, count);
  for (index_t j = 0; j < count; ++j)
    for (index_t i = 0; i < m.rows; ++i) out(i, j) = g(i, m.rows - 1 - j);
  return out;
}

Matrix solve_least_squares(const Matrix& a, const Matrix& rhs) {
  if (a.rows != rhs.rows) throw UsageError("solve_least_squares: row counts differ");
  if (a.rows < a.cols)
    throw IllPosedError("solve_least_squares: underdetermined system (" +
                            std::to_string(a.rows) + " rows < " + std::to_string(a.cols) +
                            " cols)",
                        std::min(a.rows, a.cols));
  const index_t m = a.rows, n = a.cols, nrhs = rhs.cols;
  std::vector<double> qr = a.values, tau(std::max<index_t>(1, n));
  std::vector<int64_t> jpvt(n, 0);
  scipy_LAPACKE_dgeqp364_(kColMajor, m, n, qr.data(), m, jpvt.data(), tau.data());
  double maxpivot = 0.0;
  for (index_t i = 0; i < n; ++i) maxpivot = std::max(maxpivot, std::fabs(qr[i + m * i]));
  const double thr = maxpivot * std::numeric_limits<double>::epsilon() * static_cast<double>(n);
  index_t rank = 0;
  for (index_t i = 0; i < n; ++i) rank += std::fabs(qr[i + m * i]) > thr;
  if (rank < n)
    throw IllPosedError("solve_least_squares: rank-deficient system (rank " +
                            std::to_string(rank) + " of " + std::to_string(n) + ")",
                        rank);
  std::vector<double> b = rhs.values;
  scipy_LAPACKE_dormqr64_(kColMajor, 'L', 'T', m, nrhs, n, qr.data(), m, tau.data(), b.data(), m);
  scipy_LAPACKE_dtrtrs64_(kColMajor, 'U', 'N', 'N', n, nrhs, qr.data(), m, b.data(), m);
  Matrix out(n, nrhs);
  for (index_t c = 0; c < nrhs; ++c)
    for (index_t i = 0; i < n; ++i) out(jpvt[i] - 1, c) = b[i + m * c];
  return out;
}

}  // namespace xts
