// K10 — stacked least squares on the device (fp64, column-pivoted Householder QR).
//
// Reference: solve_stacked_ls (/root/reference/proj/src/alignment.cpp:220-252)
// -> solve_least_squares (linalg.cpp:76-92, Eigen::ColPivHouseholderQR):
// stack [f_1; ...; f_P] = [U_1; ...; U_P] x, throw IllPosedError(rank) when
// the stack is underdetermined or rank-deficient (|R_ii| <= eps * cols *
// max|R_ii|, Eigen's default threshold), else return the LS solution.
//
// Device algorithm (one column per step, all state resident in HBM/L2):
//   pivot kernel  (1 CTA): argmax of the trailing column norms (first index on
//                 ties, like Eigen/LAPACK), column swap, Householder vector of
//                 the pivot column (LAPACK dlarfg conventions)
//   update kernel (1 CTA per trailing column, plus one per right-hand side):
//                 w = v' A[k:, j]; A[k:, j] -= tau * w * v; the exact trailing
//                 norm is recomputed from the updated column (no downdating)
// then a blocked back substitution (diagonal 128x128 solves + SIMT GEMM
// updates) and the inverse column permutation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gemm_simt.cuh"

namespace xtsg {

namespace {

constexpr int NT = 256;

__device__ double bsum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

__global__ void col_norms_kernel(const double* A, int64_t m, int64_t n, double* vn) {
  __shared__ double red[32];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(A[i + m * j], A[i + m * j], acc);
    acc = bsum(acc, red);
    if (threadIdx.x == 0) vn[j] = sqrt(acc);
    __syncthreads();
  }
}

// step k: pivot, swap, Householder of column k. hh[0] = tau.
__global__ void pivot_householder_kernel(double* A, int64_t m, int64_t n, int64_t k, double* vn, int64_t* perm,
                                         double* tau) {
  __shared__ double red[32];
  __shared__ double s_val[NT];
  __shared__ int64_t s_idx[NT];
  // argmax over vn[k:n], lowest index on ties
  double best = -1.0;
  int64_t bi = k;
  for (int64_t j = k + threadIdx.x; j < n; j += blockDim.x)
    if (vn[j] > best) {
      best = vn[j];
      bi = j;
    }
  s_val[threadIdx.x] = best;
  s_idx[threadIdx.x] = bi;
  __syncthreads();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = s_val[threadIdx.x + s];
      const int64_t oi = s_idx[threadIdx.x + s];
      if (ov > s_val[threadIdx.x] || (ov == s_val[threadIdx.x] && oi < s_idx[threadIdx.x])) {
        s_val[threadIdx.x] = ov;
        s_idx[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const int64_t piv = s_idx[0];
  if (piv != k) {
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      const double t = A[i + m * k];
      A[i + m * k] = A[i + m * piv];
      A[i + m * piv] = t;
    }
    if (threadIdx.x == 0) {
      const double t = vn[k];
      vn[k] = vn[piv];
      vn[piv] = t;
      const int64_t p = perm[k];
      perm[k] = perm[piv];
      perm[piv] = p;
    }
  }
  __syncthreads();
  // dlarfg on A[k:, k]
  double xs = 0.0;
  for (int64_t i = k + 1 + threadIdx.x; i < m; i += blockDim.x) xs = fma(A[i + m * k], A[i + m * k], xs);
  xs = bsum(xs, red);
  const double alpha = A[k + m * k];
  const double xnorm = sqrt(xs);
  if (xnorm == 0.0) {
    if (threadIdx.x == 0) *tau = 0.0;
    return;
  }
  const double beta = -copysign(hypot(alpha, xnorm), alpha);
  const double t = (beta - alpha) / beta;
  const double scale = 1.0 / (alpha - beta);
  for (int64_t i = k + 1 + threadIdx.x; i < m; i += blockDim.x) A[i + m * k] *= scale;
  __syncthreads();
  if (threadIdx.x == 0) {
    A[k + m * k] = beta;
    *tau = t;
  }
}

// Apply H_k to trailing columns of A (blocks [0, n-k-1)) and to rhs B (blocks after).
__global__ void apply_householder_kernel(double* A, int64_t m, int64_t n, int64_t k, const double* tau,
                                         double* vn, double* B, int64_t nrhs) {
  __shared__ double red[32];
  const double t = *tau;
  const int64_t ncols = n - k - 1;
  for (int64_t c = blockIdx.x; c < ncols + nrhs; c += gridDim.x) {
    double* col = c < ncols ? A + m * (k + 1 + c) : B + m * (c - ncols);
    if (t != 0.0) {
      double w = 0.0;
      for (int64_t i = k + threadIdx.x; i < m; i += blockDim.x) {
        const double vi = i == k ? 1.0 : A[i + m * k];
        w = fma(vi, col[i], w);
      }
      w = bsum(w, red) * t;
      for (int64_t i = k + threadIdx.x; i < m; i += blockDim.x) {
        const double vi = i == k ? 1.0 : A[i + m * k];
        col[i] = fma(-w, vi, col[i]);
      }
      __syncthreads();
    }
    if (c < ncols) {
      double acc = 0.0;
      for (int64_t i = k + 1 + threadIdx.x; i < m; i += blockDim.x) acc = fma(col[i], col[i], acc);
      acc = bsum(acc, red);
      if (threadIdx.x == 0) vn[k + 1 + c] = sqrt(acc);
    }
    __syncthreads();
  }
}

// Solve the upper-triangular diagonal block R[b0:b1, b0:b1] x = Y[b0:b1, :] in place.
__global__ void trsm_diag_kernel(const double* R, int64_t m, int64_t b0, int64_t b1, double* Y, int64_t ldy,
                                 int64_t nrhs) {
  for (int64_t c = blockIdx.x; c < nrhs; c += gridDim.x) {
    double* y = Y + ldy * c;
    for (int64_t i = b1 - 1; i >= b0; --i) {
      __syncthreads();
      if (threadIdx.x == 0) y[i] /= R[i + m * i];
      __syncthreads();
      const double xi = y[i];
      for (int64_t r = b0 + threadIdx.x; r < i; r += blockDim.x) y[r] = fma(-R[r + m * i], xi, y[r]);
    }
    __syncthreads();
  }
}

__global__ void unpermute_kernel(const double* Y, int64_t ldy, int64_t n, int64_t nrhs, const int64_t* perm,
                                 double* X) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * nrhs;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, c = e / n;
    X[perm[i] + n * c] = Y[i + ldy * c];
  }
}

__global__ void diag_kernel(const double* A, int64_t m, int64_t n, double* d) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = fabs(A[i + m * i]);
}

__global__ void stack_kernel(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ld, int64_t row0) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    dst[row0 + i + ld * j] = src[e];
  }
}

}  // namespace

// Column-pivoted QR least squares of the device system A (m x n) X = B (m x r).
// Returns the numerical rank; X (n x r) is written only when rank == n.
int64_t lsq_colpiv_dev(double* A, int64_t m, int64_t n, double* B, int64_t r, double* X, cudaStream_t st) {
  DevBuf<double> vn(static_cast<size_t>(n), st), tau(1, st), diag(static_cast<size_t>(n), st);
  std::vector<int64_t> hperm(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) hperm[static_cast<size_t>(i)] = i;
  DevBuf<int64_t> perm(static_cast<size_t>(n), st);
  XCUDA(cudaMemcpyAsync(perm.ptr, hperm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  col_norms_kernel<<<static_cast<int>(std::min<int64_t>(n, 4096)), NT, 0, st>>>(A, m, n, vn.ptr);
  XLAUNCH_CHECK();
  const int64_t steps = std::min(m, n);
  const int blocks_cap = 148 * 8;
  for (int64_t k = 0; k < steps; ++k) {
    pivot_householder_kernel<<<1, NT, 0, st>>>(A, m, n, k, vn.ptr, perm.ptr, tau.ptr);
    XLAUNCH_CHECK();
    const int64_t work = n - k - 1 + r;
    if (work > 0) {
      apply_householder_kernel<<<static_cast<int>(std::min<int64_t>(work, blocks_cap)), NT, 0, st>>>(
          A, m, n, k, tau.ptr, vn.ptr, B, r);
      XLAUNCH_CHECK();
    }
  }
  diag_kernel<<<static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 1024))), 256, 0, st>>>(
      A, m, n, diag.ptr);
  XLAUNCH_CHECK();
  std::vector<double> hd(static_cast<size_t>(n));
  XCUDA(cudaMemcpyAsync(hd.data(), diag.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  XCUDA(cudaStreamSynchronize(st));
  double mx = 0.0;
  for (double v : hd) mx = std::max(mx, v);
  const double thr = mx * DBL_EPSILON * static_cast<double>(n);
  int64_t rank = 0;
  for (double v : hd) rank += v > thr;
  if (rank < n) return rank;
  // back substitution on (Q'B)[0:n], 128-row diagonal blocks + GEMM updates
  constexpr int64_t TB = 128;
  for (int64_t b1 = n; b1 > 0; b1 -= TB) {
    const int64_t b0 = std::max<int64_t>(0, b1 - TB);
    trsm_diag_kernel<<<static_cast<int>(std::min<int64_t>(r, 1024)), NT, 0, st>>>(A, m, b0, b1, B, m, r);
    XLAUNCH_CHECK();
    if (b0 > 0) {
      GemmArgs<double> g;  // B[0:b0, :] -= R[0:b0, b0:b1] * B[b0:b1, :]
      g.m = b0; g.n = r; g.k = b1 - b0;
      g.a = A + m * b0; g.lda = m;
      g.b = B + b0; g.ldb = m;
      g.c = B; g.ldc = m;
      g.alpha = -1.0; g.beta = 1.0;
      gemm_simt(g, st);
    }
  }
  unpermute_kernel<<<static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n * r, 256), 4096))), 256, 0,
                     st>>>(B, m, n, r, perm.ptr, X);
  XLAUNCH_CHECK();
  return rank;
}

}  // namespace xtsg

using namespace xtsg;

extern "C" int32_t xtsg_solve_stacked_ls(int64_t count, const int64_t* rows, int64_t r, int64_t cols,
                                         const double* f, const double* u, double* x) {
  return guard([&] {
    // alignment.cpp:222-237
    if (count < 1) usage("solve_stacked_ls: factor/compressor counts differ");
    int64_t m = 0;
    for (int64_t p = 0; p < count; ++p) {
      if (rows[p] < 0) usage("solve_stacked_ls: inconsistent block shapes");
      m += rows[p];
    }
    if (m < cols)
      throw Status(XTSG_E_ILLPOSED,
                   "solve_stacked_ls: stacked system is underdetermined (" + std::to_string(m) + " rows < " +
                       std::to_string(cols) + " unknowns)",
                   m);
    require_device();
    cudaStream_t st = thread_stream();
    // blocks arrive back to back (f_p: rows[p] x r, u_p: rows[p] x cols); stack them
    InView<double> fin(f, static_cast<size_t>(m * r), st), uin(u, static_cast<size_t>(m * cols), st);
    DevBuf<double> A(static_cast<size_t>(m * cols), st), B(static_cast<size_t>(m * r), st);
    int64_t fo = 0, uo = 0, row0 = 0;
    for (int64_t p = 0; p < count; ++p) {
      const int64_t rp = rows[p];
      if (rp > 0) {
        stack_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(rp * cols, 256), 4096)), 256, 0, st>>>(
            uin.dev + uo, rp, cols, A.ptr, m, row0);
        XLAUNCH_CHECK();
        stack_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(rp * r, 256), 4096)), 256, 0, st>>>(
            fin.dev + fo, rp, r, B.ptr, m, row0);
        XLAUNCH_CHECK();
      }
      fo += rp * r;
      uo += rp * cols;
      row0 += rp;
    }
    OutView<double> xo(x, static_cast<size_t>(cols * r), st);
    const int64_t rank = lsq_colpiv_dev(A.ptr, m, cols, B.ptr, r, xo.dev, st);
    if (rank < cols)
      throw Status(XTSG_E_ILLPOSED,
                   "solve_least_squares: rank-deficient system (rank " + std::to_string(rank) + " of " +
                       std::to_string(cols) + ")",
                   rank);
    xo.finish();
  });
}
