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
#include <cstdlib>
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

// ---- normal-equations fast path (large, well-conditioned stacks) ---------

constexpr int CNB = 64;  // Cholesky block

// Factor the nb x nb diagonal block at (j0, j0) of the lower Cholesky in place
// (right-looking, in shared memory) and write its triangular inverse to Linv
// (nb x nb, leading dim CNB). Pivots <= tau flag `fail`.
__global__ void __launch_bounds__(256) potrf_block_kernel(double* G, int64_t n, int64_t j0, int nb, double* Linv,
                                                          int* fail, double tau) {
  extern __shared__ double shm[];
  double* L = shm;                   // CNB x (CNB + 1), row i col j at L[i * (CNB + 1) + j]
  double* V = shm + CNB * (CNB + 1);  // inverse, same layout
  constexpr int LD = CNB + 1;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    L[i * LD + j] = i >= j ? G[(j0 + i) + n * (j0 + j)] : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < nb; ++k) {
    if (threadIdx.x == 0) {
      double d = L[k * LD + k];
      if (!(d > tau)) {
        *fail = 1;
        d = 1.0;
      }
      L[k * LD + k] = sqrt(d);
    }
    __syncthreads();
    const double dk = L[k * LD + k];
    for (int i = k + 1 + threadIdx.x; i < nb; i += blockDim.x) L[i * LD + k] /= dk;
    __syncthreads();
    const int rem = nb - k - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int i = k + 1 + e % rem, j = k + 1 + e / rem;
      if (i >= j) L[i * LD + j] = fma(-L[i * LD + k], L[j * LD + k], L[i * LD + j]);
    }
    __syncthreads();
  }
  // inverse by forward substitution, one column per thread
  for (int c = threadIdx.x; c < nb; c += blockDim.x) {
    for (int i = 0; i < nb; ++i) {
      double acc = i == c ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) acc = fma(-L[i * LD + k], V[k * LD + c], acc);
      V[i * LD + c] = i < c ? 0.0 : acc / L[i * LD + i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    if (i >= j) G[(j0 + i) + n * (j0 + j)] = L[i * LD + j];
    Linv[i + CNB * j] = V[i * LD + j];
  }
}

__global__ void axpy_kernel(double* y, const double* x, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[e] += x[e];
}

void gemm_d(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
            const double* b, int64_t ldb, double beta, double* c, int64_t ldc, cudaStream_t st, bool lower = false) {
  if (m <= 0 || n <= 0) return;
  GemmArgs<double> g;
  g.m = m; g.n = n; g.k = k;
  g.a = a; g.lda = lda; g.trans_a = ta;
  g.b = b; g.ldb = ldb; g.trans_b = tb;
  g.c = c; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta;
  g.lower_only = lower;
  gemm_simt(g, st);
}

// Y (n x r, ld n) <- L^-T L^-1 Y with L the blocked Cholesky factor in G.
void chol_solve(const double* G, int64_t n, const double* Linv, double* Y, int64_t r, double* tmp, cudaStream_t st) {
  const int64_t nblk = ceil_div(n, CNB);
  for (int64_t b = 0; b < nblk; ++b) {  // forward: L z = y
    const int64_t j0 = b * CNB, nb = std::min<int64_t>(CNB, n - j0), n2 = n - j0 - nb;
    gemm_d(false, false, nb, r, nb, 1.0, Linv + b * CNB * CNB, CNB, Y + j0, n, 0.0, tmp, CNB, st);
    XCUDA(cudaMemcpy2DAsync(Y + j0, n * 8, tmp, CNB * 8, nb * 8, r, cudaMemcpyDeviceToDevice, st));
    gemm_d(false, false, n2, r, nb, -1.0, G + (j0 + nb) + n * j0, n, Y + j0, n, 1.0, Y + j0 + nb, n, st);
  }
  for (int64_t b = nblk - 1; b >= 0; --b) {  // backward: L' x = z
    const int64_t j0 = b * CNB, nb = std::min<int64_t>(CNB, n - j0), n2 = n - j0 - nb;
    gemm_d(true, false, nb, r, n2, -1.0, G + (j0 + nb) + n * j0, n, Y + j0 + nb, n, 1.0, Y + j0, n, st);
    gemm_d(true, false, nb, r, nb, 1.0, Linv + b * CNB * CNB, CNB, Y + j0, n, 0.0, tmp, CNB, st);
    XCUDA(cudaMemcpy2DAsync(Y + j0, n * 8, tmp, CNB * 8, nb * 8, r, cudaMemcpyDeviceToDevice, st));
  }
}

}  // namespace

// Least squares through the normal equations A'A x = A'b with a blocked
// Cholesky (DMMA GEMMs for the Gram, the trailing updates and the solves) and
// two steps of iterative refinement on the true residual b - A x. Taken only
// when every pivot of A'A exceeds 1e-6 of its largest diagonal (cond(A) of at
// most ~10^3, far from the QR rank threshold eps * n): then the system has
// full rank in the reference's sense and the refined solution matches the
// QR solution to ~cond * eps. Returns false (nothing written) otherwise.
bool lsq_chol_dev(const double* A, int64_t m, int64_t n, const double* B, int64_t r, double* X, cudaStream_t st) {
  const int64_t nblk = ceil_div(n, CNB);
  DevBuf<double> G(static_cast<size_t>(n * n), st), W(static_cast<size_t>(n * CNB), st),
      Linv(static_cast<size_t>(nblk * CNB * CNB), st), tmp(static_cast<size_t>(CNB * r), st),
      Rm(static_cast<size_t>(m * r), st), dX(static_cast<size_t>(n * r), st), diag(static_cast<size_t>(n), st);
  DevBuf<int> fail(1, st);
  fail.zero();
  gemm_d(true, false, n, n, m, 1.0, A, m, A, m, 0.0, G.ptr, n, st, true);
  diag_kernel<<<static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 1024))), 256, 0, st>>>(
      G.ptr, n, n, diag.ptr);
  XLAUNCH_CHECK();
  std::vector<double> hd(static_cast<size_t>(n));
  XCUDA(cudaMemcpyAsync(hd.data(), diag.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  XCUDA(cudaStreamSynchronize(st));
  double mx = 0.0;
  for (double v : hd) mx = std::max(mx, v);
  if (!(mx > 0.0)) return false;
  const double tau = 1e-6 * mx;
  const size_t smem = sizeof(double) * 2 * CNB * (CNB + 1);
  // per call (the attribute is per device; no unsynchronised static flag)
  XCUDA(cudaFuncSetAttribute(potrf_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t j0 = b * CNB, nb = std::min<int64_t>(CNB, n - j0), n2 = n - j0 - nb;
    potrf_block_kernel<<<1, 256, smem, st>>>(G.ptr, n, j0, static_cast<int>(nb), Linv.ptr + b * CNB * CNB, fail.ptr,
                                             tau);
    XLAUNCH_CHECK();
    if (n2 > 0) {
      // panel L21 = A21 L11^-T, then the trailing update A22 -= L21 L21'
      gemm_d(false, true, n2, nb, nb, 1.0, G.ptr + (j0 + nb) + n * j0, n, Linv.ptr + b * CNB * CNB, CNB, 0.0, W.ptr,
             n2, st);
      XCUDA(cudaMemcpy2DAsync(G.ptr + (j0 + nb) + n * j0, n * 8, W.ptr, n2 * 8, n2 * 8, nb, cudaMemcpyDeviceToDevice,
                              st));
      gemm_d(false, true, n2, n2, nb, -1.0, W.ptr, n2, W.ptr, n2, 1.0, G.ptr + (j0 + nb) * (n + 1), n, st, true);
    }
  }
  int hf = 0;
  XCUDA(cudaMemcpyAsync(&hf, fail.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  XCUDA(cudaStreamSynchronize(st));
  if (hf) return false;
  // x = (A'A)^-1 A'b, then refine twice: x += (A'A)^-1 A'(b - A x)
  gemm_d(true, false, n, r, m, 1.0, A, m, B, m, 0.0, X, n, st);
  chol_solve(G.ptr, n, Linv.ptr, X, r, tmp.ptr, st);
  for (int it = 0; it < 2; ++it) {
    XCUDA(cudaMemcpyAsync(Rm.ptr, B, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, st));
    gemm_d(false, false, m, r, n, -1.0, A, m, X, n, 1.0, Rm.ptr, m, st);
    gemm_d(true, false, n, r, m, 1.0, A, m, Rm.ptr, m, 0.0, dX.ptr, n, st);
    chol_solve(G.ptr, n, Linv.ptr, dX.ptr, r, tmp.ptr, st);
    axpy_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(n * r, 256), 4096)), 256, 0, st>>>(X, dX.ptr, n * r);
    XLAUNCH_CHECK();
  }
  return true;
}

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
    static const bool chol_on = [] {
      const char* e = std::getenv("XTSG_LS_CHOL");
      return !(e && std::atoi(e) == 0);
    }();
    // the normal-equations path replaces ~2*cols sequential QR launches by a
    // few DMMA GEMMs and blocked Cholesky steps; below 32 columns QR is cheap
    if (chol_on && cols >= 32 && m >= cols && lsq_chol_dev(A.ptr, m, cols, B.ptr, r, xo.dev, st)) {
      xo.finish();
      return;
    }
    const int64_t rank = lsq_colpiv_dev(A.ptr, m, cols, B.ptr, r, xo.dev, st);
    if (rank < cols)
      throw Status(XTSG_E_ILLPOSED,
                   "solve_least_squares: rank-deficient system (rank " + std::to_string(rank) + " of " +
                       std::to_string(cols) + ")",
                   rank);
    xo.finish();
  });
}
