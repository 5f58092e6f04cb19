// Dense linear-algebra entry points of the C ABI (the reference's linalg.hpp
// surface, /root/reference/proj/include/xts/linalg.hpp:8-24, which Eigen backs
// there) plus greedy sparse recovery (omp_recover, alignment.cpp:306-419).
//
//   gemm                          -> batched SIMT DFMA GEMM (gemm_simt.cu)
//   pseudo_inverse                -> Jacobi eigendecomposition of M'M on the device,
//                                    pinv = V diag(1/sigma) V' M' with sigma > rcond*sigma_max
//   leading_left_singular_vectors -> Jacobi eigendecomposition of M M' (descending)
//   solve_least_squares           -> column-pivoted Householder QR (lsq.cu)
//   omp_recover                   -> one CTA per measured column: correlation
//                                    scan, Cholesky-updated active set, residual
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gemm_simt.cuh"

namespace xtsg {
int64_t lsq_colpiv_dev(double* A, int64_t m, int64_t n, double* B, int64_t r, double* X, cudaStream_t st);

namespace {

constexpr int NT = 256;

__device__ double bsum2(double v, double* red) {
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

// Cyclic parallel-ordered Jacobi on a symmetric n x n matrix in global memory
// (one CTA). On return h's diagonal holds eigenvalues, v the eigenvectors.
__global__ void sym_eig_kernel(double* h, double* v, int n, double* scratch) {
  __shared__ double red[32];
  double* cs = scratch;
  double* sn = scratch + n / 2 + 2;
  int* pp = reinterpret_cast<int*>(scratch + 2 * (n / 2 + 2));
  int* qq = pp + n / 2 + 2;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) v[e] = (e % n) == (e / n) ? 1.0 : 0.0;
  __syncthreads();
  if (n < 2) return;
  const int m = n + (n & 1);
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const double x = h[e];
      tot += x * x;
      if ((e % n) != (e / n)) off += x * x;
    }
    off = bsum2(off, red);
    tot = bsum2(tot, red);
    if (off <= 1e-28 * tot || off == 0.0) break;
    for (int step = 0; step < m - 1; ++step) {
      for (int k = threadIdx.x; k < m / 2; k += blockDim.x) {
        auto who = [&](int i) { return i == 0 ? 0 : 1 + (i - 1 + step) % (m - 1); };
        int p = who(k), q = who(m - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        pp[k] = p;
        qq[k] = q;
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = h[p + n * q];
          if (apq != 0.0) {
            const double tau = (h[q + n * q] - h[p + n * p]) / (2.0 * apq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < (m / 2) * n; e += blockDim.x) {
        const int k = e / n, i = e % n, p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double hp = h[i + n * p], hq = h[i + n * q];
        h[i + n * p] = c * hp - s * hq;
        h[i + n * q] = s * hp + c * hq;
        const double vp = v[i + n * p], vq = v[i + n * q];
        v[i + n * p] = c * vp - s * vq;
        v[i + n * q] = s * vp + c * vq;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < (m / 2) * n; e += blockDim.x) {
        const int k = e / n, j = e % n, p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double hp = h[p + n * j], hq = h[q + n * j];
        h[p + n * j] = c * hp - s * hq;
        h[q + n * j] = s * hp + c * hq;
      }
      __syncthreads();
    }
  }
}

// eigenvalues (diag of h) -> descending order index list
void eig_sym_dev(double* h, double* v, int64_t n, std::vector<double>& evals, std::vector<int64_t>& order,
                 cudaStream_t st) {
  DevBuf<double> scratch(static_cast<size_t>(4 * (n / 2 + 2) + 8), st);
  sym_eig_kernel<<<1, NT, 0, st>>>(h, v, static_cast<int>(n), scratch.ptr);
  XLAUNCH_CHECK();
  std::vector<double> hh(static_cast<size_t>(n * n));
  XCUDA(cudaMemcpyAsync(hh.data(), h, sizeof(double) * n * n, cudaMemcpyDeviceToHost, st));
  XCUDA(cudaStreamSynchronize(st));
  evals.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) evals[static_cast<size_t>(i)] = hh[static_cast<size_t>(i + n * i)];
  order.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return evals[static_cast<size_t>(a)] > evals[static_cast<size_t>(b)];
  });
}

// ---- OMP (alignment.cpp:306-419): one CTA per measured column -------------
__global__ void omp_kernel(const double* __restrict__ y_all, const double* __restrict__ D, int64_t rows,
                           int64_t atoms, int sparsity, double tol, const double* __restrict__ atom_norm,
                           double* out, int64_t ldo, double* ws_all, int64_t ws_stride) {
  __shared__ double red[32];
  __shared__ double s_best[NT];
  __shared__ int64_t s_idx[NT];
  const int64_t col = blockIdx.x;
  const double* y = y_all + rows * col;
  double* ws = ws_all + ws_stride * col;
  double* res = ws;                              // rows
  double* chol = res + rows;                     // sparsity*(sparsity+1)/2
  double* rhs = chol + sparsity * (sparsity + 1) / 2;
  double* coef = rhs + sparsity;
  double* g = coef + sparsity;
  double* wv = g + sparsity;
  int64_t* active = reinterpret_cast<int64_t*>(wv + sparsity);
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) res[i] = y[i];
  __syncthreads();
  int na = 0;
  while (na < sparsity) {
    double rn = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) rn = fma(res[i], res[i], rn);
    rn = bsum2(rn, red);
    if (sqrt(rn) <= tol) break;
    // best atom by |d'r| / ||d|| (first index on ties), skipping active atoms
    double best = 0.0;
    int64_t bi = -1;
    for (int64_t j = threadIdx.x; j < atoms; j += blockDim.x) {
      bool is_act = false;
      for (int a = 0; a < na; ++a) is_act |= active[a] == j;
      if (is_act) continue;
      double dot = 0.0;
      for (int64_t i = 0; i < rows; ++i) dot = fma(D[i + rows * j], res[i], dot);
      const double corr = fabs(dot) / atom_norm[j];
      if (corr > best) {
        best = corr;
        bi = j;
      }
    }
    s_best[threadIdx.x] = best;
    s_idx[threadIdx.x] = bi;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        const double ov = s_best[threadIdx.x + s];
        const int64_t oi = s_idx[threadIdx.x + s];
        if (ov > s_best[threadIdx.x] ||
            (ov == s_best[threadIdx.x] && oi >= 0 && (s_idx[threadIdx.x] < 0 || oi < s_idx[threadIdx.x]))) {
          s_best[threadIdx.x] = ov;
          s_idx[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    const int64_t sel = s_idx[0];
    const double sel_corr = s_best[0];
    __syncthreads();
    if (sel < 0 || sel_corr == 0.0) break;
    // grow the Cholesky factor of the active Gram
    for (int a = 0; a < na; ++a) {
      double dot = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) dot = fma(D[i + rows * active[a]], D[i + rows * sel], dot);
      dot = bsum2(dot, red);
      if (threadIdx.x == 0) g[a] = dot;
    }
    double d2 = 0.0, yd = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      d2 = fma(D[i + rows * sel], D[i + rows * sel], d2);
      yd = fma(D[i + rows * sel], y[i], yd);
    }
    d2 = bsum2(d2, red);
    yd = bsum2(yd, red);
    __shared__ int stop;
    if (threadIdx.x == 0) {
      for (int i = 0; i < na; ++i) {
        double s = g[i];
        for (int j = 0; j < i; ++j) s -= chol[i * (i + 1) / 2 + j] * wv[j];
        wv[i] = s / chol[i * (i + 1) / 2 + i];
      }
      double diag2 = d2;
      for (int i = 0; i < na; ++i) diag2 -= wv[i] * wv[i];
      stop = diag2 <= 1e-28;
      if (!stop) {
        for (int i = 0; i < na; ++i) chol[na * (na + 1) / 2 + i] = wv[i];
        chol[na * (na + 1) / 2 + na] = sqrt(diag2);
        active[na] = sel;
        rhs[na] = yd;
        const int n = na + 1;
        // (L L') coef = rhs
        for (int i = 0; i < n; ++i) {
          double s = rhs[i];
          for (int j = 0; j < i; ++j) s -= chol[i * (i + 1) / 2 + j] * wv[j];
          wv[i] = s / chol[i * (i + 1) / 2 + i];
        }
        for (int ii = n - 1; ii >= 0; --ii) {
          double s = wv[ii];
          for (int j = ii + 1; j < n; ++j) s -= chol[j * (j + 1) / 2 + ii] * coef[j];
          coef[ii] = s / chol[ii * (ii + 1) / 2 + ii];
        }
      }
    }
    __syncthreads();
    if (stop) break;
    ++na;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      double fit = 0.0;
      for (int a = 0; a < na; ++a) fit = fma(D[i + rows * active[a]], coef[a], fit);
      res[i] = y[i] - fit;
    }
    __syncthreads();
  }
  for (int a = threadIdx.x; a < na; a += blockDim.x) out[active[a] + ldo * col] = coef[a];
}


// ---- OMP for large dictionaries: the atom search spread over the GPU ------
// The per-column CTA above scans every atom with one CTA per measured column
// (10^6 atoms x 512 rows: seconds). Here every iteration is three launches
// for all columns at once: (1) CTAs over atom chunks, one warp per atom,
// lanes over rows, dot products against all (up to OMP_CB) residuals held in
// shared memory -> per-CTA best (|d'r| / ||d||, lowest index on ties, active
// atoms skipped through a byte mask); (2) per-column reduction of the CTA
// candidates in CTA order (same tie rule: the reference's first maximum);
// (3) one CTA per column grows the Cholesky factor, re-solves and recomputes
// the residual exactly like omp_kernel. Finished columns are skipped.
constexpr int OMP_CB = 16;  // columns per search pass (residuals in shared memory)

__global__ void omp_search_kernel(const double* __restrict__ D, int64_t rows, int64_t atoms,
                                  const double* __restrict__ atom_norm, const double* __restrict__ res_all,
                                  const uint8_t* __restrict__ active_mask, const int* __restrict__ done,
                                  int64_t c0, int nc, double* __restrict__ cand_v, int64_t* __restrict__ cand_i,
                                  int64_t ncols) {
  extern __shared__ double sres[];  // nc x rows
  __shared__ double wbest[NT / 32][OMP_CB];
  __shared__ int64_t wbi[NT / 32][OMP_CB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < nc * rows; e += blockDim.x) sres[e] = res_all[(c0 + e / rows) * rows + e % rows];
  __syncthreads();
  double best[OMP_CB];
  int64_t bi[OMP_CB];
#pragma unroll
  for (int c = 0; c < OMP_CB; ++c) {
    best[c] = 0.0;
    bi[c] = -1;
  }
  const int64_t per = (atoms + gridDim.x - 1) / gridDim.x;
  const int64_t a0 = blockIdx.x * per, a1 = min(atoms, a0 + per);
  for (int64_t j = a0 + warp; j < a1; j += nw) {
    const double* d = D + rows * j;
    double dot[OMP_CB];
#pragma unroll
    for (int c = 0; c < OMP_CB; ++c) dot[c] = 0.0;
    for (int64_t i = lane; i < rows; i += 32) {
      const double dv = d[i];
#pragma unroll
      for (int c = 0; c < OMP_CB; ++c)
        if (c < nc) dot[c] = fma(dv, sres[c * rows + i], dot[c]);
    }
#pragma unroll
    for (int c = 0; c < OMP_CB; ++c) {
      if (c >= nc) continue;
      double v = dot[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int64_t col = c0 + c;
      if (lane == 0 && !done[col] && !active_mask[j * ncols + col]) {
        const double corr = fabs(v) / atom_norm[j];
        if (corr > best[c]) {  // ascending j within the warp: first maximum kept
          best[c] = corr;
          bi[c] = j;
        }
      }
    }
  }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < OMP_CB; ++c) {
      wbest[warp][c] = best[c];
      wbi[warp][c] = bi[c];
    }
  __syncthreads();
  if (threadIdx.x < nc) {
    const int c = threadIdx.x;
    double bv = 0.0;
    int64_t bj = -1;
    for (int w = 0; w < nw; ++w) {
      const double v = wbest[w][c];
      const int64_t i = wbi[w][c];
      if (i >= 0 && (v > bv || (v == bv && (bj < 0 || i < bj)))) {
        bv = v;
        bj = i;
      }
    }
    cand_v[(c0 + c) * gridDim.x + blockIdx.x] = bv;
    cand_i[(c0 + c) * gridDim.x + blockIdx.x] = bj;
  }
}

__global__ void omp_update_kernel(const double* __restrict__ y_all, const double* __restrict__ D, int64_t rows,
                                  int64_t atoms, int sparsity, double tol, const double* __restrict__ cand_v,
                                  const int64_t* __restrict__ cand_i, int ncand, uint8_t* __restrict__ active_mask,
                                  int64_t ncols, int* __restrict__ done, int* __restrict__ na_all,
                                  double* __restrict__ res_all, double* ws_all, int64_t ws_stride) {
  __shared__ double red[32];
  __shared__ int stop;
  __shared__ int64_t s_sel;
  __shared__ double s_corr;
  const int64_t col = blockIdx.x;
  if (done[col]) return;
  const double* y = y_all + rows * col;
  double* res = res_all + rows * col;
  double* ws = ws_all + ws_stride * col;
  double* chol = ws;
  double* rhs = chol + sparsity * (sparsity + 1) / 2;
  double* coef = rhs + sparsity;
  double* g = coef + sparsity;
  double* wv = g + sparsity;
  int64_t* active = reinterpret_cast<int64_t*>(wv + sparsity);
  const int na = na_all[col];
  if (threadIdx.x == 0) {
    double bv = 0.0;
    int64_t bj = -1;
    for (int q = 0; q < ncand; ++q) {  // CTA order = ascending atom chunks
      const double v = cand_v[col * ncand + q];
      const int64_t i = cand_i[col * ncand + q];
      if (i >= 0 && (v > bv || (v == bv && (bj < 0 || i < bj)))) {
        bv = v;
        bj = i;
      }
    }
    s_sel = bj;
    s_corr = bv;
  }
  __syncthreads();
  const int64_t sel = s_sel;
  if (sel < 0 || s_corr == 0.0) {
    if (threadIdx.x == 0) done[col] = 1;
    return;
  }
  for (int a = 0; a < na; ++a) {
    double dot = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) dot = fma(D[i + rows * active[a]], D[i + rows * sel], dot);
    dot = bsum2(dot, red);
    if (threadIdx.x == 0) g[a] = dot;
  }
  double d2 = 0.0, yd = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    d2 = fma(D[i + rows * sel], D[i + rows * sel], d2);
    yd = fma(D[i + rows * sel], y[i], yd);
  }
  d2 = bsum2(d2, red);
  yd = bsum2(yd, red);
  if (threadIdx.x == 0) {
    for (int i = 0; i < na; ++i) {
      double sacc = g[i];
      for (int j = 0; j < i; ++j) sacc -= chol[i * (i + 1) / 2 + j] * wv[j];
      wv[i] = sacc / chol[i * (i + 1) / 2 + i];
    }
    double diag2 = d2;
    for (int i = 0; i < na; ++i) diag2 -= wv[i] * wv[i];
    stop = diag2 <= 1e-28;
    if (!stop) {
      for (int i = 0; i < na; ++i) chol[na * (na + 1) / 2 + i] = wv[i];
      chol[na * (na + 1) / 2 + na] = sqrt(diag2);
      active[na] = sel;
      rhs[na] = yd;
      const int n = na + 1;
      for (int i = 0; i < n; ++i) {
        double sacc = rhs[i];
        for (int j = 0; j < i; ++j) sacc -= chol[i * (i + 1) / 2 + j] * wv[j];
        wv[i] = sacc / chol[i * (i + 1) / 2 + i];
      }
      for (int ii = n - 1; ii >= 0; --ii) {
        double sacc = wv[ii];
        for (int j = ii + 1; j < n; ++j) sacc -= chol[j * (j + 1) / 2 + ii] * coef[j];
        coef[ii] = sacc / chol[ii * (ii + 1) / 2 + ii];
      }
      active_mask[sel * ncols + col] = 1;
      na_all[col] = n;
    } else {
      done[col] = 1;
    }
  }
  __syncthreads();
  if (stop) return;
  const int n = na + 1;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    double fit = 0.0;
    for (int a = 0; a < n; ++a) fit = fma(D[i + rows * active[a]], coef[a], fit);
    res[i] = y[i] - fit;
  }
  // the next iteration's residual-norm test (alignment.cpp:343-345)
  double rn = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) rn = fma(res[i], res[i], rn);
  rn = bsum2(rn, red);
  if (threadIdx.x == 0 && (sqrt(rn) <= tol || n >= sparsity)) done[col] = 1;
}

__global__ void omp_init_kernel(const double* __restrict__ y_all, int64_t rows, int64_t ncols, double tol,
                                double* __restrict__ res_all, int* __restrict__ done, int* __restrict__ na_all) {
  __shared__ double red[32];
  const int64_t col = blockIdx.x;
  double rn = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double v = y_all[rows * col + i];
    res_all[rows * col + i] = v;
    rn = fma(v, v, rn);
  }
  rn = bsum2(rn, red);
  if (threadIdx.x == 0) {
    done[col] = sqrt(rn) <= tol ? 1 : 0;
    na_all[col] = 0;
  }
}

__global__ void omp_scatter_kernel(const double* __restrict__ ws_all, int64_t ws_stride, int sparsity,
                                   const int* __restrict__ na_all, double* __restrict__ out, int64_t ldo) {
  const int64_t col = blockIdx.x;
  const double* ws = ws_all + ws_stride * col;
  const double* coef = ws + sparsity * (sparsity + 1) / 2 + sparsity;
  const int64_t* active = reinterpret_cast<const int64_t*>(coef + 3 * sparsity);
  for (int a = threadIdx.x; a < na_all[col]; a += blockDim.x) out[active[a] + ldo * col] = coef[a];
}

__global__ void scale_cols_kernel(const double* v, int64_t rows, int64_t cols, const double* s, double* out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = v[e] * s[e / rows];
}

__global__ void atom_norm_kernel(const double* D, int64_t rows, int64_t atoms, double* nrm, int* zero_col) {
  __shared__ double red[32];
  for (int64_t j = blockIdx.x; j < atoms; j += gridDim.x) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) acc = fma(D[i + rows * j], D[i + rows * j], acc);
    acc = bsum2(acc, red);
    if (threadIdx.x == 0) {
      nrm[j] = sqrt(acc);
      if (acc == 0.0) atomicMin(zero_col, static_cast<int>(j));
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace xtsg

using namespace xtsg;

extern "C" {

// C = op(A) op(B), column-major fp64 (linalg.cpp:24-43)
int32_t xtsg_gemm(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                  const double* b, int64_t ldb, double* c, int64_t ldc) {
  return guard([&] {
    if (m < 0 || n < 0 || k < 0) usage("gemm: negative dimension");
    if (m == 0 || n == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    const int64_t asz = trans_a ? lda * m : lda * k, bsz = trans_b ? ldb * k : ldb * n;
    InView<double> aa(a, static_cast<size_t>(k ? asz : 0), st), bb(b, static_cast<size_t>(k ? bsz : 0), st);
    OutView<double> cc(c, static_cast<size_t>(ldc * n), st);
    if (k == 0) {
      XCUDA(cudaMemsetAsync(cc.dev, 0, sizeof(double) * ldc * n, st));
    } else {
      GemmArgs<double> g;
      g.m = m; g.n = n; g.k = k;
      g.a = aa.dev; g.lda = lda; g.trans_a = trans_a != 0;
      g.b = bb.dev; g.ldb = ldb; g.trans_b = trans_b != 0;
      g.c = cc.dev; g.ldc = ldc;
      gemm_simt(g, st);
    }
    cc.finish();
  });
}

// leading_left_singular_vectors (linalg.cpp:63-74)
int32_t xtsg_leading_left_singular_vectors(const double* m, int64_t rows, int64_t cols, int64_t count,
                                           double* out) {
  return guard([&] {
    if (count < 1 || count > rows) usage("leading_left_singular_vectors: count out of range");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> mm(m, static_cast<size_t>(rows * cols), st);
    DevBuf<double> g(static_cast<size_t>(rows * rows), st), v(static_cast<size_t>(rows * rows), st);
    GemmArgs<double> ga;
    ga.m = rows; ga.n = rows; ga.k = cols;
    ga.a = mm.dev; ga.lda = rows;
    ga.b = mm.dev; ga.ldb = rows; ga.trans_b = true;
    ga.c = g.ptr; ga.ldc = rows;
    if (cols > 0) gemm_simt(ga, st);
    else g.zero();
    std::vector<double> ev;
    std::vector<int64_t> order;
    eig_sym_dev(g.ptr, v.ptr, rows, ev, order, st);
    OutView<double> o(out, static_cast<size_t>(rows * count), st);
    for (int64_t j = 0; j < count; ++j)  // descending eigenvalue order (linalg.cpp:71)
      XCUDA(cudaMemcpyAsync(o.dev + rows * j, v.ptr + rows * order[static_cast<size_t>(j)], sizeof(double) * rows,
                            cudaMemcpyDeviceToDevice, st));
    o.finish();
  });
}

// pseudo_inverse (linalg.cpp:52-61): out (cols x rows)
int32_t xtsg_pseudo_inverse(const double* m, int64_t rows, int64_t cols, double rcond, double* out) {
  return guard([&] {
    require_device();
    cudaStream_t st = thread_stream();
    if (rows == 0 || cols == 0) {
      return;
    }
    InView<double> mm(m, static_cast<size_t>(rows * cols), st);
    DevBuf<double> g(static_cast<size_t>(cols * cols), st), v(static_cast<size_t>(cols * cols), st);
    GemmArgs<double> ga;  // M'M
    ga.m = cols; ga.n = cols; ga.k = rows;
    ga.a = mm.dev; ga.lda = rows; ga.trans_a = true;
    ga.b = mm.dev; ga.ldb = rows;
    ga.c = g.ptr; ga.ldc = cols;
    gemm_simt(ga, st);
    std::vector<double> ev;
    std::vector<int64_t> order;
    eig_sym_dev(g.ptr, v.ptr, cols, ev, order, st);
    // sigma = sqrt(lambda); keep sigma > rcond * sigma_max
    const double smax = std::sqrt(std::max(0.0, ev[static_cast<size_t>(order[0])]));
    std::vector<double> inv(static_cast<size_t>(cols), 0.0);
    for (int64_t q = 0; q < cols; ++q) {
      const double lam = ev[static_cast<size_t>(q)];
      if (lam > 0.0 && std::sqrt(lam) > rcond * smax) inv[static_cast<size_t>(q)] = 1.0 / lam;
    }
    // W = (V diag(1/lambda)) V' (cols x cols), then pinv = W M'
    DevBuf<double> dinv(static_cast<size_t>(cols), st), vs(static_cast<size_t>(cols * cols), st),
        w(static_cast<size_t>(cols * cols), st);
    XCUDA(cudaMemcpyAsync(dinv.ptr, inv.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, st));
    scale_cols_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(cols * cols, 256), 1024)), 256, 0, st>>>(
        v.ptr, cols, cols, dinv.ptr, vs.ptr);
    XLAUNCH_CHECK();
    GemmArgs<double> gw;
    gw.m = cols; gw.n = cols; gw.k = cols;
    gw.a = vs.ptr; gw.lda = cols;
    gw.b = v.ptr; gw.ldb = cols; gw.trans_b = true;
    gw.c = w.ptr; gw.ldc = cols;
    gemm_simt(gw, st);
    OutView<double> o(out, static_cast<size_t>(cols * rows), st);
    GemmArgs<double> gb;
    gb.m = cols; gb.n = rows; gb.k = cols;
    gb.a = w.ptr; gb.lda = cols;
    gb.b = mm.dev; gb.ldb = rows; gb.trans_b = true;
    gb.c = o.dev; gb.ldc = cols;
    gemm_simt(gb, st);
    o.finish();
  });
}

// solve_least_squares (linalg.cpp:76-92)
int32_t xtsg_solve_least_squares(const double* a, int64_t rows, int64_t cols, const double* rhs, int64_t nrhs,
                                 double* x) {
  return guard([&] {
    if (rows < cols)
      throw Status(XTSG_E_ILLPOSED,
                   "solve_least_squares: underdetermined system (" + std::to_string(rows) + " rows < " +
                       std::to_string(cols) + " cols)",
                   std::min(rows, cols));
    require_device();
    cudaStream_t st = thread_stream();
    DevBuf<double> A(static_cast<size_t>(rows * cols), st), B(static_cast<size_t>(rows * nrhs), st);
    XCUDA(cudaMemcpyAsync(A.ptr, a, sizeof(double) * rows * cols, cudaMemcpyDefault, st));
    XCUDA(cudaMemcpyAsync(B.ptr, rhs, sizeof(double) * rows * nrhs, cudaMemcpyDefault, st));
    OutView<double> xo(x, static_cast<size_t>(cols * nrhs), st);
    const int64_t rank = lsq_colpiv_dev(A.ptr, rows, cols, B.ptr, nrhs, xo.dev, st);
    if (rank < cols)
      throw Status(XTSG_E_ILLPOSED,
                   "solve_least_squares: rank-deficient system (rank " + std::to_string(rank) + " of " +
                       std::to_string(cols) + ")",
                   rank);
    xo.finish();
  });
}

// omp_recover (alignment.cpp:306-419): out atoms x ncols
int32_t xtsg_omp_recover(const double* measured, int64_t rows, int64_t ncols, const double* dictionary,
                         int64_t atoms, int64_t sparsity, double residual_tol, double* out) {
  return guard([&] {
    if (sparsity < 1) usage("omp_recover: sparsity must be >= 1");
    if (sparsity > atoms) usage("omp_recover: sparsity exceeds dictionary size");
    if (sparsity >= rows) usage("omp_recover: sparsity must be below the measurement count");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> y(measured, static_cast<size_t>(rows * ncols), st), d(dictionary, static_cast<size_t>(rows * atoms), st);
    DevBuf<double> nrm(static_cast<size_t>(atoms), st);
    DevBuf<int> zc(1, st);
    const int big = 0x7fffffff;
    XCUDA(cudaMemcpyAsync(zc.ptr, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    atom_norm_kernel<<<static_cast<int>(std::min<int64_t>(atoms, 4096)), NT, 0, st>>>(d.dev, rows, atoms, nrm.ptr,
                                                                                      zc.ptr);
    XLAUNCH_CHECK();
    int hz = big;
    XCUDA(cudaMemcpyAsync(&hz, zc.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    XCUDA(cudaStreamSynchronize(st));
    if (hz != big) usage("omp_recover: dictionary column " + std::to_string(hz) + " is zero");
    OutView<double> o(out, static_cast<size_t>(atoms * ncols), st);
    XCUDA(cudaMemsetAsync(o.dev, 0, sizeof(double) * atoms * ncols, st));
    const int64_t ws_stride = rows + sparsity * (sparsity + 1) / 2 + 4 * sparsity + sparsity + 8;
    DevBuf<double> ws(static_cast<size_t>(std::max<int64_t>(1, ncols) * ws_stride), st);
    static const int64_t wide_from = [] {
      const char* e = std::getenv("XTSG_OMP_WIDE_FROM");
      return e ? static_cast<int64_t>(std::atoll(e)) : int64_t(4096);
    }();
    // residuals of `cb` columns must fit the opt-in shared memory next to the
    // kernel's static arrays; with not even one column (rows > ~28k) the
    // per-column omp_kernel (no rows limit) runs instead
    int dev = 0, optin = 0;
    XCUDA(cudaGetDevice(&dev));
    XCUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int64_t static_smem = (NT / 32) * OMP_CB * (sizeof(double) + sizeof(int64_t)) + 1024;
    const int64_t cb = std::min<int64_t>(OMP_CB, (optin - static_smem) / (sizeof(double) * std::max<int64_t>(1, rows)));
    if (ncols > 0 && atoms >= wide_from && cb >= 1) {
      // large dictionaries: the atom search over the whole GPU (omp_search_kernel)
      const int nsearch = std::max(1, std::min(sm_count() * 4, static_cast<int>(ceil_div(atoms, 64))));
      DevBuf<double> res(static_cast<size_t>(rows * ncols), st), cv(static_cast<size_t>(ncols * nsearch), st);
      DevBuf<int64_t> ci(static_cast<size_t>(ncols * nsearch), st);
      DevBuf<uint8_t> mask(static_cast<size_t>(atoms * ncols), st);
      DevBuf<int> done(static_cast<size_t>(ncols), st), na(static_cast<size_t>(ncols), st);
      mask.zero();
      omp_init_kernel<<<static_cast<unsigned>(ncols), NT, 0, st>>>(y.dev, rows, ncols, residual_tol, res.ptr,
                                                                   done.ptr, na.ptr);
      XLAUNCH_CHECK();
      const size_t smem = sizeof(double) * cb * rows;
      if (smem > 48 * 1024)
        XCUDA(cudaFuncSetAttribute(omp_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      for (int64_t it = 0; it < sparsity; ++it) {
        for (int64_t c0 = 0; c0 < ncols; c0 += cb) {
          const int nc = static_cast<int>(std::min<int64_t>(cb, ncols - c0));
          omp_search_kernel<<<nsearch, NT, sizeof(double) * nc * rows, st>>>(
              d.dev, rows, atoms, nrm.ptr, res.ptr, mask.ptr, done.ptr, c0, nc, cv.ptr, ci.ptr, ncols);
          XLAUNCH_CHECK();
        }
        omp_update_kernel<<<static_cast<unsigned>(ncols), NT, 0, st>>>(
            y.dev, d.dev, rows, atoms, static_cast<int>(sparsity), residual_tol, cv.ptr, ci.ptr, nsearch, mask.ptr,
            ncols, done.ptr, na.ptr, res.ptr, ws.ptr, ws_stride);
        XLAUNCH_CHECK();
      }
      omp_scatter_kernel<<<static_cast<unsigned>(ncols), NT, 0, st>>>(ws.ptr, ws_stride, static_cast<int>(sparsity),
                                                                      na.ptr, o.dev, atoms);
      XLAUNCH_CHECK();
    } else if (ncols > 0) {
      omp_kernel<<<static_cast<unsigned>(ncols), NT, 0, st>>>(y.dev, d.dev, rows, atoms, static_cast<int>(sparsity),
                                                              residual_tol, nrm.ptr, o.dev, atoms, ws.ptr, ws_stride);
      XLAUNCH_CHECK();
    }
    o.finish();
  });
}

}  // extern "C"
