// K9 — batched CP-ALS on the device (fp64), one CTA per ALS instance.
//
// Reference: cp_als (/root/reference/proj/src/cp_als.cpp:46-111) and
// relative_error (:37-44). Each sweep updates
//   A <- X(1) KR(C,B) pinv(C'C .* B'B),  B <- X(2) KR(C,A) pinv(C'C .* A'A),
//   C <- X(3) KR(B,A) pinv(B'B .* A'A),
// moves the a/b column norms into c (:84-96) and computes the residual
// explicitly (:98-99; the ||X||^2 - 2<X,Xh> + ||Xh||^2 shortcut cannot resolve
// the 1e-10 tolerance). Stops when the relative error changes by < tol.
// pinv (linalg.cpp:52-61, rcond 1e-12 of the largest singular value) is taken
// from a parallel-ordered cyclic Jacobi eigendecomposition of the symmetric
// PSD Hadamard Gram (singular values == |eigenvalues| there). nvecs init
// (:62-76, linalg.cpp:63-74) uses the same Jacobi on X(n) X(n)'.
//
// The replicas of one decomposition stage are independent, so a batch of P
// replicas (x restarts) runs as P CTAs; each replica tensor (<= a few MB) stays
// L2-resident across its sweeps. The Khatri-Rao products are never formed: the
// MTTKRPs contract one mode at a time (L*M*N*R FMAs each).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "sm100_ptx.cuh"
#include "xrng.cuh"

namespace xtsg {

namespace {

constexpr int NT = 256;
constexpr int RC = 4;  // ranks per work item in the MTTKRPs

struct AlsInst {
  const double* t;
  double* a;
  double* b;
  double* c;
  double* hist;
  int64_t* iters;
  int32_t* conv;
  double* nvec_ws;  // rows_max * rows_max * 2 doubles when nvecs
  double* pbuf;     // n2 * n3 * R doubles: A-contracted tensor of the sweep
  xtsg_als_config cfg;
};

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// Symmetric eigendecomposition of the n x n matrix h (leading dim ld) in place
// by parallel-ordered cyclic Jacobi; v receives the eigenvectors (columns),
// the diagonal of h the eigenvalues. cs/sn/pp/qq scratch of n/2+1 entries.
__device__ void jacobi_eig(double* h, double* v, int n, int ld, double* cs, double* sn, int* pp, int* qq,
                           double* red) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) v[(e % n) + ld * (e / n)] = (e % n) == (e / n) ? 1.0 : 0.0;
  __syncthreads();
  if (n < 2) return;
  const int m = n + (n & 1);  // even number of players; index n is a dummy when n is odd
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e % n, j = e / n;
      const double x = h[i + ld * j];
      tot += x * x;
      if (i != j) off += x * x;
    }
    off = block_sum(off, red);
    tot = block_sum(tot, red);
    if (off <= 1e-26 * tot || off == 0.0) break;
    for (int step = 0; step < m - 1; ++step) {
      for (int k = threadIdx.x; k < m / 2; k += blockDim.x) {
        auto who = [&](int i) { return i == 0 ? 0 : 1 + (i - 1 + step) % (m - 1); };
        int p = who(k), q = who(m - 1 - k);
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        pp[k] = p;
        qq[k] = q;
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = h[p + ld * q];
          if (apq != 0.0) {
            const double app = h[p + ld * p], aqq = h[q + ld * q];
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      // H <- H J (columns p, q) and V <- V J
      for (int e = threadIdx.x; e < (m / 2) * n; e += blockDim.x) {
        const int k = e / n, i = e % n;
        const int p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double hp = h[i + ld * p], hq = h[i + ld * q];
        h[i + ld * p] = c * hp - s * hq;
        h[i + ld * q] = s * hp + c * hq;
        const double vp = v[i + ld * p], vq = v[i + ld * q];
        v[i + ld * p] = c * vp - s * vq;
        v[i + ld * q] = s * vp + c * vq;
      }
      __syncthreads();
      // H <- J' H (rows p, q)
      for (int e = threadIdx.x; e < (m / 2) * n; e += blockDim.x) {
        const int k = e / n, j = e % n;
        const int p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double hp = h[p + ld * j], hq = h[q + ld * j];
        h[p + ld * j] = c * hp - s * hq;
        h[q + ld * j] = s * hp + c * hq;
      }
      __syncthreads();
    }
  }
}

struct Smem {
  double *A, *B, *C, *G1, *G2, *G3, *H, *V, *P, *M, *cs, *sn, *red, *nrm, *red2;
  int *pp, *qq;
};

// out[x, r] for one mode (mode 0: A, 1: B, 2: C) of T (n1 x n2 x n3).
__device__ void mttkrp(const double* __restrict__ T, int n1, int n2, int n3, int R, int mode, const Smem& s,
                       double* out) {
  const int rows = mode == 0 ? n1 : mode == 1 ? n2 : n3;
  const int nrq = (R + RC - 1) / RC;
  for (int item = threadIdx.x; item < rows * nrq; item += blockDim.x) {
    const int x = item % rows, r0 = (item / rows) * RC;
    double acc[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) acc[c] = 0.0;
    if (mode == 0) {  // sum_k C[k,r] sum_j T[x,j,k] B[j,r]
      for (int k = 0; k < n3; ++k) {
        double tmp[RC] = {0.0, 0.0, 0.0, 0.0};
        const double* tk = T + x + static_cast<int64_t>(n1) * n2 * k;
        for (int j = 0; j < n2; ++j) {
          const double tv = tk[static_cast<int64_t>(n1) * j];
#pragma unroll
          for (int c = 0; c < RC; ++c)
            if (r0 + c < R) tmp[c] = fma(tv, s.B[j + n2 * (r0 + c)], tmp[c]);
        }
#pragma unroll
        for (int c = 0; c < RC; ++c)
          if (r0 + c < R) acc[c] = fma(s.C[k + n3 * (r0 + c)], tmp[c], acc[c]);
      }
    } else if (mode == 1) {  // sum_k C[k,r] sum_i T[i,x,k] A[i,r]
      for (int k = 0; k < n3; ++k) {
        double tmp[RC] = {0.0, 0.0, 0.0, 0.0};
        const double* tk = T + static_cast<int64_t>(n1) * (x + static_cast<int64_t>(n2) * k);
        for (int i = 0; i < n1; ++i) {
          const double tv = tk[i];
#pragma unroll
          for (int c = 0; c < RC; ++c)
            if (r0 + c < R) tmp[c] = fma(tv, s.A[i + n1 * (r0 + c)], tmp[c]);
        }
#pragma unroll
        for (int c = 0; c < RC; ++c)
          if (r0 + c < R) acc[c] = fma(s.C[k + n3 * (r0 + c)], tmp[c], acc[c]);
      }
    } else {  // sum_j B[j,r] sum_i T[i,j,x] A[i,r]
      for (int j = 0; j < n2; ++j) {
        double tmp[RC] = {0.0, 0.0, 0.0, 0.0};
        const double* tj = T + static_cast<int64_t>(n1) * (j + static_cast<int64_t>(n2) * x);
        for (int i = 0; i < n1; ++i) {
          const double tv = tj[i];
#pragma unroll
          for (int c = 0; c < RC; ++c)
            if (r0 + c < R) tmp[c] = fma(tv, s.A[i + n1 * (r0 + c)], tmp[c]);
        }
#pragma unroll
        for (int c = 0; c < RC; ++c)
          if (r0 + c < R) acc[c] = fma(s.B[j + n2 * (r0 + c)], tmp[c], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < RC; ++c)
      if (r0 + c < R) out[x + rows * (r0 + c)] = acc[c];
  }
}

// Mode-1 MTTKRP with warp lanes over i (coalesced T reads) and thread groups
// over k: out[i, r] = sum_k C[k,r] sum_j T[i,j,k] B[j,r]. Per-group partials
// are reduced in a fixed order (bitwise-deterministic, like the reference).
constexpr int RED_DOUBLES = 4096;
// RCH: ranks per register chunk, chosen per launch to waste the fewest
// predicated FMA slots for the batch's rank (rch_for below)
template <int RCH>
__device__ void mttkrp0(const double* __restrict__ T, int n1, int n2, int n3, int R, const Smem& s, double* out,
                        double* red) {
  const int n1r = (n1 + 31) & ~31;
  const int W = n1r < (int)blockDim.x ? n1r : (int)blockDim.x;  // lanes over i per group
  const int G = (int)blockDim.x / W;                               // groups over k
  const int gid = threadIdx.x / W;
  for (int r0 = 0; r0 < R; r0 += RCH) {
    const int rc = R - r0 < RCH ? R - r0 : RCH;
    for (int i0 = 0; i0 < n1; i0 += W) {
      const int i = i0 + (threadIdx.x % W);
      double acc[RCH];
#pragma unroll
      for (int c = 0; c < RCH; ++c) acc[c] = 0.0;
      if (i < n1) {
        for (int k = gid; k < n3; k += G) {
          double tmp[RCH];
#pragma unroll
          for (int c = 0; c < RCH; ++c) tmp[c] = 0.0;
          const double* tk = T + i + static_cast<int64_t>(n1) * n2 * k;
#pragma unroll 4
          for (int j = 0; j < n2; ++j) {
            const double tv = __ldg(tk + static_cast<int64_t>(n1) * j);
#pragma unroll
            for (int c = 0; c < RCH; ++c)
              if (c < rc) tmp[c] = fma(tv, s.B[j + n2 * (r0 + c)], tmp[c]);
          }
#pragma unroll
          for (int c = 0; c < RCH; ++c)
            if (c < rc) acc[c] = fma(s.C[k + n3 * (r0 + c)], tmp[c], acc[c]);
        }
      }
      // fixed-order reduction over the G groups through shared scratch
      const int span = W < n1 - i0 ? W : n1 - i0;  // rows in this pass
      const int per_round = RED_DOUBLES / (G * RCH);
      for (int base = 0; base < span; base += per_round) {
        const int li = (threadIdx.x % W) - base;
        if (li >= 0 && li < per_round && i < n1)
#pragma unroll
          for (int c = 0; c < RCH; ++c) red[(gid * per_round + li) * RCH + c] = acc[c];
        __syncthreads();
        for (int e = threadIdx.x; e < per_round * rc; e += blockDim.x) {
          const int row = e / rc, c = e % rc;
          if (base + row >= span) continue;
          double v = 0.0;
          for (int g = 0; g < G; ++g) v += red[(g * per_round + row) * RCH + c];
          out[(i0 + base + row) + n1 * (r0 + c)] = v;
        }
        __syncthreads();
      }
    }
  }
}

// P[r][k][j] = sum_i T[i,j,k] A[i,r] (the A-contracted tensor shared by the B
// and C updates of a sweep), threads over (j, k) fibers, contiguous i reads.
template <int RCH>
__device__ void contract_a(const double* __restrict__ T, int n1, int n2, int n3, int R, const Smem& s,
                           double* __restrict__ P) {
  const int fibers = n2 * n3;
  for (int f = threadIdx.x; f < fibers; f += blockDim.x) {
    const double* col = T + static_cast<int64_t>(n1) * f;
    for (int r0 = 0; r0 < R; r0 += RCH) {
      double acc[RCH];
#pragma unroll
      for (int c = 0; c < RCH; ++c) acc[c] = 0.0;
#pragma unroll 4
      for (int i = 0; i < n1; ++i) {
        const double tv = __ldg(col + i);
#pragma unroll
        for (int c = 0; c < RCH; ++c)
          if (r0 + c < R) acc[c] = fma(tv, s.A[i + n1 * (r0 + c)], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < RCH; ++c)
        if (r0 + c < R) P[static_cast<int64_t>(r0 + c) * fibers + f] = acc[c];
    }
  }
}

// out_B[j, r] = sum_k C[k,r] P[r][k][j]
__device__ void mttkrp1_from_p(const double* __restrict__ P, int n2, int n3, int R, const Smem& s, double* out) {
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
    const int j = e % n2, r = e / n2;
    const double* pr = P + static_cast<int64_t>(r) * n2 * n3 + j;
    double acc = 0.0;
#pragma unroll 4
    for (int k = 0; k < n3; ++k) acc = fma(s.C[k + n3 * r], pr[static_cast<int64_t>(n2) * k], acc);
    out[e] = acc;
  }
}

// out_C[k, r] = sum_j B[j,r] P[r][k][j]
__device__ void mttkrp2_from_p(const double* __restrict__ P, int n2, int n3, int R, const Smem& s, double* out) {
  for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) {
    const int k = e % n3, r = e / n3;
    const double* pr = P + static_cast<int64_t>(r) * n2 * n3 + static_cast<int64_t>(n2) * k;
    double acc = 0.0;
#pragma unroll 4
    for (int j = 0; j < n2; ++j) acc = fma(s.B[j + n2 * r], pr[j], acc);
    out[e] = acc;
  }
}

// G = F' F (R x R, symmetric): four lanes per (r, q) pair, each summing every
// fourth row, combined by two xor-shuffles (a fixed, symmetric order).
__device__ void gram(const double* F, int rows, int R, double* G) {
  const int npair = R * (R + 1) / 2;
  for (int t0 = 0; t0 < 4 * npair; t0 += blockDim.x) {
    const int t = t0 + static_cast<int>(threadIdx.x);
    const int pidx = t >> 2, part = t & 3;
    double v = 0.0;
    int r = 0, q = 0;
    if (pidx < npair) {
      q = static_cast<int>((sqrt(8.0 * pidx + 1.0) - 1.0) * 0.5);
      while (q * (q + 1) / 2 > pidx) --q;
      while ((q + 1) * (q + 2) / 2 <= pidx) ++q;
      r = pidx - q * (q + 1) / 2;
      const double* fr = F + rows * r;
      const double* fq = F + rows * q;
      for (int i = part; i < rows; i += 4) v = fma(fr[i], fq[i], v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (pidx < npair && part == 0) {
      G[r + R * q] = v;
      G[q + R * r] = v;
    }
  }
}

// P = pinv(H) for symmetric PSD H (R x R), via Jacobi (H is destroyed).
__device__ void pinv_sym(double* H, int R, const Smem& s) {
  jacobi_eig(H, s.V, R, R, s.cs, s.sn, s.pp, s.qq, s.red);
  double mx = 0.0;
  for (int i = 0; i < R; ++i) mx = fmax(mx, fabs(H[i + R * i]));
  const double cut = 1e-12 * mx;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e % R, j = e / R;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) {
      const double lam = H[q + R * q];
      if (fabs(lam) > cut) acc += s.V[i + R * q] * s.V[j + R * q] / lam;
    }
    s.P[e] = acc;
  }
  __syncthreads();
}

// F[x, r] = sum_q Mt[x, q] P[q, r]
__device__ void apply_pinv(const double* Mt, int rows, int R, const double* P, double* F) {
  for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
    const int x = e % rows, r = e / rows;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) acc = fma(Mt[x + rows * q], P[q + R * r], acc);
    F[e] = acc;
  }
}

// F = Mt * pinv(H) for the symmetric Hadamard Gram H (R x R, in s.H).
// Fast path: Cholesky H = L L' by warp 0 (L into s.P) and one forward/back
// substitution per row of Mt (no block-wide syncs inside). When H is not
// safely positive definite (a pivot below 1e-11 of the largest diagonal —
// well above the reference's rcond = 1e-12 of sigma_max cut, linalg.cpp:56)
// it falls back to the Jacobi pseudo-inverse, i.e. the reference semantics.
// Cholesky trailing update of row i: L(i, j) -= L(i, k) L(j, k) for k < j <= i.
// The row (stride R) and column k never share an element, and saying so
// (__restrict__) lets the loads of successive j issue ahead of the stores.
__device__ __forceinline__ void chol_row_update(double* __restrict__ row, const double* __restrict__ colk, int R, int k,
                                                int i, double lik) {
  int j = k + 1;
  for (; j + 3 <= i; j += 4) {
    const double c0 = colk[j], c1 = colk[j + 1], c2 = colk[j + 2], c3 = colk[j + 3];
    const double r0 = row[R * j], r1 = row[R * (j + 1)], r2 = row[R * (j + 2)], r3 = row[R * (j + 3)];
    row[R * j] = fma(-lik, c0, r0);
    row[R * (j + 1)] = fma(-lik, c1, r1);
    row[R * (j + 2)] = fma(-lik, c2, r2);
    row[R * (j + 3)] = fma(-lik, c3, r3);
  }
  for (; j <= i; ++j) row[R * j] = fma(-lik, colk[j], row[R * j]);
}

// solve_gram in two halves: gram_factor_warp0 (warp 0: Cholesky of s.H into
// s.P / s.V, *ok) and gram_solve_factored (every thread, after a barrier:
// substitution, or the Jacobi pseudo-inverse when the factor failed). The
// cluster kernel runs the first half for the B update while the other warps
// compute P = A' T, since its input G3 .* G1 is known one phase early.
__device__ void gram_factor_warp0(int R, const Smem& s, int* ok);
__device__ void gram_solve_factored(const double* Mt, int rows, int R, const Smem& s, double* F, const int* ok);

__device__ void solve_gram(const double* Mt, int rows, int R, const Smem& s, double* F, int* ok) {
  if (threadIdx.x < 32) gram_factor_warp0(R, s, ok);
  __syncthreads();
  gram_solve_factored(Mt, rows, R, s, F, ok);
}

__device__ void gram_factor_warp0(int R, const Smem& s, int* ok) {
  {
    const int lane = threadIdx.x & 31;
    double* Lm = s.P;  // lower triangle, column-major R x R
    if (R > 64) {  // the per-row substitution keeps R values in registers/local memory
      if (lane == 0) *ok = 0;
    } else {
    // right-looking Cholesky in place (lower triangle of s.P), warp-synchronous
    for (int e = lane; e < R * R; e += 32) Lm[e] = s.H[e];
    __syncwarp();
    // largest diagonal: one load per lane and a warp max (not R dependent loads)
    double mxd = 0.0;
    for (int i = lane; i < R; i += 32) mxd = fmax(mxd, Lm[i + R * i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
    bool good = mxd > 0.0;
    for (int k = 0; k < R && good; ++k) {
      const double d = Lm[k + R * k];
      __syncwarp();
      if (!(d > 1e-11 * mxd)) {
        good = false;
        break;
      }
      // one reciprocal square root per pivot (no divisions): L(k,k) = d * rsqrt(d),
      // 1 / L(k,k) kept on the diagonal of s.V for the inverse below
      const double rl = rsqrt(d);
      for (int i = k + 1 + lane; i < R; i += 32) Lm[i + R * k] *= rl;
      if (lane == 0) {
        Lm[k + R * k] = d * rl;
        s.V[k + R * k] = rl;
      }
      __syncwarp();
      // trailing update, lane over rows i (the same fma per element as a
      // flat (i, j) walk, without an integer division per element; a row's
      // columns are independent, so their loads overlap)
      for (int i = k + 1 + lane; i < R; i += 32) chol_row_update(Lm + i, Lm + R * k, R, k, i, Lm[i + R * k]);
      __syncwarp();
    }
    if (good && R > 16) {
      // L^-1 column by column (lane c), still inside warp 0: H^-1 = L^-T L^-1
      for (int c = lane; c < R; c += 32)
        for (int i = c + 1; i < R; ++i) {
          double acc = 0.0;
          for (int j = c; j < i; ++j) acc = fma(Lm[i + R * j], s.V[j + R * c], acc);
          s.V[i + R * c] = -acc * s.V[i + R * i];
        }
    }
    if (lane == 0) *ok = good ? 1 : 0;
    }
  }
}

__device__ void gram_solve_factored(const double* Mt, int rows, int R, const Smem& s, double* F, const int* ok) {
  if (*ok && R <= 16) {
    // R <= 16: one forward and one back substitution per row of Mt
    // (L y = m_x, L' f = y; 1 / L(k,k) on the diagonal of s.V), every
    // thread a row, the R values of the row in registers
    const double* Lm = s.P;
    for (int x = threadIdx.x; x < rows; x += blockDim.x) {
      double y[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k < R) {
          double acc = Mt[x + rows * k];
#pragma unroll
          for (int j = 0; j < k; ++j) acc = fma(-Lm[k + R * j], y[j], acc);
          y[k] = acc * s.V[k + R * k];
        } else {
          y[k] = 0.0;
        }
      }
#pragma unroll
      for (int k = 15; k >= 0; --k) {
        if (k < R) {
          double acc = y[k];
#pragma unroll
          for (int j = k + 1; j < 16; ++j)
            if (j < R) acc = fma(-Lm[j + R * k], y[j], acc);
          y[k] = acc * s.V[k + R * k];
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < R) F[x + rows * k] = y[k];
    }
  } else if (*ok) {
    // H^-1 (into s.H) and F = Mt H^-1 over all threads
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int a = e % R, b = e / R;
      double acc = 0.0;
      for (int i = a > b ? a : b; i < R; ++i) acc = fma(s.V[i + R * a], s.V[i + R * b], acc);
      s.H[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
      const int x = e % rows, r = e / rows;
      double acc = 0.0;
      for (int q = 0; q < R; ++q) acc = fma(Mt[x + rows * q], s.H[q + R * r], acc);
      F[e] = acc;
    }
  } else {
    pinv_sym(s.H, R, s);
    apply_pinv(Mt, rows, R, s.P, F);
  }
}

// sum over (i, j, k) of (T - [[A, B, C]])^2: lanes over i, warps over (j, k)
// fibers (no 64-bit index arithmetic per element), two interleaved rank
// chains per element.
__device__ double residual_sq(const double* __restrict__ T, int n1, int n2, int n3, int R, const Smem& s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int fibers = n2 * n3;
  double acc = 0.0;
  for (int i0 = 0; i0 < n1; i0 += 32) {
    const int i = i0 + lane;
    const bool on = i < n1;
    const double* Ai = s.A + (on ? i : 0);
    for (int f = warp; f < fibers; f += nw) {
      const int j = f % n2, k = f / n2;
      const double* Bj = s.B + j;
      const double* Ck = s.C + k;
      double r0 = 0.0, r1 = 0.0;
      int r = 0;
      for (; r + 1 < R; r += 2) {
        r0 = fma(Ai[n1 * r], Bj[n2 * r] * Ck[n3 * r], r0);
        r1 = fma(Ai[n1 * (r + 1)], Bj[n2 * (r + 1)] * Ck[n3 * (r + 1)], r1);
      }
      if (r < R) r0 = fma(Ai[n1 * r], Bj[n2 * r] * Ck[n3 * r], r0);
      const double d = on ? T[i + static_cast<int64_t>(n1) * f] - (r0 + r1) : 0.0;
      acc = fma(d, d, acc);
    }
  }
  return block_sum(acc, s.red);
}

__device__ double norm_sq(const double* __restrict__ T, int64_t total, double* red) {
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) acc = fma(T[e], T[e], acc);
  return block_sum(acc, red);
}

// One polar stream of `n` normals (gaussian_matrix, cp_als.cpp:14-19) into dst,
// block-cooperative (same compaction as ensemble.cu).
__device__ void block_normals(uint64_t seed, int n, double* dst, double* red) {
  int* cnt = reinterpret_cast<int*>(red);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int produced = 0;
  uint64_t t0 = 0;
  while (produced < n) {
    double n0 = 0.0, n1 = 0.0;
    const bool acc = polar_candidate(seed, t0 + threadIdx.x, n0, n1);
    const unsigned mask = __ballot_sync(0xffffffffu, acc);
    __syncthreads();
    if (lane == 0) cnt[wid] = __popc(mask);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < wid) before += cnt[w];
      total += cnt[w];
    }
    before += __popc(mask & ((1u << lane) - 1u));
    const int pos = produced + 2 * before;
    if (acc) {
      if (pos < n) dst[pos] = n0;
      if (pos + 1 < n) dst[pos + 1] = n1;
    }
    produced += 2 * total;
    t0 += blockDim.x;
  }
  __syncthreads();
}

// leading eigenvectors of X(n) X(n)' into the first lead columns of F (rows x R)
__device__ void nvecs_init(const double* __restrict__ T, int n1, int n2, int n3, int mode, int R, double* F,
                           double* ws, const Smem& s) {
  const int rows = mode == 0 ? n1 : mode == 1 ? n2 : n3;
  double* G = ws;                 // rows x rows
  double* V = ws + rows * rows;   // rows x rows
  for (int e = threadIdx.x; e < rows * rows; e += blockDim.x) {
    const int p = e % rows, q = e / rows;
    if (p > q) continue;
    double acc = 0.0;
    if (mode == 0) {
      for (int64_t c = 0; c < static_cast<int64_t>(n2) * n3; ++c) acc = fma(T[p + n1 * c], T[q + n1 * c], acc);
    } else if (mode == 1) {
      for (int k = 0; k < n3; ++k)
        for (int i = 0; i < n1; ++i) {
          const int64_t base = i + static_cast<int64_t>(n1) * n2 * k;
          acc = fma(T[base + static_cast<int64_t>(n1) * p], T[base + static_cast<int64_t>(n1) * q], acc);
        }
    } else {
      const int64_t sl = static_cast<int64_t>(n1) * n2;
      for (int64_t c = 0; c < sl; ++c) acc = fma(T[c + sl * p], T[c + sl * q], acc);
    }
    G[p + rows * q] = acc;
    G[q + rows * p] = acc;
  }
  __syncthreads();
  jacobi_eig(G, V, rows, rows, s.cs, s.sn, s.pp, s.qq, s.red);
  // order by descending eigenvalue (stable: ties keep the lower index first)
  const int lead = R < rows ? R : rows;
  for (int jj = threadIdx.x; jj < lead; jj += blockDim.x) {
    // jj-th largest: count eigenvalues strictly greater (or equal with lower index)
    for (int cidx = 0; cidx < rows; ++cidx) {
      const double lc = G[cidx + rows * cidx];
      int rank = 0;
      for (int o = 0; o < rows; ++o) {
        const double lo = G[o + rows * o];
        if (lo > lc || (lo == lc && o < cidx)) ++rank;
      }
      if (rank == jj) {
        for (int i = 0; i < rows; ++i) F[i + rows * jj] = V[i + rows * cidx];
        break;
      }
    }
  }
  __syncthreads();
}

template <int RCH>
__global__ void __launch_bounds__(NT) als_kernel(const AlsInst* __restrict__ insts, int n1, int n2, int n3) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  const AlsInst in = insts[blockIdx.x];
  const int R = static_cast<int>(in.cfg.rank);
  const int mx = max(n1, max(n2, n3));
  Smem s;
  double* q = sm;
  s.A = q; q += n1 * R;
  s.B = q; q += n2 * R;
  s.C = q; q += n3 * R;
  s.G1 = q; q += R * R;
  s.G2 = q; q += R * R;
  s.G3 = q; q += R * R;
  s.H = q; q += R * R;
  s.V = q; q += R * R;
  s.P = q; q += R * R;
  s.M = q; q += mx * R;
  s.red2 = q; q += RED_DOUBLES;
  s.cs = q; q += std::max(mx, R) / 2 + 2;
  s.sn = q; q += std::max(mx, R) / 2 + 2;
  s.nrm = q; q += 2 * R;
  s.red = q; q += 64;
  s.pp = reinterpret_cast<int*>(q); q += std::max(mx, R) / 2 + 2;
  s.qq = reinterpret_cast<int*>(q);

  const double* T = in.t;
  const int64_t total = static_cast<int64_t>(n1) * n2 * n3;
  const double tn = sqrt(norm_sq(T, total, s.red));
  // init (cp_als.cpp:62-76)
  block_normals(derive(in.cfg.seed, 1), n1 * R, s.A, s.red);
  block_normals(derive(in.cfg.seed, 2), n2 * R, s.B, s.red);
  block_normals(derive(in.cfg.seed, 3), n3 * R, s.C, s.red);
  if (in.cfg.init == 1 && tn > 0.0) {
    nvecs_init(T, n1, n2, n3, 0, R, s.A, in.nvec_ws, s);
    nvecs_init(T, n1, n2, n3, 1, R, s.B, in.nvec_ws, s);
    nvecs_init(T, n1, n2, n3, 2, R, s.C, in.nvec_ws, s);
  }
  __syncthreads();
  gram(s.B, n2, R, s.G2);
  gram(s.C, n3, R, s.G3);
  __syncthreads();

  int64_t it = 0;
  bool converged = false;
  double prev = 0.0;
  for (; it < in.cfg.max_iters; ++it) {
    // A update
    mttkrp0<RCH>(T, n1, n2, n3, R, s, s.M, s.red2);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G3[e] * s.G2[e];
    __syncthreads();
    solve_gram(s.M, n1, R, s, s.A, &s_ok);
    __syncthreads();
    gram(s.A, n1, R, s.G1);
    __syncthreads();
    // B update
    contract_a<RCH>(T, n1, n2, n3, R, s, in.pbuf);
    __syncthreads();
    mttkrp1_from_p(in.pbuf, n2, n3, R, s, s.M);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G3[e] * s.G1[e];
    __syncthreads();
    solve_gram(s.M, n2, R, s, s.B, &s_ok);
    __syncthreads();
    gram(s.B, n2, R, s.G2);
    __syncthreads();
    // C update
    mttkrp2_from_p(in.pbuf, n2, n3, R, s, s.M);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G2[e] * s.G1[e];
    __syncthreads();
    solve_gram(s.M, n3, R, s, s.C, &s_ok);
    __syncthreads();
    // move a/b column norms into c (cp_als.cpp:84-96)
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double na = 0.0, nb = 0.0;
      for (int i = 0; i < n1; ++i) na = fma(s.A[i + n1 * r], s.A[i + n1 * r], na);
      for (int i = 0; i < n2; ++i) nb = fma(s.B[i + n2 * r], s.B[i + n2 * r], nb);
      s.nrm[r] = sqrt(na);
      s.nrm[R + r] = sqrt(nb);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
      const double na = s.nrm[e / n1];
      if (na > 0.0) s.A[e] /= na;
    }
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
      const double nb = s.nrm[R + e / n2];
      if (nb > 0.0) s.B[e] /= nb;
    }
    for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) {
      const int r = e / n3;
      s.C[e] *= s.nrm[r] * s.nrm[R + r];
    }
    __syncthreads();
    gram(s.A, n1, R, s.G1);
    gram(s.B, n2, R, s.G2);
    gram(s.C, n3, R, s.G3);
    const double res = sqrt(residual_sq(T, n1, n2, n3, R, s));
    const double err = tn > 0.0 ? res / tn : res;
    if (threadIdx.x == 0) in.hist[it] = err;
    if (it >= 1 && fabs(prev - err) < in.cfg.tol) {
      converged = true;
      ++it;
      break;
    }
    prev = err;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) in.a[e] = s.A[e];
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) in.b[e] = s.B[e];
  for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) in.c[e] = s.C[e];
  if (threadIdx.x == 0) {
    *in.iters = it;
    *in.conv = converged ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// Large replicas (e.g. config 3: 124 replicas of 128^3, rank 20): the same
// sweep, restructured so that T streams through shared memory twice per sweep
// and the contractions run on the fp64 tensor cores (DMMA m8n8k4):
//   pass 1  M_A = T(1) (C kr B) fused with the explicit residual of the
//           previous sweep (X^_k = (A diag(c_k)) B' tile by tile, compared
//           with the staged T tile): one T read serves both;
//   pass 2  P = T x1 A' (the A-contracted tensor, as contract_a) with M_B
//           accumulated on the fly; M_C from P and the new B as before.
// T arrives by 1-D bulk copies (cp.async.bulk, one per 8-column chunk column)
// into a 4-stage ring with a padded leading dimension (n1 + 4 doubles) that
// makes every DMMA fragment load bank-conflict free. Convergence is checked
// one pass later than in als_kernel (the residual of sweep s is computed in
// pass 1 of sweep s + 1), with identical semantics: iteration counts, history
// and returned factors are those of the sweep that met the tolerance.
constexpr int BJC = 8;       // T columns per staged chunk
constexpr int BNS_MAX = 8;   // chunk stages (as many as fit)

struct BigSmem {
  double *Ts, *Bp, *red;
  uint64_t *full, *empty;
  int ldt, ldb, ns;
  int sub;               // BJC-column sub-chunks per ring stage (1 or 2)
  uint32_t ns_m, cpk_m;  // multiply-high reciprocals of ns and n2 / (sub * BJC)
};

// x / d for d >= 2 and x < 2^32 / d: one IMAD.HI instead of the ~20-deep
// dependent integer-division sequence, which (int64 `%`/`/` by the runtime
// ring depth) was the per-chunk critical path of the ring (~1000 cycles per
// chunk, measured: tools/micro/bulk_ring.cu)
__host__ __device__ __forceinline__ uint32_t fdiv_magic(uint32_t d) { return 0xFFFFFFFFu / d + 1u; }
__device__ __forceinline__ uint32_t fdiv(uint32_t x, uint32_t m) { return __umulhi(x, m); }

__device__ __forceinline__ int big_ld(int n) { return n + 4; }  // n % 16 == 0 -> ld % 16 == 4

// refresh the zero-padded DMMA copy of B (n2 x Rp, leading dim ldb)
__device__ void big_refresh(const Smem& s, const BigSmem& g, int n2, int R) {
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) g.Bp[(e % n2) + g.ldb * (e / n2)] = s.B[e];
}

// thread 0: stage global chunk number `gnum` (local chunk c of the pass)
// (gnum: the chunk's global number, only compared with ns; x: the same number
// reduced by a multiple of 2 * ns, small enough for fdiv)
__device__ __forceinline__ void big_issue(const BigSmem& g, const double* T, int n1, int n2, int64_t gnum, uint32_t x,
                                          int c) {
  const uint32_t gq = fdiv(x, g.ns_m);
  const int stage = static_cast<int>(x - gq * g.ns);
  if (gnum >= g.ns) ptx::mbar_wait(&g.empty[stage], (gq - 1u) & 1u);
  const int w = g.sub * BJC, cpk = n2 / w;
  const int k = static_cast<int>(fdiv(c, g.cpk_m)), jb = (c - k * cpk) * w;
  const uint32_t col_bytes = static_cast<uint32_t>(n1) * 8u;
  ptx::mbar_arrive_expect_tx(&g.full[stage], col_bytes * w);
  double* dst = g.Ts + stage * w * g.ldt;
  const double* src = T + static_cast<int64_t>(n1) * (jb + static_cast<int64_t>(n2) * k);
  for (int jj = 0; jj < w; ++jj)
    ptx::bulk_g2s(dst + jj * g.ldt, src + static_cast<int64_t>(n1) * jj, col_bytes, &g.full[stage]);
}

__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(ptx::smem_u32(bar)), "r"(n) : "memory");
}

// Pass 1: M_A -> s.M (n1 x R); returns this thread's residual partial
// sum_(ijk) (T - [[A, B, C]])^2 when `want_res`.
template <int MTPW, int NTR>
__device__ double big_pass1(const double* __restrict__ T, int n1, int n2, int n3, int R, const Smem& s,
                            const BigSmem& g, int64_t& gcn, bool want_res) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int cpk = n2 / (g.sub * BJC), nch = n3 * cpk;
  double q[MTPW][NTR][2], macc[MTPW][NTR][2], areg[MTPW][2 * NTR], ahat[MTPW][2 * NTR];
#pragma unroll
  for (int m = 0; m < MTPW; ++m)
#pragma unroll
    for (int t = 0; t < NTR; ++t) q[m][t][0] = q[m][t][1] = macc[m][t][0] = macc[m][t][1] = 0.0;
  // A fragments (M = i, K = r) of this warp's row tiles (once per pass)
#pragma unroll
  for (int m = 0; m < MTPW; ++m)
#pragma unroll
    for (int kr = 0; kr < 2 * NTR; ++kr) {
      const int r = kr * 4 + lc;
      areg[m][kr] = r < R ? s.A[((warp * MTPW + m) * 8 + lr) + n1 * r] : 0.0;
    }
  double res = 0.0;
  const uint32_t gb = static_cast<uint32_t>(gcn % (2 * g.ns));  // ring position, once per pass
  for (int c = 0; c < nch; ++c, ++gcn) {
    if (threadIdx.x == 0 && c == 0)
      for (int q0 = 0; q0 < g.ns && q0 < nch; ++q0) big_issue(g, T, n1, n2, gcn + q0, gb + q0, q0);
    const int k = static_cast<int>(fdiv(c, g.cpk_m)), jb0 = (c - k * cpk) * (g.sub * BJC);
    const uint32_t gq = fdiv(gb + c, g.ns_m);
    const int stage = static_cast<int>(gb + c - gq * g.ns);
    ptx::mbar_wait(&g.full[stage], gq & 1u);
    for (int sb = 0; sb < g.sub; ++sb) {
      const int jb = jb0 + sb * BJC;
      const double* ts = g.Ts + (stage * g.sub + sb) * BJC * g.ldt;
      if (jb == 0) {
#pragma unroll
        for (int kr = 0; kr < 2 * NTR; ++kr) {
          const int r = kr * 4 + lc;
          const double ck = r < R ? s.C[k + n3 * r] : 0.0;
#pragma unroll
          for (int m = 0; m < MTPW; ++m) ahat[m][kr] = areg[m][kr] * ck;
        }
      }
      // GEMM 1: q[i, r] += sum_j T[i, j] B[j, r]
#pragma unroll
      for (int ks = 0; ks < BJC / 4; ++ks) {
        double b[NTR];
#pragma unroll
        for (int t = 0; t < NTR; ++t) b[t] = g.Bp[(jb + ks * 4 + lc) + g.ldb * (t * 8 + lr)];
#pragma unroll
        for (int m = 0; m < MTPW; ++m) {
          const double a = ts[((warp * MTPW + m) * 8 + lr) + g.ldt * (ks * 4 + lc)];
#pragma unroll
          for (int t = 0; t < NTR; ++t) ptx::dmma(q[m][t][0], q[m][t][1], a, b[t]);
        }
      }
      // GEMM 2 + residual: X^[i, j] = sum_r (A[i, r] C[k, r]) B[j, r]
      if (want_res) {
        double bb[2 * NTR];
#pragma unroll
        for (int kr = 0; kr < 2 * NTR; ++kr) bb[kr] = g.Bp[(jb + lr) + g.ldb * (kr * 4 + lc)];
#pragma unroll
        for (int m = 0; m < MTPW; ++m) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int kr = 0; kr < 2 * NTR; ++kr) ptx::dmma(d0, d1, ahat[m][kr], bb[kr]);
          const int i = (warp * MTPW + m) * 8 + lr;
          const double t0 = ts[i + g.ldt * (2 * lc)], t1 = ts[i + g.ldt * (2 * lc + 1)];
          res = fma(t0 - d0, t0 - d0, res);
          res = fma(t1 - d1, t1 - d1, res);
        }
      }
      if (sb == g.sub - 1) {  // stage fully read: release it, refill
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&g.empty[stage]);
        if (threadIdx.x == 0 && c + g.ns < nch) big_issue(g, T, n1, n2, gcn + g.ns, gb + c + g.ns, c + g.ns);
      }
      if (jb + BJC == n2) {  // slice k complete: macc += c_k .* q
#pragma unroll
        for (int t = 0; t < NTR; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = t * 8 + 2 * lc + e;
            const double ck = r < R ? s.C[k + n3 * r] : 0.0;
#pragma unroll
            for (int m = 0; m < MTPW; ++m) {
              macc[m][t][e] = fma(ck, q[m][t][e], macc[m][t][e]);
              q[m][t][e] = 0.0;
            }
          }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MTPW; ++m)
#pragma unroll
    for (int t = 0; t < NTR; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = t * 8 + 2 * lc + e;
        if (r < R) s.M[((warp * MTPW + m) * 8 + lr) + n1 * r] = macc[m][t][e];
      }
  return res;
}

// Pass 2: P[r][k][j] = sum_i T[i, j, k] A[i, r] into global P, and
// M_B[j, r] = sum_k C[k, r] P[r][k][j] into s.M (n2 x R). Two groups of four
// warps take alternate chunks (K = i split over a group's warps, partials
// reduced in a fixed order behind a group barrier); an even number of ring
// chunks per slice keeps every j column's slices in one group, so M_B
// accumulates over k in order.
template <int NTR>
__device__ void big_pass2(const double* __restrict__ T, int n1, int n2, int n3, int R, const Smem& s,
                          const BigSmem& g, int64_t& gcn, double* __restrict__ P) {
  constexpr int KS_MAX = 8;  // n1 <= 128
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp >> 2, wq = warp & 3, gtid = threadIdx.x & 127;
  const int lr = lane >> 2, lc = lane & 3;
  const int cpk = n2 / (g.sub * BJC), nch = n3 * cpk;  // cpk even: see big_sub()
  const int iw = n1 / 4, ks2 = iw / 4;  // i rows per warp, K steps
  double areg[NTR][KS_MAX];
#pragma unroll
  for (int t = 0; t < NTR; ++t)
#pragma unroll
    for (int ks = 0; ks < KS_MAX; ++ks) {
      const int r = t * 8 + lr;
      areg[t][ks] = (ks < ks2 && r < R) ? s.A[(wq * iw + ks * 4 + lc) + n1 * r] : 0.0;
    }
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) s.M[e] = 0.0;
  __syncthreads();
  const int rp = NTR * 8;
  int use = 0;
  const uint32_t gb = static_cast<uint32_t>(gcn % (2 * g.ns));  // ring position, once per pass
  for (int c = 0; c < nch; ++c, ++gcn) {
    if (threadIdx.x == 0 && c == 0)
      for (int q0 = 0; q0 < g.ns && q0 < nch; ++q0) big_issue(g, T, n1, n2, gcn + q0, gb + q0, q0);
    if ((c & 1) == grp) {
      const uint32_t gq = fdiv(gb + c, g.ns_m);
      const int stage = static_cast<int>(gb + c - gq * g.ns);
      const int k = static_cast<int>(fdiv(c, g.cpk_m)), jb0 = (c - k * cpk) * (g.sub * BJC);
      ptx::mbar_wait(&g.full[stage], gq & 1u);
      for (int sb = 0; sb < g.sub; ++sb) {
        const int jb = jb0 + sb * BJC;
        const double* ts = g.Ts + (stage * g.sub + sb) * BJC * g.ldt;
        double acc[NTR][2];
#pragma unroll
        for (int t = 0; t < NTR; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS_MAX; ++ks) {
          if (ks < ks2) {
            const double b = ts[(wq * iw + ks * 4 + lc) + g.ldt * lr];
#pragma unroll
            for (int t = 0; t < NTR; ++t) ptx::dmma(acc[t][0], acc[t][1], areg[t][ks], b);
          }
        }
        if (sb == g.sub - 1) {  // stage fully read by this warp
          __syncwarp();
          if (lane == 0) mbar_arrive_cnt(&g.empty[stage], 2);
        }
        double* red = g.red + (grp * 2 + (use & 1)) * 4 * rp * BJC;
        ++use;
#pragma unroll
        for (int t = 0; t < NTR; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) red[(wq * rp + t * 8 + lr) * BJC + 2 * lc + e] = acc[t][e];
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        for (int e = gtid; e < R * BJC; e += 128) {
          const int r = e / BJC, jj = e % BJC;
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < 4; ++w) v += red[(w * rp + r) * BJC + jj];
          const int j = jb + jj;
          P[static_cast<int64_t>(r) * n2 * n3 + static_cast<int64_t>(n2) * k + j] = v;
          s.M[j + n2 * r] = fma(s.C[k + n3 * r], v, s.M[j + n2 * r]);
        }
      }
    }
    // pass 2: the group that just consumed chunk c refills that stage with
    // chunk c + ns (its empty barrier only needs this group's arrivals), so
    // the two groups pipeline independently instead of waiting on each other
    if ((c & 1) == grp && gtid == 0 && c + g.ns < nch) big_issue(g, T, n1, n2, gcn + g.ns, gb + c + g.ns, c + g.ns);
  }
  __syncthreads();
}

size_t big_fixed_doubles(int n1, int n2, int n3, int R) {
  const int mx = std::max(n1, std::max(n2, n3));
  const int rp = (R + 7) / 8 * 8;
  return static_cast<size_t>(n2 + 4) * rp + 4 * 4 * rp * BJC + static_cast<size_t>(n1 + n2 + n3) * R + 6 * R * R +
         static_cast<size_t>(mx) * R + 2 * (std::max(mx, R) / 2 + 2) + 2 * R + 64 + 2 * (std::max(mx, R) / 2 + 2);
}
constexpr size_t BIG_SMEM_CAP = 225 * 1024;

// stages of `sub` sub-chunks that fit next to the fixed working set (0 when
// not even 3 do)
int big_stages(int n1, int n2, int n3, int R, int sub = 1) {
  const size_t fixed = big_fixed_doubles(n1, n2, n3, R) * 8;
  const size_t per = static_cast<size_t>(sub) * BJC * (n1 + 4) * 8;
  if (fixed + 3 * per > BIG_SMEM_CAP) return 0;
  return static_cast<int>(std::min<size_t>(BNS_MAX, (BIG_SMEM_CAP - fixed) / per));
}

template <int MTPW, int NTR>
__global__ void __launch_bounds__(NT, 1) als_big_kernel(const AlsInst* __restrict__ insts, int n1, int n2, int n3,
                                                        int ns, int sub, int dbg) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_ok;
  __shared__ __align__(8) uint64_t bars[2 * BNS_MAX];
  const AlsInst in = insts[blockIdx.x];
  const int R = static_cast<int>(in.cfg.rank);
  const int mx = max(n1, max(n2, n3));
  const int rp = NTR * 8;
  Smem s;
  BigSmem g;
  g.ldt = big_ld(n1);
  g.ldb = big_ld(n2);
  g.ns = ns;
  g.sub = sub;
  g.ns_m = fdiv_magic(static_cast<uint32_t>(ns));
  g.cpk_m = fdiv_magic(static_cast<uint32_t>(n2 / (sub * BJC)));
  double* q = sm;
  g.Ts = q; q += ns * sub * BJC * g.ldt;
  g.Bp = q; q += g.ldb * rp;
  g.red = q; q += 4 * 4 * rp * BJC;
  s.A = q; q += n1 * R;
  s.B = q; q += n2 * R;
  s.C = q; q += n3 * R;
  s.G1 = q; q += R * R;
  s.G2 = q; q += R * R;
  s.G3 = q; q += R * R;
  s.H = q; q += R * R;
  s.V = q; q += R * R;
  s.P = q; q += R * R;
  s.M = q; q += mx * R;
  s.red2 = nullptr;
  s.cs = q; q += std::max(mx, R) / 2 + 2;
  s.sn = q; q += std::max(mx, R) / 2 + 2;
  s.nrm = q; q += 2 * R;
  s.red = q; q += 64;
  s.pp = reinterpret_cast<int*>(q); q += std::max(mx, R) / 2 + 2;
  s.qq = reinterpret_cast<int*>(q);
  g.full = bars;
  g.empty = bars + BNS_MAX;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      ptx::mbar_init(&g.full[i], 1);
      ptx::mbar_init(&g.empty[i], 8);
    }
    ptx::fence_barrier_init();
  }
  for (int e = threadIdx.x; e < g.ldb * rp; e += blockDim.x) g.Bp[e] = 0.0;
  __syncthreads();

  const double* T = in.t;
  const int64_t total = static_cast<int64_t>(n1) * n2 * n3;
  const double tn = sqrt(norm_sq(T, total, s.red));
  block_normals(derive(in.cfg.seed, 1), n1 * R, s.A, s.red);
  block_normals(derive(in.cfg.seed, 2), n2 * R, s.B, s.red);
  block_normals(derive(in.cfg.seed, 3), n3 * R, s.C, s.red);
  if (in.cfg.init == 1 && tn > 0.0) {
    nvecs_init(T, n1, n2, n3, 0, R, s.A, in.nvec_ws, s);
    nvecs_init(T, n1, n2, n3, 1, R, s.B, in.nvec_ws, s);
    nvecs_init(T, n1, n2, n3, 2, R, s.C, in.nvec_ws, s);
  }
  __syncthreads();
  gram(s.B, n2, R, s.G2);
  gram(s.C, n3, R, s.G3);
  big_refresh(s, g, n2, R);
  __syncthreads();

  int64_t gcn = 0, it = 0, iters = 0;
  bool converged = false, stopped = false;
  double prev = 0.0;
  long long tp1 = 0, tp2 = 0, tc = 0, t00 = clock64();
  for (; it < in.cfg.max_iters; ++it) {
    // pass 1: M_A for sweep it, residual of sweep it - 1
    long long t0 = clock64();
    const double part = big_pass1<MTPW, NTR>(T, n1, n2, n3, R, s, g, gcn, it >= 1);
    tp1 += clock64() - t0;
    if (it >= 1) {
      const double res = sqrt(block_sum(part, s.red));
      const double err = tn > 0.0 ? res / tn : res;
      if (threadIdx.x == 0) in.hist[it - 1] = err;
      if (it - 1 >= 1 && fabs(prev - err) < in.cfg.tol) {
        converged = true;
        stopped = true;
        iters = it;
        break;
      }
      prev = err;
    }
    __syncthreads();
    // A update
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G3[e] * s.G2[e];
    __syncthreads();
    solve_gram(s.M, n1, R, s, s.A, &s_ok);
    __syncthreads();
    gram(s.A, n1, R, s.G1);
    __syncthreads();
    // pass 2 + B update
    t0 = clock64();
    big_pass2<NTR>(T, n1, n2, n3, R, s, g, gcn, in.pbuf);
    tp2 += clock64() - t0;
    t0 = clock64();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G3[e] * s.G1[e];
    __syncthreads();
    solve_gram(s.M, n2, R, s, s.B, &s_ok);
    __syncthreads();
    gram(s.B, n2, R, s.G2);
    __syncthreads();
    // C update
    mttkrp2_from_p(in.pbuf, n2, n3, R, s, s.M);
    tc += clock64() - t0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G2[e] * s.G1[e];
    __syncthreads();
    solve_gram(s.M, n3, R, s, s.C, &s_ok);
    __syncthreads();
    // move a/b column norms into c (cp_als.cpp:84-96)
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double na = 0.0, nb = 0.0;
      for (int i = 0; i < n1; ++i) na = fma(s.A[i + n1 * r], s.A[i + n1 * r], na);
      for (int i = 0; i < n2; ++i) nb = fma(s.B[i + n2 * r], s.B[i + n2 * r], nb);
      s.nrm[r] = sqrt(na);
      s.nrm[R + r] = sqrt(nb);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
      const double na = s.nrm[e / n1];
      if (na > 0.0) s.A[e] /= na;
    }
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
      const double nb = s.nrm[R + e / n2];
      if (nb > 0.0) s.B[e] /= nb;
    }
    for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) {
      const int r = e / n3;
      s.C[e] *= s.nrm[r] * s.nrm[R + r];
    }
    __syncthreads();
    gram(s.A, n1, R, s.G1);
    gram(s.B, n2, R, s.G2);
    gram(s.C, n3, R, s.G3);
    big_refresh(s, g, n2, R);
    __syncthreads();
  }
  if (dbg & 8) {
    if (threadIdx.x == 0) {
      in.hist[0] = double(tp1);
      in.hist[1] = double(tp2);
      in.hist[2] = double(tc);
      in.hist[3] = double(clock64() - t00);
      in.hist[4] = double(it);
    }
    return;
  }
  if (!stopped) {
    // residual of the last sweep (no next pass 1 to carry it)
    const double res = sqrt(residual_sq(T, n1, n2, n3, R, s));
    const double err = tn > 0.0 ? res / tn : res;
    const int64_t last = in.cfg.max_iters - 1;
    if (threadIdx.x == 0) in.hist[last] = err;
    converged = last >= 1 && fabs(prev - err) < in.cfg.tol;
    iters = in.cfg.max_iters;
  }
  for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) in.a[e] = s.A[e];
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) in.b[e] = s.B[e];
  for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) in.c[e] = s.C[e];
  if (threadIdx.x == 0) {
    *in.iters = iters;
    *in.conv = converged ? 1 : 0;
  }
}

// Shapes the large-replica kernel takes: 64 | n1 <= 128, 16 | n2, rank <= 24.
// ---------------------------------------------------------------------------
// Small replicas on CTA clusters (config 1's 30^3 replicas, the sampled
// blocks): the single-CTA kernel is latency-bound (every pass re-reads T from
// L2, ~150 us per sweep at 30^3). Here a cluster of CL CTAs owns one ALS
// instance: CTA c keeps the mode-3 slab k in [c*kc, (c+1)*kc) of T resident in
// its shared memory, the factors are replicated, and the three updates
// exchange only R-column partials through distributed shared memory:
//   M_A = sum_c (slab-c partial of T(1) (C kr B))       reduced in rank order
//   P_c = T_c x1 A' (own slab), M_B = sum_c (P_c with C) reduced in rank order
//   C rows of slab c solved by CTA c, all-gathered from the owners
//   residual = sum_c (slab-c partial), every CTA takes the same decision.
// Every reduction runs in a fixed order, so results are deterministic. The
// sweep, normalisation, residual and convergence rule are als_kernel's
// (cp_als.cpp:77-104); initial factors come from als_init_kernel.
namespace cg = cooperative_groups;

// init (cp_als.cpp:62-76): normals, nvecs on attempt 1, and ||T||
__global__ void __launch_bounds__(NT) als_init_kernel(const AlsInst* __restrict__ insts, int n1, int n2, int n3,
                                                      double* ia, double* ib, double* ic, double* tnorm) {
  // one CTA per (instance, mode): the three modes' normals and nvecs
  // eigenproblems are independent, and the Gram + Jacobi workspace (2 rows^2,
  // rows <= 64 on this path) lives in shared memory — the same arithmetic in
  // the same order as the one-CTA in-kernel version, without an L2 round trip
  // between the three barriers of every Jacobi rotation step
  extern __shared__ double sm[];
  const AlsInst in = insts[blockIdx.x];
  const int mode = static_cast<int>(blockIdx.y);
  const int R = static_cast<int>(in.cfg.rank);
  const int mx = max(n1, max(n2, n3));
  const int jac = max(mx, R) / 2 + 2;
  Smem s{};
  double* q = sm;
  s.red = q; q += 64;
  s.cs = q; q += jac;
  s.sn = q; q += jac;
  s.pp = reinterpret_cast<int*>(q); q += jac;
  s.qq = reinterpret_cast<int*>(q); q += jac;
  double* ws = q;  // G, V: rows x rows each
  const int rows = mode == 0 ? n1 : mode == 1 ? n2 : n3;
  double* F = mode == 0 ? ia + static_cast<int64_t>(blockIdx.x) * n1 * R
            : mode == 1 ? ib + static_cast<int64_t>(blockIdx.x) * n2 * R
                        : ic + static_cast<int64_t>(blockIdx.x) * n3 * R;
  const double tn = sqrt(norm_sq(in.t, static_cast<int64_t>(n1) * n2 * n3, s.red));
  block_normals(derive(in.cfg.seed, 1 + static_cast<uint64_t>(mode)), rows * R, F, s.red);
  if (in.cfg.init == 1 && tn > 0.0) nvecs_init(in.t, n1, n2, n3, mode, R, F, ws, s);
  if (mode == 0 && threadIdx.x == 0) tnorm[blockIdx.x] = tn;
}

struct ClusterLayout {
  int kc;
  size_t doubles;
};

__host__ __device__ inline ClusterLayout cluster_layout(int n1, int n2, int n3, int R, int CL) {
  const int kc = (n3 + CL - 1) / CL;
  const int mx = n1 > n2 ? (n1 > n3 ? n1 : n3) : (n2 > n3 ? n2 : n3);
  const int jac = (mx > R ? mx : R) / 2 + 2;
  size_t d = static_cast<size_t>(n1) * n2 * kc            // T slab
             + static_cast<size_t>(n1 + n2 + n3) * R      // A, B, C
             + static_cast<size_t>(kc) * R                // own C rows
             + static_cast<size_t>(n1 + n2) * R           // M_A / M_B partials
             + static_cast<size_t>(mx) * R                // reduced M
             + 6 * static_cast<size_t>(R) * R             // G1..G3, H, V, P
             + static_cast<size_t>(R) * n2 * kc           // P of the slab
             + 64 + 2 * R + 2 + 4 * jac;
  return {kc, d};
}

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT)
    als_cluster_kernel(const AlsInst* __restrict__ insts, int n1, int n2, int n3, const double* __restrict__ ia,
                       const double* __restrict__ ib, const double* __restrict__ ic,
                       const double* __restrict__ tnorm, int dbg) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = static_cast<int>(cl.block_rank());
  const int item = blockIdx.x / CL;
  const AlsInst in = insts[item];
  const int R = static_cast<int>(in.cfg.rank);
  const int mx = max(n1, max(n2, n3));
  const ClusterLayout lay = cluster_layout(n1, n2, n3, R, CL);
  const int kc = lay.kc;
  const int k0 = min(n3, crank * kc), nk = min(n3, k0 + kc) - k0;
  const int jac = max(mx, R) / 2 + 2;
  Smem s{};
  double* q = sm;
  double* Ts = q; q += static_cast<int64_t>(n1) * n2 * kc;
  s.A = q; q += n1 * R;
  s.B = q; q += n2 * R;
  s.C = q; q += n3 * R;
  double* Cown = q; q += kc * R;
  double* MAp = q; q += n1 * R;
  double* MBp = q; q += n2 * R;
  s.M = q; q += mx * R;
  s.G1 = q; q += R * R;
  s.G2 = q; q += R * R;
  s.G3 = q; q += R * R;
  s.H = q; q += R * R;
  s.V = q; q += R * R;
  s.P = q; q += R * R;
  double* Pl = q; q += R * n2 * kc;
  s.red = q; q += 64;
  s.nrm = q; q += 2 * R;
  double* rs = q; q += 2;
  s.cs = q; q += jac;
  s.sn = q; q += jac;
  s.pp = reinterpret_cast<int*>(q); q += jac;
  s.qq = reinterpret_cast<int*>(q);
  // the slab is contiguous in the column-major replica
  const int64_t slab = static_cast<int64_t>(n1) * n2 * nk;
  const double* Tg = in.t + static_cast<int64_t>(n1) * n2 * k0;
  for (int64_t e = threadIdx.x; e < slab; e += blockDim.x) Ts[e] = Tg[e];
  for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) s.A[e] = ia[static_cast<int64_t>(item) * n1 * R + e];
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) s.B[e] = ib[static_cast<int64_t>(item) * n2 * R + e];
  for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) s.C[e] = ic[static_cast<int64_t>(item) * n3 * R + e];
  const double tn = tnorm[item];
  __syncthreads();
  gram(s.B, n2, R, s.G2);
  gram(s.C, n3, R, s.G3);
  __syncthreads();
  const int nf = n2 * nk;  // fibers (j, kk) of the slab
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;  // DMMA m8n8k4 fragment coordinates

  int64_t it = 0;
  bool converged = false;
  double prev = 0.0;
  // dbg: per-phase SM cycles of crank 0 / thread 0 (tools/als_small_probe.py)
  long long tph[7] = {0, 0, 0, 0, 0, 0, 0}, tl = clock64(), tsub[4] = {0, 0, 0, 0}, tl2 = 0;
  auto phase = [&](int ph) {
    if (dbg) {
      const long long t = clock64();
      tph[ph] += t - tl;
      tl = t;
    }
  };
  for (; it < in.cfg.max_iters; ++it) {
    // ---- A update: slab partial of T(1) (C kr B) on the fp64 tensor cores
    // (DMMA m8n8k4: 8 i x 8 r tiles, K = the slab's (j, kk) fibers),
    // reduced over the cluster
    {
      const int nti = (n1 + 7) / 8, ntr = (R + 7) / 8;
      for (int tile = warp; tile < nti * ntr; tile += nwarps) {
        const int i0 = (tile % nti) * 8, r0 = (tile / nti) * 8;
        const int ia = i0 + lr, rb = r0 + lr;
        double d0 = 0.0, d1 = 0.0;
        // fiber f = f0 + lc -> (j, kk) = (f % n2, f / n2), stepped by 4
        // without a runtime division per DMMA (it sat on the chain's critical path)
        int j = lc % n2, kk = lc / n2;
        for (int f0 = 0; f0 < nf; f0 += 4) {
          const int f = f0 + lc;
          const double a = (ia < n1 && f < nf) ? Ts[ia + static_cast<int64_t>(n1) * f] : 0.0;
          const double b = (f < nf && rb < R) ? s.B[j + n2 * rb] * s.C[(k0 + kk) + n3 * rb] : 0.0;
          ptx::dmma(d0, d1, a, b);
          j += 4;
          while (j >= n2) {
            j -= n2;
            ++kk;
          }
        }
        const int rc = r0 + 2 * lc;
        if (ia < n1) {
          if (rc < R) MAp[ia + n1 * rc] = d0;
          if (rc + 1 < R) MAp[ia + n1 * (rc + 1)] = d1;
        }
      }
    }
    phase(0);
    if (dbg) tl2 = clock64();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) s.H[e] = s.G3[e] * s.G2[e];
    cl.sync();
    if (dbg) { const long long t = clock64(); tsub[0] += t - tl2; tl2 = t; }
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < CL; ++c) v += cl.map_shared_rank(MAp, c)[e];
      s.M[e] = v;
    }
    __syncthreads();
    if (dbg) { const long long t = clock64(); tsub[1] += t - tl2; tl2 = t; }
    solve_gram(s.M, n1, R, s, s.A, &s_ok);
    __syncthreads();
    if (dbg) { const long long t = clock64(); tsub[2] += t - tl2; tl2 = t; }
    gram(s.A, n1, R, s.G1);
    __syncthreads();
    if (dbg) { const long long t = clock64(); tsub[3] += t - tl2; tl2 = t; }
    phase(1);
    // ---- P = A' T_c on the slab (DMMA: 8 r x 8 fibers tiles, K = i) by warps
    // 1..7 while warp 0 factors the B update's Gram H = G3 .* G1 (known now:
    // the same Cholesky solve_gram would run after the M_B reduction)
    if (warp == 0) {
      for (int e = lane; e < R * R; e += 32) s.H[e] = s.G3[e] * s.G1[e];
      __syncwarp();
      gram_factor_warp0(R, s, &s_ok);
    } else {
      const int ntr = (R + 7) / 8, ntf = (nf + 7) / 8;
      for (int tile = warp - 1; tile < ntr * ntf; tile += nwarps - 1) {
        const int r0 = (tile % ntr) * 8, f0 = (tile / ntr) * 8;
        const int ra = r0 + lr, fb = f0 + lr;
        double d0 = 0.0, d1 = 0.0;
        for (int i0 = 0; i0 < n1; i0 += 4) {
          const int i = i0 + lc;
          const double a = (ra < R && i < n1) ? s.A[i + n1 * ra] : 0.0;
          const double b = (fb < nf && i < n1) ? Ts[i + static_cast<int64_t>(n1) * fb] : 0.0;
          ptx::dmma(d0, d1, a, b);
        }
        const int fc = f0 + 2 * lc;
        if (ra < R) {
          if (fc < nf) Pl[static_cast<int64_t>(ra) * n2 * kc + fc] = d0;
          if (fc + 1 < nf) Pl[static_cast<int64_t>(ra) * n2 * kc + fc + 1] = d1;
        }
      }
    }
    __syncthreads();
    phase(2);
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
      const int j = e % n2, r = e / n2;
      const double* pr = Pl + static_cast<int64_t>(r) * n2 * kc + j;
      double acc = 0.0;
      for (int kk = 0; kk < nk; ++kk) acc = fma(s.C[(k0 + kk) + n3 * r], pr[n2 * kk], acc);
      MBp[e] = acc;
    }
    cl.sync();
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < CL; ++c) v += cl.map_shared_rank(MBp, c)[e];
      s.M[e] = v;
    }
    __syncthreads();
    gram_solve_factored(s.M, n2, R, s, s.B, &s_ok);
    __syncthreads();
    gram(s.B, n2, R, s.G2);
    __syncthreads();
    phase(3);
    // ---- C rows of this slab: M_C[kk, r] = sum_j B[j, r] P[r][kk][j] by
    // warps 1..7 while warp 0 factors H = G2 .* G1
    if (warp == 0) {
      for (int e = lane; e < R * R; e += 32) s.H[e] = s.G2[e] * s.G1[e];
      __syncwarp();
      gram_factor_warp0(R, s, &s_ok);
    } else {
      for (int e = threadIdx.x - 32; e < nk * R; e += blockDim.x - 32) {
        const int kk = e % nk, r = e / nk;
        const double* pr = Pl + static_cast<int64_t>(r) * n2 * kc + n2 * kk;
        const double* Br = s.B + n2 * r;
        double acc = 0.0;
        for (int j = 0; j < n2; ++j) acc = fma(Br[j], pr[j], acc);
        s.M[e] = acc;
      }
    }
    __syncthreads();
    gram_solve_factored(s.M, nk, R, s, Cown, &s_ok);
    cl.sync();
    // all-gather the new C rows from their owners
    for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) {
      const int k = e % n3, r = e / n3;
      const int c = k / kc, kk = k - c * kc;
      const int nkc = min(n3, (c + 1) * kc) - c * kc;
      s.C[e] = cl.map_shared_rank(Cown, c)[kk + nkc * r];
    }
    __syncthreads();
    phase(4);
    // ---- move a/b column norms into c (cp_als.cpp:84-96)
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double na = 0.0, nb = 0.0;
      for (int i = 0; i < n1; ++i) na = fma(s.A[i + n1 * r], s.A[i + n1 * r], na);
      for (int i = 0; i < n2; ++i) nb = fma(s.B[i + n2 * r], s.B[i + n2 * r], nb);
      s.nrm[r] = sqrt(na);
      s.nrm[R + r] = sqrt(nb);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
      const double na = s.nrm[e / n1];
      if (na > 0.0) s.A[e] /= na;
    }
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
      const double nb = s.nrm[R + e / n2];
      if (nb > 0.0) s.B[e] /= nb;
    }
    for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) {
      const int r = e / n3;
      s.C[e] *= s.nrm[r] * s.nrm[R + r];
    }
    __syncthreads();
    gram(s.A, n1, R, s.G1);
    gram(s.B, n2, R, s.G2);
    gram(s.C, n3, R, s.G3);
    phase(5);
    // ---- residual of the slab: X^ = A (C kr B)' tile by tile on DMMA
    // (8 i x 8 fibers, K = r), compared with the resident T
    {
      double acc = 0.0;
      const int nti = (n1 + 7) / 8, ntf = (nf + 7) / 8;
      for (int tile = warp; tile < nti * ntf; tile += nwarps) {
        const int i0 = (tile % nti) * 8, f0 = (tile / nti) * 8;
        const int ia = i0 + lr, fb = f0 + lr;
        int jb = 0, kb = 0;
        if (fb < nf) {
          jb = fb % n2;
          kb = fb / n2;
        }
        double d0 = 0.0, d1 = 0.0;
        for (int r0 = 0; r0 < R; r0 += 4) {
          const int r = r0 + lc;
          const double a = (ia < n1 && r < R) ? s.A[ia + n1 * r] : 0.0;
          const double b = (fb < nf && r < R) ? s.B[jb + n2 * r] * s.C[(k0 + kb) + n3 * r] : 0.0;
          ptx::dmma(d0, d1, a, b);
        }
        const int fc = f0 + 2 * lc;
        if (ia < n1) {
          if (fc < nf) {
            const double dd = Ts[ia + static_cast<int64_t>(n1) * fc] - d0;
            acc = fma(dd, dd, acc);
          }
          if (fc + 1 < nf) {
            const double dd = Ts[ia + static_cast<int64_t>(n1) * (fc + 1)] - d1;
            acc = fma(dd, dd, acc);
          }
        }
      }
      acc = block_sum(acc, s.red);
      if (threadIdx.x == 0) rs[0] = acc;
    }
    cl.sync();
    double res2 = 0.0;
#pragma unroll
    for (int c = 0; c < CL; ++c) res2 += cl.map_shared_rank(rs, c)[0];
    const double res = sqrt(res2);
    const double err = tn > 0.0 ? res / tn : res;
    phase(6);
    if (crank == 0 && threadIdx.x == 0) in.hist[it] = err;
    if (it >= 1 && fabs(prev - err) < in.cfg.tol) {
      converged = true;
      ++it;
      break;
    }
    prev = err;
  }
  if (dbg && crank == 0 && threadIdx.x == 0 && in.cfg.max_iters >= 8) {
    for (int ph = 0; ph < 7; ++ph) in.hist[ph] = static_cast<double>(tph[ph]);
    in.hist[7] = static_cast<double>(it);
    if (in.cfg.max_iters >= 12)
      for (int q = 0; q < 4; ++q) in.hist[8 + q] = static_cast<double>(tsub[q]);
  }
  if (crank == 0) {
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) in.a[e] = s.A[e];
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) in.b[e] = s.B[e];
    for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) in.c[e] = s.C[e];
    if (threadIdx.x == 0) {
      *in.iters = it;
      *in.conv = converged ? 1 : 0;
    }
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

// cluster size for the small-replica kernel: the largest CL in {8, 4, 2}
// (at most one slice per CTA) whose per-CTA working set fits 110 KB — more
// CTAs per instance shorten every phase of the latency-bound sweep (30^3:
// 61 -> 51 us per sweep from CL 4 to 8); 0 when none fits (or
// XTSG_ALS_CLUSTER=0; XTSG_ALS_CLUSTER=1|2|4|8 forces a size)
int als_cluster_size(int64_t n1, int64_t n2, int64_t n3, int64_t R) {
  static const int env = [] {
    const char* e = std::getenv("XTSG_ALS_CLUSTER");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0 || R > 32 || n1 > 64 || n2 > 64 || n3 > 64 || n3 < 2) return 0;
  // two CTAs per SM when the slab fits 110 KB; else one per SM (up to 200 KB:
  // 40^3 replicas at rank 20, 155 KB with 8 CTAs) rather than the one-CTA kernel
  for (const size_t cap : {size_t(110) * 1024, size_t(200) * 1024})
    for (int cl : {16, 8, 4, 2, 1}) {
      if (env > 0 && cl != env) continue;
      if (env <= 0 && (cl == 1 || cl == 16)) continue;  // 1 and 16 (non-portable) only on request
      if (cl > n3) continue;
      if (cluster_layout(int(n1), int(n2), int(n3), int(R), cl).doubles * 8 <= cap) return cl;
    }
  return 0;
}

void launch_als_cluster(const AlsInst* din, int64_t count, int n1, int n2, int n3, int R, int CL, cudaStream_t st) {
  DevBuf<double> ia(static_cast<size_t>(count * n1 * R), st), ib(static_cast<size_t>(count * n2 * R), st),
      ic(static_cast<size_t>(count * n3 * R), st), tn(static_cast<size_t>(count), st);
  const int mx = std::max(n1, std::max(n2, n3));
  const size_t ismem = sizeof(double) * (64 + 4 * (std::max(mx, R) / 2 + 2) + 2 * static_cast<size_t>(mx) * mx);
  XCUDA(cudaFuncSetAttribute(als_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ismem)));
  als_init_kernel<<<dim3(static_cast<unsigned>(count), 3), NT, ismem, st>>>(din, n1, n2, n3, ia.ptr, ib.ptr, ic.ptr,
                                                                           tn.ptr);
  XLAUNCH_CHECK();
  const size_t smem = cluster_layout(n1, n2, n3, R, CL).doubles * 8;
  auto go = [&](auto kern) {
    XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (CL > 8) XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    static const int dbg = [] {
      const char* e = std::getenv("XTSG_ALS_CL_DBG");  // per-phase cycles into history[0..7]
      return e ? std::atoi(e) : 0;
    }();
    kern<<<static_cast<unsigned>(count * CL), NT, smem, st>>>(din, n1, n2, n3, ia.ptr, ib.ptr, ic.ptr, tn.ptr, dbg);
  };
  if (CL == 16) go(als_cluster_kernel<16>);
  else if (CL == 1) go(als_cluster_kernel<1>);
  else if (CL == 2) go(als_cluster_kernel<2>);
  else if (CL == 4) go(als_cluster_kernel<4>);
  else go(als_cluster_kernel<8>);
  XLAUNCH_CHECK();
}

bool als_big_eligible(int64_t n1, int64_t n2, int64_t n3, int64_t R) {
  static const bool off = [] {
    const char* e = std::getenv("XTSG_ALS_BIG");
    return e && std::atoi(e) == 0;
  }();
  if (off) return false;
  if (!(n1 % 64 == 0 && n1 <= 128 && n2 % 16 == 0 && n2 <= 1024 && n3 >= 1 && n3 <= 1024 && R >= 1 && R <= 24))
    return false;
  return big_stages(int(n1), int(n2), int(n3), int(R)) >= 3;
}

// sub-chunks per ring stage: two (16 columns: half the per-stage ring
// bookkeeping, barrier waits and refills) when n2 % 32 == 0 keeps an even
// number of stages per slice and at least 3 such stages fit, else one
int big_sub(int n1, int n2, int n3, int R) {
  if (const char* e = std::getenv("XTSG_ALS_BIG_SUB"))  // "1": 8-column stages (A/B runs)
    if (std::atoi(e) == 1) return 1;
  return (n2 % 32 == 0 && big_stages(n1, n2, n3, R, 2) >= 3) ? 2 : 1;
}

void launch_als_big(const AlsInst* din, int64_t count, int n1, int n2, int n3, int R, cudaStream_t st) {
  const int sub = big_sub(n1, n2, n3, R);
  const int ns = big_stages(n1, n2, n3, R, sub);
  const size_t smem = 8 * (big_fixed_doubles(n1, n2, n3, R) + static_cast<size_t>(ns) * sub * BJC * (n1 + 4));
  const int mtpw = n1 / 64, ntr = (R + 7) / 8;
  auto go = [&](auto kern) {
    XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    static const int dbg = [] {
      const char* e = std::getenv("XTSG_ALS_BIG_DBG");  // 8: per-phase cycle counts (tools/als_big_cycles.py)
      return e ? std::atoi(e) : 0;
    }();
    kern<<<static_cast<unsigned>(count), NT, smem, st>>>(din, n1, n2, n3, ns, sub, dbg);
  };
  if (mtpw == 1) {
    if (ntr == 1) go(als_big_kernel<1, 1>); else if (ntr == 2) go(als_big_kernel<1, 2>); else go(als_big_kernel<1, 3>);
  } else {
    if (ntr == 1) go(als_big_kernel<2, 1>); else if (ntr == 2) go(als_big_kernel<2, 2>); else go(als_big_kernel<2, 3>);
  }
  XLAUNCH_CHECK();
}

// register chunk of ranks for the small-replica kernel: fewest wasted
// (predicated) FMA slots over ceil(R / RCH) chunks, larger chunks on ties
int rch_for(int R) {
  int best = 16, waste = 1 << 30;
  for (int c : {16, 12, 10, 8, 4}) {
    const int w = ((R + c - 1) / c) * c - R;
    if (w < waste) {
      waste = w;
      best = c;
    }
  }
  return best;
}

size_t als_smem_bytes(int n1, int n2, int n3, int R) {
  const int mx = std::max(n1, std::max(n2, n3));
  return sizeof(double) * (static_cast<size_t>(n1 + n2 + n3) * R + 6 * R * R + static_cast<size_t>(mx) * R + 4096 +
                           2 * (std::max(mx, R) / 2 + 2) + 2 * R + 64 + 2 * (std::max(mx, R) / 2 + 2));
}

__global__ void finite_kernel(const double* t, int64_t n, int* bad) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(t[e])) *bad = 1;
}

__global__ void relerr_kernel(const double* T, int n1, int n2, int n3, const double* a, const double* b,
                              const double* c, int R, double* out) {
  extern __shared__ double sm[];
  Smem s{};
  s.A = sm;
  s.B = sm + n1 * R;
  s.C = sm + (n1 + n2) * R;
  s.red = sm + (n1 + n2 + n3) * R;
  for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) s.A[e] = a[e];
  for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) s.B[e] = b[e];
  for (int e = threadIdx.x; e < n3 * R; e += blockDim.x) s.C[e] = c[e];
  __syncthreads();
  const double res = sqrt(residual_sq(T, n1, n2, n3, R, s));
  const double tn = sqrt(norm_sq(T, static_cast<int64_t>(n1) * n2 * n3, s.red));
  if (threadIdx.x == 0) *out = tn > 0.0 ? res / tn : res;
}

}  // namespace

}  // namespace xtsg

using namespace xtsg;

extern "C" {

int32_t xtsg_cp_als_batched(int64_t count, const double* t, int64_t n1, int64_t n2, int64_t n3,
                            const xtsg_als_config* cfg, double* a, double* b, double* c, int64_t* iters,
                            int32_t* converged, double* history) {
  return guard([&] {
    if (count < 0) usage("cp_als: negative batch");
    if (count == 0) return;
    int64_t max_it = 0, rank = cfg[0].rank;
    for (int64_t q = 0; q < count; ++q) {
      // cp_als.cpp:47-55
      if (cfg[q].rank < 1) usage("cp_als: rank must be >= 1");
      if (cfg[q].max_iters < 1) usage("cp_als: max_iters must be >= 1");
      if (!(cfg[q].tol > 0.0)) usage("cp_als: tol must be positive");
      if (cfg[q].rank != rank) usage("cp_als: a batch shares one rank");
      max_it = std::max(max_it, cfg[q].max_iters);
    }
    const int64_t cap = std::min({n2 * n3, n1 * n3, n1 * n2});
    if (rank > cap)
      usage("cp_als: rank " + std::to_string(rank) + " exceeds the identifiable bound " + std::to_string(cap));
    require_device();
    cudaStream_t st = thread_stream();
    const int64_t tsz = n1 * n2 * n3;
    InView<double> tt(t, static_cast<size_t>(count * tsz), st);
    {
      DevBuf<int> bad(1, st);
      bad.zero();
      finite_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(count * tsz, 256), 4096)), 256, 0, st>>>(
          tt.dev, count * tsz, bad.ptr);
      XLAUNCH_CHECK();
      int hb = 0;
      XCUDA(cudaMemcpyAsync(&hb, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
      XCUDA(cudaStreamSynchronize(st));
      if (hb) data_error("cp_als: input tensor has non-finite values");
    }
    const int R = static_cast<int>(rank);
    const size_t smem = als_smem_bytes(static_cast<int>(n1), static_cast<int>(n2), static_cast<int>(n3), R);
    if (smem > 220 * 1024) usage("cp_als: factors do not fit the device ALS working set (reduce rank/dims)");
    OutView<double> oa(a, static_cast<size_t>(count * n1 * rank), st), ob(b, static_cast<size_t>(count * n2 * rank), st),
        oc(c, static_cast<size_t>(count * n3 * rank), st);
    OutView<double> oh(history, static_cast<size_t>(count * max_it), st);
    OutView<int64_t> oi(iters, static_cast<size_t>(count), st);
    OutView<int32_t> ov(converged, static_cast<size_t>(count), st);
    bool any_nvecs = false;
    for (int64_t q = 0; q < count; ++q) any_nvecs |= cfg[q].init == 1;
    const int64_t rmax = std::max({n1, n2, n3});
    DevBuf<double> ws(any_nvecs ? static_cast<size_t>(count * rmax * rmax * 2) : 0, st);
    DevBuf<double> pb(static_cast<size_t>(count * n2 * n3 * rank), st);
    std::vector<AlsInst> hin(static_cast<size_t>(count));
    for (int64_t q = 0; q < count; ++q) {
      AlsInst& in = hin[static_cast<size_t>(q)];
      in.t = tt.dev + q * tsz;
      in.a = oa.dev + q * n1 * rank;
      in.b = ob.dev + q * n2 * rank;
      in.c = oc.dev + q * n3 * rank;
      in.hist = oh.dev + q * max_it;
      in.iters = oi.dev + q;
      in.conv = ov.dev + q;
      in.nvec_ws = any_nvecs ? ws.ptr + q * rmax * rmax * 2 : nullptr;
      in.pbuf = pb.ptr + q * n2 * n3 * rank;
      in.cfg = cfg[q];
    }
    DevBuf<AlsInst> din(static_cast<size_t>(count), st);
    XCUDA(cudaMemcpyAsync(din.ptr, hin.data(), sizeof(AlsInst) * count, cudaMemcpyHostToDevice, st));
    const int ccl = als_cluster_size(n1, n2, n3, rank);
    if (ccl > 0) {
      launch_als_cluster(din.ptr, count, static_cast<int>(n1), static_cast<int>(n2), static_cast<int>(n3), R, ccl,
                         st);
    } else if (als_big_eligible(n1, n2, n3, rank)) {
      launch_als_big(din.ptr, count, static_cast<int>(n1), static_cast<int>(n2), static_cast<int>(n3), R, st);
    } else {
      auto go = [&](auto kern) {
        XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<static_cast<unsigned>(count), NT, smem, st>>>(din.ptr, static_cast<int>(n1), static_cast<int>(n2),
                                                             static_cast<int>(n3));
      };
      switch (rch_for(R)) {
        case 4: go(als_kernel<4>); break;
        case 8: go(als_kernel<8>); break;
        case 10: go(als_kernel<10>); break;
        case 12: go(als_kernel<12>); break;
        default: go(als_kernel<16>); break;
      }
      XLAUNCH_CHECK();
    }
    oa.finish();
    ob.finish();
    oc.finish();
    oh.finish();
    oi.finish();
    ov.finish();
  });
}

int32_t xtsg_relative_error(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* a, const double* b,
                            const double* c, int64_t rank, double* out) {
  return guard([&] {
    if (rank < 1) usage("relative_error: rank must be >= 1");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> tt(t, static_cast<size_t>(n1 * n2 * n3), st);
    InView<double> aa(a, static_cast<size_t>(n1 * rank), st), bb(b, static_cast<size_t>(n2 * rank), st),
        cc(c, static_cast<size_t>(n3 * rank), st);
    OutView<double> o(out, 1, st);
    const size_t smem = sizeof(double) * (static_cast<size_t>(n1 + n2 + n3) * rank + 64);
    XCUDA(cudaFuncSetAttribute(relerr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    relerr_kernel<<<1, NT, smem, st>>>(tt.dev, static_cast<int>(n1), static_cast<int>(n2), static_cast<int>(n3),
                                       aa.dev, bb.dev, cc.dev, static_cast<int>(rank), o.dev);
    XLAUNCH_CHECK();
    o.finish();
  });
}

}  // extern "C"
