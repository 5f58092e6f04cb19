// K8 — fp64 compression chain on the device (compatibility / drop-in path).
//
// comp_with (compression.cpp:202-209) evaluates Y = X x1 U x2 V x3 W as three
// successive mode products in the fixed order 1 -> 2 -> 3. The reference
// materialises matricize/fold copies (tensor.cpp:32-83) around each GEMM; here
// the unfoldings are expressed as strided GEMM views, so no copy is made:
//   mode 1: Y1 (L x J*K)        = U (L x I) * X(1) (I x J*K)
//   mode 2: Y2[:, :, k] (L x M) = Y1[:, :, k] (L x J) * V^T        (batched over k)
//   mode 3: Y (L*M x N)         = Y2 (L*M x K) * W^T
// Column slices of U/V/W (col_slice, :280-287) are pointer offsets with the
// original leading dimension, which is how blocked compression feeds them.
#include "comp_f64.cuh"
#include "common.cuh"
#include "gemm_simt.cuh"

namespace xtsg {

void comp_f64_dev(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                  int64_t ldu, int64_t l, const double* v, int64_t ldv, int64_t m,
                  const double* w, int64_t ldw, int64_t n, double* y, double beta,
                  cudaStream_t st) {
  DevBuf<double> y1(static_cast<size_t>(l * n2 * n3), st);
  DevBuf<double> y2(static_cast<size_t>(l * m * n3), st);
  GemmArgs<double> g1;
  g1.m = l; g1.n = n2 * n3; g1.k = n1;
  g1.a = u; g1.lda = ldu;
  g1.b = t; g1.ldb = n1;
  g1.c = y1.ptr; g1.ldc = l;
  gemm_simt(g1, st);
  GemmArgs<double> g2;
  g2.m = l; g2.n = m; g2.k = n2; g2.batch = n3;
  g2.a = y1.ptr; g2.lda = l; g2.stride_a = l * n2;
  g2.b = v; g2.ldb = ldv; g2.trans_b = true; g2.stride_b = 0;
  g2.c = y2.ptr; g2.ldc = l; g2.stride_c = l * m;
  gemm_simt(g2, st);
  GemmArgs<double> g3;
  g3.m = l * m; g3.n = n; g3.k = n3;
  g3.a = y2.ptr; g3.lda = l * m;
  g3.b = w; g3.ldb = ldw; g3.trans_b = true;
  g3.c = y; g3.ldc = l * m; g3.beta = beta;
  gemm_simt(g3, st);
}

namespace {

// reconstruct (tensor.cpp:133-150): t(i,j,k) = sum_r a(i,r) * (b(j,r) * c(k,r)),
// accumulated in increasing r with one rounding per product and per add,
// exactly as the reference's scalar loop (built without FMA contraction).
__global__ void reconstruct_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   const double* __restrict__ c, int64_t ni, int64_t nj,
                                   int64_t nk, int64_t rank, double* __restrict__ out) {
  const int64_t total = ni * nj * nk;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % ni;
    const int64_t jk = e / ni;
    const int64_t j = jk % nj;
    const int64_t k = jk / nj;
    double acc = 0.0;
    for (int64_t r = 0; r < rank; ++r) {
      const double s = __dmul_rn(b[j + nj * r], c[k + nk * r]);
      acc = __dadd_rn(acc, __dmul_rn(a[i + ni * r], s));
    }
    out[e] = acc;
  }
}

}  // namespace

void reconstruct_dev(const double* a, const double* b, const double* c, int64_t ni, int64_t nj,
                     int64_t nk, int64_t rank, double* out, cudaStream_t st) {
  const int64_t total = ni * nj * nk;
  if (total == 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 8 * 148 * 4));
  reconstruct_kernel<<<blocks, 256, 0, st>>>(a, b, c, ni, nj, nk, rank, out);
  XLAUNCH_CHECK();
}

void comp_from_factors_dev(const double* a, const double* b, const double* c, int64_t ni,
                           int64_t nj, int64_t nk, int64_t rank, const double* u, int64_t l,
                           const double* v, int64_t m, const double* w, int64_t n, double* y,
                           cudaStream_t st) {
  // compression.cpp:215-220: reconstruct(u*a, v*b, w*c)
  DevBuf<double> ua(static_cast<size_t>(l * rank), st), vb(static_cast<size_t>(m * rank), st),
      wc(static_cast<size_t>(n * rank), st);
  auto mul = [&](const double* lhs, int64_t rows, int64_t inner, const double* rhs, double* o) {
    GemmArgs<double> g;
    g.m = rows; g.n = rank; g.k = inner;
    g.a = lhs; g.lda = rows;
    g.b = rhs; g.ldb = inner;
    g.c = o; g.ldc = rows;
    gemm_simt(g, st);
  };
  mul(u, l, ni, a, ua.ptr);
  mul(v, m, nj, b, vb.ptr);
  mul(w, n, nk, c, wc.ptr);
  reconstruct_dev(ua.ptr, vb.ptr, wc.ptr, l, m, n, rank, y, st);
}

}  // namespace xtsg
