// C ABI entry points of the precision model (half.hpp, mixed.hpp): device
// replays of the reference's binary16 splits and half_gemm products,
// bit-identical to the reference (see mixed.cu).
#include "common.cuh"
#include "mixed.cuh"

using namespace xtsg;

extern "C" {

int32_t xtsg_split_half(const double* x, int64_t n, int32_t mode, double* half, double* residual) {
  // round_matrix_to_half / round_tensor_to_half (mixed.cpp:47-61), fp16_split(_stored)
  // over split_matrix / split_tensor (mixed.cpp:11-45)
  return guard([&] {
    if (n < 0) usage("split: negative size");
    if (mode < 0 || mode > 2) usage("split: mode must be 0 (round), 1 (split) or 2 (stored split)");
    if (n == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> xx(x, static_cast<size_t>(n), st);
    OutView<double> h(half, static_cast<size_t>(n), st);
    OutView<double> r(mode ? residual : nullptr, static_cast<size_t>(n), st);
    split_dev(xx.dev, n, mode, h.dev, r.dev, st);
    h.finish();
    if (mode) r.finish();
  });
}

int32_t xtsg_half_gemm(const double* a, int64_t rows, int64_t inner, const double* b, int64_t b_rows,
                       int64_t cols, double* out) {
  // half_gemm (mixed.cpp:63-76)
  return guard([&] {
    if (inner != b_rows) usage("half_gemm: inner dimensions differ");
    if (rows < 0 || inner < 0 || cols < 0) usage("half_gemm: negative dimension");
    if (rows * cols == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> aa(a, static_cast<size_t>(rows * inner), st), bb(b, static_cast<size_t>(inner * cols), st);
    OutView<double> o(out, static_cast<size_t>(rows * cols), st);
    half_gemm_dev(aa.dev, rows, inner, bb.dev, cols, o.dev, st);
    o.finish();
  });
}

int32_t xtsg_comp_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                       const double* v, int64_t m, const double* w, int64_t n, double* y) {
  // comp_with(t, u, v, w, &half_gemm) (compression.cpp:202-209, mixed.cpp:84-86)
  return guard([&] {
    if (n1 < 0 || n2 < 0 || n3 < 0 || l < 0 || m < 0 || n < 0) usage("comp: negative dimension");
    if (l * m * n == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> tt(t, static_cast<size_t>(n1 * n2 * n3), st);
    InView<double> uu(u, static_cast<size_t>(l * n1), st), vv(v, static_cast<size_t>(m * n2), st),
        ww(w, static_cast<size_t>(n * n3), st);
    OutView<double> o(y, static_cast<size_t>(l * m * n), st);
    comp_half_dev(tt.dev, n1, n2, n3, uu.dev, l, vv.dev, m, ww.dev, n, o.dev, st);
    o.finish();
  });
}

int32_t xtsg_comp_mixed(const double* t_half, const double* t_res, int64_t n1, int64_t n2, int64_t n3,
                        const double* u_half, const double* u_res, int64_t l, const double* v_half,
                        const double* v_res, int64_t m, const double* w_half, const double* w_res,
                        int64_t n, double* y) {
  // comp_mixed (mixed.cpp:88-98)
  return guard([&] {
    if (n1 < 0 || n2 < 0 || n3 < 0 || l < 0 || m < 0 || n < 0) usage("comp: negative dimension");
    if (l * m * n == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    const size_t nt = static_cast<size_t>(n1 * n2 * n3);
    InView<double> th(t_half, nt, st), tr(t_res, nt, st);
    InView<double> uh(u_half, static_cast<size_t>(l * n1), st), ur(u_res, static_cast<size_t>(l * n1), st);
    InView<double> vh(v_half, static_cast<size_t>(m * n2), st), vr(v_res, static_cast<size_t>(m * n2), st);
    InView<double> wh(w_half, static_cast<size_t>(n * n3), st), wr(w_res, static_cast<size_t>(n * n3), st);
    OutView<double> o(y, static_cast<size_t>(l * m * n), st);
    comp_mixed_dev(th.dev, tr.dev, n1, n2, n3, uh.dev, ur.dev, l, vh.dev, vr.dev, m, wh.dev, wr.dev, n,
                   o.dev, st);
    o.finish();
  });
}

int32_t xtsg_comp_naive_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                             int64_t l, const double* v, int64_t m, const double* w, int64_t n,
                             double* y) {
  // comp_naive_half (mixed.cpp:100-104): every operand rounded to binary16, then comp_half
  return guard([&] {
    if (n1 < 0 || n2 < 0 || n3 < 0 || l < 0 || m < 0 || n < 0) usage("comp: negative dimension");
    require_device();
    cudaStream_t st = thread_stream();
    const size_t nt = static_cast<size_t>(n1 * n2 * n3);
    InView<double> tt(t, nt, st);
    InView<double> uu(u, static_cast<size_t>(l * n1), st), vv(v, static_cast<size_t>(m * n2), st),
        ww(w, static_cast<size_t>(n * n3), st);
    // the reference rounds t, u, v, w in this order (argument evaluation of
    // comp_half(...) is unspecified, but every rounding either throws the same
    // HalfRangeError or none does)
    DevBuf<double> th(nt, st), uh(static_cast<size_t>(l * n1), st), vh(static_cast<size_t>(m * n2), st),
        wh(static_cast<size_t>(n * n3), st);
    split_dev(tt.dev, static_cast<int64_t>(nt), 0, th.ptr, nullptr, st);
    split_dev(uu.dev, l * n1, 0, uh.ptr, nullptr, st);
    split_dev(vv.dev, m * n2, 0, vh.ptr, nullptr, st);
    split_dev(ww.dev, n * n3, 0, wh.ptr, nullptr, st);
    if (l * m * n == 0) return;
    OutView<double> o(y, static_cast<size_t>(l * m * n), st);
    comp_half_dev(th.ptr, n1, n2, n3, uh.ptr, l, vh.ptr, m, wh.ptr, n, o.dev, st);
    o.finish();
  });
}

}  // extern "C"
