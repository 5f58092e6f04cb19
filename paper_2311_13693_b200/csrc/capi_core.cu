// C ABI entry points: runtime, ensembles and the fp64 compression path.
// Each function cites the reference function it replaces; see include/xtsg.h.
#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "comp_f64.cuh"
#include "ensemble.cuh"
#include "gemm_simt.cuh"
#include "xrng.cuh"

namespace xtsg {

ErrState& err_state() {
  thread_local ErrState s;
  return s;
}

std::atomic<int64_t>& launch_counter() {
  thread_local std::atomic<int64_t> c{0};
  return c;
}

cudaStream_t thread_stream() {
  struct Holder {
    cudaStream_t s = nullptr;
    int dev = -1;
    ~Holder() {
      if (s) cudaStreamDestroy(s);
    }
  };
  thread_local Holder h;
  int dev = 0;
  XCUDA(cudaGetDevice(&dev));
  if (!h.s || h.dev != dev) {
    XCUDA(cudaStreamCreateWithFlags(&h.s, cudaStreamNonBlocking));
    h.dev = dev;
  }
  return h.s;
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Status(XTSG_E_CUDA, "no CUDA device available (xtsg has no CPU fallback)");
  }
  int dev = 0, major = 0;
  XCUDA(cudaGetDevice(&dev));
  XCUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw Status(XTSG_E_CUDA, "xtsg is built for sm_100a (B200) only");
  // stream-ordered allocations (DevBuf) stay mapped in the device's default
  // pool across synchronizations instead of being unmapped and remapped on
  // every call (multi-GB slab buffers otherwise cost ~100 ms per call)
  static thread_local int pool_dev = -1;
  if (pool_dev != dev) {
    cudaMemPool_t pool;
    XCUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    XCUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    pool_dev = dev;
  }
}

PhaseTrace::PhaseTrace(const char* n, cudaStream_t s) : name(n), st(s) {
  const char* e = std::getenv("XTSG_TRACE");
  on = e && std::atoi(e) != 0;
  if (on) mark("begin");
}

void PhaseTrace::mark(const char* label) {
  if (!on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  ev.emplace_back(label, e);
  host.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
}

PhaseTrace::~PhaseTrace() {
  if (!on) return;
  mark("end");
  cudaEventSynchronize(ev.back().second);
  std::string out = std::string("[xtsg trace] ") + name + ":";
  for (size_t q = 1; q < ev.size(); ++q) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[q - 1].second, ev[q].second);
    char buf[160];
    std::snprintf(buf, sizeof(buf), " %s %.2f/%.2f", ev[q].first, ms, host[q] - host[q - 1]);
    out += buf;
  }
  std::fprintf(stderr, "%s (device/host ms)\n", out.c_str());
  for (auto& e : ev) cudaEventDestroy(e.second);
}

int sm_count() {
  int dev = 0, n = 0;
  XCUDA(cudaGetDevice(&dev));
  XCUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

namespace {

// Generates one mode's P matrices in the reference layout (P back-to-back
// column-major rows x cols fp64) on the device.
void gen_mode_f64(int64_t rows, int64_t cols, int64_t count, int64_t shared_rows, int32_t kind,
                  double s, uint64_t shared_seed, uint64_t seed, uint64_t tag, double* out,
                  cudaStream_t st) {
  RowJob job{};
  job.rows = rows; job.cols = cols; job.shared_rows = shared_rows;
  job.kind = kind; job.s = s;
  job.shared_seed = shared_seed; job.seed = seed; job.mode_tag = tag; job.p_offset = 0;
  job.stride_p = rows * cols; job.stride_r = 1; job.stride_c = rows;
  launch_mode_rows<double>(job, count, out, st);
}

}  // namespace

}  // namespace xtsg

using namespace xtsg;

extern "C" {

const char* xtsg_last_error(void) { return err_state().msg.c_str(); }
int64_t xtsg_last_payload(int32_t which) { return which == 0 ? err_state().p0 : err_state().p1; }
int32_t xtsg_version(void) { return 100; }
int64_t xtsg_launch_count(void) { return launch_counter().load(); }

int32_t xtsg_device_ready(void) {
  return guard([] { require_device(); }) == XTSG_OK ? 1 : 0;
}

int32_t xtsg_warmup(void) {
  return guard([] {
    require_device();
    XCUDA(cudaFree(nullptr));
    (void)thread_stream();
  });
}

int32_t xtsg_replica_count(const int64_t dims[3], const int64_t reduced[3], int64_t slack,
                           int64_t* out) {
  // compression.cpp:82-95 (host arithmetic, no device needed)
  return guard([&] {
    for (int m = 0; m < 3; ++m) {
      if (reduced[m] < 3) usage("compute_replica_count: reduced dims must be >= 3");
      if (reduced[m] > dims[m]) usage("compute_replica_count: reduced dim exceeds original");
    }
    if (slack < 0) usage("compute_replica_count: slack must be >= 0");
    const int64_t bound = std::max({ceil_div(dims[0] - 2, reduced[0] - 2), ceil_div(dims[1], reduced[1]),
                                    ceil_div(dims[2], reduced[2])});
    *out = bound + slack;
  });
}

int32_t xtsg_gen_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  // compression.cpp:97-103
  return guard([&] {
    if (rows < 1 || cols < 1) usage("gen_gaussian: dims must be >= 1");
    require_device();
    cudaStream_t st = thread_stream();
    OutView<double> o(out, static_cast<size_t>(rows * cols), st);
    launch_stream_normals(seed, rows * cols, o.dev, st);
    o.finish();
  });
}

int32_t xtsg_gen_sparse_projection(int64_t rows, int64_t cols, double s, uint64_t seed,
                                   double* out) {
  // compression.cpp:105-113
  return guard([&] {
    if (rows < 1 || cols < 1) usage("gen_sparse_projection: dims must be >= 1");
    check_sparse_spec(s, cols);
    require_device();
    cudaStream_t st = thread_stream();
    OutView<double> o(out, static_cast<size_t>(rows * cols), st);
    launch_stream_sparse(seed, rows * cols, s, o.dev, st);
    o.finish();
  });
}

int32_t xtsg_make_ensemble(const int64_t dims[3], const int64_t reduced[3], int64_t count,
                           int64_t shared_rows, const xtsg_ensemble_spec* spec, uint64_t seed,
                           double* u, double* v, double* w, double* inner_u, double* inner_v,
                           double* inner_w, double* outer_u, double* outer_v,
                           double* outer_w) {
  // compression.cpp:115-200
  return guard([&] {
    const xtsg_ensemble_spec sp = *spec;
    const EnsembleShape sh = validate_ensemble(dims, reduced, count, shared_rows, sp);
    require_device();
    cudaStream_t st = thread_stream();
    const uint64_t shared_seed[3] = {derive(seed, 101), derive(seed, 102), derive(seed, 103)};
    double* outs[3] = {u, v, w};
    if (sp.kind != XTSG_KIND_TWO_STAGE) {
      for (int m = 0; m < 3; ++m) {
        OutView<double> o(outs[m], static_cast<size_t>(count * reduced[m] * dims[m]), st);
        gen_mode_f64(reduced[m], dims[m], count, shared_rows, sp.kind, sp.s, shared_seed[m], seed,
                     static_cast<uint64_t>(m), o.dev, st);
        o.finish();
      }
      return;
    }
    double* inners[3] = {inner_u, inner_v, inner_w};
    double* outers[3] = {outer_u, outer_v, outer_w};
    for (int m = 0; m < 3; ++m) {
      const int64_t ir = sh.inner[m];
      DevBuf<double> inner(static_cast<size_t>(ir * dims[m]), st);
      DevBuf<double> outer(static_cast<size_t>(count * reduced[m] * ir), st);
      const uint64_t tag_seed = derive(seed, 201 + static_cast<uint64_t>(m));
      if (sp.inner_kind == XTSG_KIND_SPARSE)
        launch_stream_sparse(tag_seed, ir * dims[m], sp.inner_s, inner.ptr, st);
      else
        launch_stream_normals(tag_seed, ir * dims[m], inner.ptr, st);
      gen_mode_f64(reduced[m], ir, count, shared_rows, XTSG_KIND_GAUSSIAN, 1.0, shared_seed[m], seed,
                   static_cast<uint64_t>(m), outer.ptr, st);
      OutView<double> o(outs[m], static_cast<size_t>(count * reduced[m] * dims[m]), st);
      GemmArgs<double> g;  // u[p] = outer[p] * inner (:190-194)
      g.m = reduced[m]; g.n = dims[m]; g.k = ir; g.batch = count;
      g.a = outer.ptr; g.lda = reduced[m]; g.stride_a = reduced[m] * ir;
      g.b = inner.ptr; g.ldb = ir; g.stride_b = 0;
      g.c = o.dev; g.ldc = reduced[m]; g.stride_c = reduced[m] * dims[m];
      gemm_simt(g, st);
      if (inners[m])
        XCUDA(cudaMemcpyAsync(inners[m], inner.ptr, sizeof(double) * ir * dims[m], cudaMemcpyDefault, st));
      if (outers[m])
        XCUDA(cudaMemcpyAsync(outers[m], outer.ptr, sizeof(double) * count * reduced[m] * ir,
                              cudaMemcpyDefault, st));
      o.finish();
    }
  });
}

int32_t xtsg_comp(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                  const double* v, int64_t m, const double* w, int64_t n, double* y) {
  // compression.cpp:202-213
  return guard([&] {
    if (n1 < 0 || n2 < 0 || n3 < 0 || l < 0 || m < 0 || n < 0) usage("comp: negative dimension");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> tt(t, static_cast<size_t>(n1 * n2 * n3), st);
    InView<double> uu(u, static_cast<size_t>(l * n1), st), vv(v, static_cast<size_t>(m * n2), st),
        ww(w, static_cast<size_t>(n * n3), st);
    OutView<double> o(y, static_cast<size_t>(l * m * n), st);
    if (l * m * n > 0) {
      if (n1 * n2 * n3 == 0)
        XCUDA(cudaMemsetAsync(o.dev, 0, sizeof(double) * l * m * n, st));
      else
        comp_f64_dev(tt.dev, n1, n2, n3, uu.dev, l, l, vv.dev, m, m, ww.dev, n, n, o.dev, 0.0, st);
    }
    o.finish();
  });
}

int32_t xtsg_reconstruct(const double* a, const double* b, const double* c, int64_t i, int64_t j,
                         int64_t k, int64_t rank, double* out) {
  // tensor.cpp:133-150
  return guard([&] {
    if (rank < 1) usage("reconstruct: rank must be >= 1");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> aa(a, static_cast<size_t>(i * rank), st), bb(b, static_cast<size_t>(j * rank), st),
        cc(c, static_cast<size_t>(k * rank), st);
    OutView<double> o(out, static_cast<size_t>(i * j * k), st);
    reconstruct_dev(aa.dev, bb.dev, cc.dev, i, j, k, rank, o.dev, st);
    o.finish();
  });
}

int32_t xtsg_comp_from_factors(const double* a, const double* b, const double* c, int64_t i,
                               int64_t j, int64_t k, int64_t rank, const double* u, int64_t l,
                               const double* v, int64_t m, const double* w, int64_t n,
                               double* y) {
  // compression.cpp:215-220
  return guard([&] {
    if (rank < 1) usage("reconstruct: rank must be >= 1");
    require_device();
    cudaStream_t st = thread_stream();
    InView<double> aa(a, static_cast<size_t>(i * rank), st), bb(b, static_cast<size_t>(j * rank), st),
        cc(c, static_cast<size_t>(k * rank), st);
    InView<double> uu(u, static_cast<size_t>(l * i), st), vv(v, static_cast<size_t>(m * j), st),
        ww(w, static_cast<size_t>(n * k), st);
    OutView<double> o(y, static_cast<size_t>(l * m * n), st);
    comp_from_factors_dev(aa.dev, bb.dev, cc.dev, i, j, k, rank, uu.dev, l, vv.dev, m, ww.dev, n, o.dev,
                          st);
    o.finish();
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// comp_blocked (compression.cpp:332-404) as a push stream.

struct xtsg_blocked {
  int64_t dims[3], block[3], cells[3], count, red[3];
  bool deterministic;
  cudaStream_t st;
  DevBuf<double> u, v, w;          // ensemble, P matrices back to back
  DevBuf<double> assembled;        // deterministic mode
  DevBuf<double> acc;              // fast mode: P replicas, fp64
  DevBuf<double> blockbuf;
  std::vector<char> seen;
  int64_t seen_count = 0;
};

namespace blocked_detail {

int64_t extent_len(const xtsg_blocked* h, int mode, int64_t cell, int64_t* offset) {
  *offset = cell * h->block[mode];
  return std::min(h->block[mode], h->dims[mode] - *offset);
}

__global__ void scatter_block_kernel(const double* __restrict__ src, int64_t b1, int64_t b2,
                                     int64_t b3, double* __restrict__ dst, int64_t n1, int64_t n2,
                                     int64_t o1, int64_t o2, int64_t o3) {
  const int64_t total = b1 * b2 * b3;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % b1, jk = e / b1, j = jk % b2, k = jk / b2;
    dst[(o1 + i) + n1 * ((o2 + j) + n2 * (o3 + k))] = src[e];
  }
}

}  // namespace blocked_detail
using namespace blocked_detail;

extern "C" {

int32_t xtsg_blocked_begin(const int64_t dims[3], const int64_t block[3], int64_t count,
                           const int64_t reduced[3], const double* u, const double* v,
                           const double* w, int32_t deterministic, xtsg_blocked** out) {
  return guard([&] {
    *out = nullptr;
    // BlockGrid ctor (compression.cpp:222-230)
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1) usage("BlockGrid: dims must be >= 1");
    if (block[0] < 1 || block[1] < 1 || block[2] < 1) usage("BlockGrid: block dims must be >= 1");
    if (block[0] > dims[0] || block[1] > dims[1] || block[2] > dims[2])
      usage("BlockGrid: block dims exceed tensor dims");
    if (count < 1) usage("comp_blocked: ensemble is empty");
    require_device();
    auto* h = new xtsg_blocked();
    try {
      h->st = thread_stream();
      for (int m = 0; m < 3; ++m) {
        h->dims[m] = dims[m];
        h->block[m] = block[m];
        h->cells[m] = ceil_div(dims[m], block[m]);
        h->red[m] = reduced[m];
      }
      h->count = count;
      h->deterministic = deterministic != 0;
      const double* src[3] = {u, v, w};
      DevBuf<double>* dst[3] = {&h->u, &h->v, &h->w};
      for (int m = 0; m < 3; ++m) {
        const size_t sz = static_cast<size_t>(count * reduced[m] * dims[m]);
        *dst[m] = DevBuf<double>(sz, h->st);
        XCUDA(cudaMemcpyAsync(dst[m]->ptr, src[m], sz * sizeof(double), cudaMemcpyDefault, h->st));
      }
      h->seen.assign(static_cast<size_t>(h->cells[0] * h->cells[1] * h->cells[2]), 0);
      if (h->deterministic) {
        h->assembled = DevBuf<double>(static_cast<size_t>(dims[0] * dims[1] * dims[2]), h->st);
      } else {
        h->acc = DevBuf<double>(static_cast<size_t>(count * reduced[0] * reduced[1] * reduced[2]), h->st);
        h->acc.zero();
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int32_t xtsg_blocked_push(xtsg_blocked* h, const int64_t cell[3], const int64_t shape[3],
                          const double* data) {
  return guard([&] {
    // validate_record (compression.cpp:319-328) and duplicate check (:344-351)
    int64_t off[3], len[3];
    for (int m = 0; m < 3; ++m) {
      if (cell[m] < 0 || cell[m] >= h->cells[m]) data_error("comp_blocked: block cell index out of range");
      len[m] = extent_len(h, m, cell[m], &off[m]);
    }
    if (shape[0] != len[0] || shape[1] != len[1] || shape[2] != len[2])
      data_error("comp_blocked: block shape does not match its cell");
    const int64_t linear = cell[0] + h->cells[0] * (cell[1] + h->cells[1] * cell[2]);
    if (h->seen[static_cast<size_t>(linear)])
      data_error("comp_blocked: duplicate block for cell " + std::to_string(linear));
    h->seen[static_cast<size_t>(linear)] = 1;
    ++h->seen_count;
    const size_t bsz = static_cast<size_t>(len[0] * len[1] * len[2]);
    InView<double> blk(data, bsz, h->st);
    if (h->deterministic) {
      const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(static_cast<int64_t>(bsz), 256), 4096));
      scatter_block_kernel<<<blocks, 256, 0, h->st>>>(blk.dev, len[0], len[1], len[2], h->assembled.ptr,
                                                       h->dims[0], h->dims[1], off[0], off[1], off[2]);
      XLAUNCH_CHECK();
    } else {
      const int64_t L = h->red[0], M = h->red[1], N = h->red[2];
      for (int64_t p = 0; p < h->count; ++p) {
        const double* up = h->u.ptr + p * L * h->dims[0] + off[0] * L;
        const double* vp = h->v.ptr + p * M * h->dims[1] + off[1] * M;
        const double* wp = h->w.ptr + p * N * h->dims[2] + off[2] * N;
        comp_f64_dev(blk.dev, len[0], len[1], len[2], up, L, L, vp, M, M, wp, N, N,
                     h->acc.ptr + p * L * M * N, 1.0, h->st);
      }
    }
    XCUDA(cudaStreamSynchronize(h->st));
  });
}

int32_t xtsg_blocked_push_region(xtsg_blocked* h, const int64_t offset[3], const int64_t shape[3],
                                 const double* data) {
  return guard([&] {
    int64_t c0[3], c1[3];
    for (int m = 0; m < 3; ++m) {
      const int64_t end = offset[m] + shape[m];
      if (offset[m] < 0 || shape[m] < 1 || end > h->dims[m]) data_error("comp_blocked: region outside the tensor");
      if (offset[m] % h->block[m] || (end % h->block[m] && end != h->dims[m]))
        data_error("comp_blocked: region not aligned to the block grid");
      c0[m] = offset[m] / h->block[m];
      c1[m] = ceil_div(end, h->block[m]);
    }
    for (int64_t k = c0[2]; k < c1[2]; ++k)
      for (int64_t j = c0[1]; j < c1[1]; ++j)
        for (int64_t i = c0[0]; i < c1[0]; ++i) {
          const int64_t linear = i + h->cells[0] * (j + h->cells[1] * k);
          if (h->seen[static_cast<size_t>(linear)])
            data_error("comp_blocked: duplicate block for cell " + std::to_string(linear));
          h->seen[static_cast<size_t>(linear)] = 1;
          ++h->seen_count;
        }
    const size_t bsz = static_cast<size_t>(shape[0] * shape[1] * shape[2]);
    if (!h->deterministic) {
      // fast mode: the region is compressed like one block (the sum of its
      // cells' contributions, fp64 accumulators)
      InView<double> blk(data, bsz, h->st);
      const int64_t L = h->red[0], M = h->red[1], N = h->red[2];
      for (int64_t p = 0; p < h->count; ++p)
        comp_f64_dev(blk.dev, shape[0], shape[1], shape[2], h->u.ptr + p * L * h->dims[0] + offset[0] * L, L, L,
                     h->v.ptr + p * M * h->dims[1] + offset[1] * M, M, M,
                     h->w.ptr + p * N * h->dims[2] + offset[2] * N, N, N, h->acc.ptr + p * L * M * N, 1.0, h->st);
    } else if (shape[0] == h->dims[0] && shape[1] == h->dims[1] && shape[2] == h->dims[2]) {
      XCUDA(cudaMemcpyAsync(h->assembled.ptr, data, bsz * sizeof(double), cudaMemcpyDefault, h->st));
    } else {
      InView<double> blk(data, bsz, h->st);
      const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(static_cast<int64_t>(bsz), 256), 4096));
      scatter_block_kernel<<<blocks, 256, 0, h->st>>>(blk.dev, shape[0], shape[1], shape[2], h->assembled.ptr,
                                                       h->dims[0], h->dims[1], offset[0], offset[1], offset[2]);
      XLAUNCH_CHECK();
    }
    XCUDA(cudaStreamSynchronize(h->st));
  });
}

int32_t xtsg_blocked_finish(xtsg_blocked* h, double* y) {
  return guard([&] {
    const int64_t total = h->cells[0] * h->cells[1] * h->cells[2];
    if (h->seen_count != total)
      data_error("comp_blocked: missing blocks (" + std::to_string(h->seen_count) + " of " +
                 std::to_string(total) + ")");
    const int64_t L = h->red[0], M = h->red[1], N = h->red[2];
    OutView<double> o(y, static_cast<size_t>(h->count * L * M * N), h->st);
    if (h->deterministic) {
      for (int64_t p = 0; p < h->count; ++p)
        comp_f64_dev(h->assembled.ptr, h->dims[0], h->dims[1], h->dims[2], h->u.ptr + p * L * h->dims[0], L, L,
                     h->v.ptr + p * M * h->dims[1], M, M, h->w.ptr + p * N * h->dims[2], N, N,
                     o.dev + p * L * M * N, 0.0, h->st);
    } else {
      XCUDA(cudaMemcpyAsync(o.dev, h->acc.ptr, sizeof(double) * h->count * L * M * N,
                            cudaMemcpyDeviceToDevice, h->st));
    }
    o.finish();
  });
}

void xtsg_blocked_destroy(xtsg_blocked* h) {
  if (!h) return;
  cudaStreamSynchronize(h->st);
  delete h;
}

}  // extern "C"

namespace xtsg {
void set_host_error(const std::string& msg, int64_t p0, int64_t p1) { err_state() = {msg, p0, p1}; }
}  // namespace xtsg
