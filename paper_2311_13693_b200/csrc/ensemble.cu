// K1 — on-device generation of compression ensembles, bit-exact with the
// reference's make_ensemble (/root/reference/proj/src/compression.cpp:15-200).
//
// The reference fills every matrix row from its own splitmix64 stream
// (fill_row :40-46, gen_mode_matrices :51-72): row r of replica p draws from
// Rng(derive(r < S ? shared_seed : derive(seed, 1000 + 8p + tag), r)); anchor
// rows (r < S) are always Gaussian. Because splitmix64 is counter based, one
// warp evaluates 32 polar candidates of a row at once and compacts accepted
// pairs with a ballot + popc prefix, writing two normals per accepted pair in
// stream order. Sparse (three-point) rows need one output per entry and are
// embarrassingly parallel.
//
// Outputs are written through a strided "row sink" so the same generator
// feeds (a) the reference layout (column-major fp64 per replica) and (b) the
// tensor-core plan's operand layouts (row-major bf16 stacked U, transposed
// bf16 V, fp32 W) directly, without a conversion pass.
#include <cuda_bf16.h>

#include "common.cuh"
#include "ensemble.cuh"
#include "xrng.cuh"

namespace xtsg {

namespace {

template <class T>
__device__ __forceinline__ void store_val(T* p, double v);
template <>
__device__ __forceinline__ void store_val<double>(double* p, double v) { *p = v; }
template <>
__device__ __forceinline__ void store_val<float>(float* p, double v) { *p = static_cast<float>(v); }
template <>
__device__ __forceinline__ void store_val<__nv_bfloat16>(__nv_bfloat16* p, double v) {
  *p = __double2bfloat16(v);
}

// One warp per (replica, row). gridDim.y = replica count.
template <class T>
__global__ void mode_rows_kernel(RowJob job, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t p = blockIdx.y;
  if (row >= job.rows) return;
  const bool shared = row < job.shared_rows;
  const uint64_t base = shared ? job.shared_seed
                               : derive(job.seed, 1000 + 8 * static_cast<uint64_t>(p + job.p_offset) + job.mode_tag);
  const uint64_t rs = derive(base, static_cast<uint64_t>(row));
  T* dst = out + p * job.stride_p + row * job.stride_r;
  const int64_t cols = job.cols;
  if (!shared && job.kind == XTSG_KIND_SPARSE) {
    const double root = XSQRT(job.s);
    for (int64_t j = lane; j < cols; j += 32)
      store_val(dst + j * job.stride_c, three_point(stream_at(rs, static_cast<uint64_t>(j)), job.s, root));
    return;
  }
  int64_t produced = 0;
  uint64_t t0 = 0;
  while (produced < cols) {
    double n0 = 0.0, n1 = 0.0;
    const bool acc = polar_candidate(rs, t0 + lane, n0, n1);
    const unsigned mask = __ballot_sync(0xffffffffu, acc);
    const int64_t pos = produced + 2 * __popc(mask & ((1u << lane) - 1u));
    if (acc) {
      if (pos < cols) store_val(dst + pos * job.stride_c, n0);
      if (pos + 1 < cols) store_val(dst + (pos + 1) * job.stride_c, n1);
    }
    produced += 2 * __popc(mask);
    t0 += 32;
  }
}

// One block per whole-matrix stream (gen_gaussian :97-103 and the Gaussian
// factor generators): values are consecutive draws of a single Rng, stored in
// column-major order. Block-wide compaction of accepted candidates.
__global__ void stream_normals_kernel(uint64_t seed, int64_t n, double* __restrict__ out) {
  __shared__ int warp_cnt[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t produced = 0;
  uint64_t t0 = 0;
  while (produced < n) {
    double n0 = 0.0, n1 = 0.0;
    const bool acc = polar_candidate(seed, t0 + threadIdx.x, n0, n1);
    const unsigned mask = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) warp_cnt[wid] = __popc(mask);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      const int c = warp_cnt[w];
      if (w < wid) before += c;
      total += c;
    }
    before += __popc(mask & ((1u << lane) - 1u));
    const int64_t pos = produced + 2 * static_cast<int64_t>(before);
    if (acc) {
      if (pos < n) out[pos] = n0;
      if (pos + 1 < n) out[pos + 1] = n1;
    }
    produced += 2 * static_cast<int64_t>(total);
    t0 += blockDim.x;
    __syncthreads();
  }
}

// gen_sparse_projection (:105-113): entry idx (column-major) uses output idx.
__global__ void stream_sparse_kernel(uint64_t seed, int64_t n, double s, double* __restrict__ out) {
  const double root = XSQRT(s);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = three_point(stream_at(seed, static_cast<uint64_t>(i)), s, root);
}

}  // namespace

template <class T>
void launch_mode_rows(const RowJob& job, int64_t count, T* out, cudaStream_t st) {
  if (job.rows == 0 || count == 0 || job.cols == 0) return;
  constexpr int kWarps = 4;
  dim3 grid(static_cast<unsigned>(ceil_div(job.rows, kWarps)), static_cast<unsigned>(count));
  mode_rows_kernel<T><<<grid, kWarps * 32, 0, st>>>(job, out);
  XLAUNCH_CHECK();
}
template void launch_mode_rows<double>(const RowJob&, int64_t, double*, cudaStream_t);
template void launch_mode_rows<float>(const RowJob&, int64_t, float*, cudaStream_t);
template void launch_mode_rows<__nv_bfloat16>(const RowJob&, int64_t, __nv_bfloat16*, cudaStream_t);

void launch_stream_normals(uint64_t seed, int64_t n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  stream_normals_kernel<<<1, 1024, 0, st>>>(seed, n, out);
  XLAUNCH_CHECK();
}

void launch_stream_sparse(uint64_t seed, int64_t n, double s, double* out, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 4096));
  stream_sparse_kernel<<<blocks, 256, 0, st>>>(seed, n, s, out);
  XLAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Host-side validation shared by every ensemble consumer.

void check_sparse_spec(double s, int64_t cols) {
  // compression.cpp:27-38
  if (s < 1.0) usage("sparse projection: s must be >= 1");
  if (cols > 1) {
    const double bound = static_cast<double>(cols) / std::log(static_cast<double>(cols));
    if (s > bound)
      usage("sparse projection: s = " + std::to_string(s) +
            " exceeds the validity bound dim/log(dim) = " + std::to_string(bound));
  } else if (s != 1.0) {
    usage("sparse projection: s must be 1 for a single column");
  }
}

EnsembleShape validate_ensemble(const int64_t dims[3], const int64_t reduced[3], int64_t count,
                                int64_t shared_rows, const xtsg_ensemble_spec& spec) {
  // compression.cpp:119-128, :145-146, :157-169
  if (count < 1) usage("make_ensemble: count must be >= 1");
  if (shared_rows < 0) usage("make_ensemble: shared_rows must be >= 0");
  for (int m = 0; m < 3; ++m) {
    if (dims[m] < 1 || reduced[m] < 1) usage("make_ensemble: dims must be >= 1");
    if (reduced[m] > dims[m]) usage("make_ensemble: reduced dim exceeds original");
    if (shared_rows > reduced[m]) usage("make_ensemble: shared_rows exceeds reduced dim");
  }
  EnsembleShape sh{};
  for (int m = 0; m < 3; ++m) sh.inner[m] = dims[m];
  if (spec.kind == XTSG_KIND_SPARSE) {
    for (int m = 0; m < 3; ++m) check_sparse_spec(spec.s, dims[m]);
  } else if (spec.kind == XTSG_KIND_TWO_STAGE) {
    if (!(spec.alpha > 1.0 && spec.beta > 1.0 && spec.gamma > 1.0))
      usage("make_ensemble: two-stage ratios must be > 1");
    const double ratio[3] = {spec.alpha, spec.beta, spec.gamma};
    for (int m = 0; m < 3; ++m) {
      sh.inner[m] = static_cast<int64_t>(std::llround(ratio[m] * static_cast<double>(reduced[m])));
      if (sh.inner[m] <= reduced[m] || sh.inner[m] > dims[m])
        usage("make_ensemble: inner dimension out of range");
      if (spec.inner_kind == XTSG_KIND_SPARSE) check_sparse_spec(spec.inner_s, dims[m]);
    }
  } else if (spec.kind != XTSG_KIND_GAUSSIAN) {
    usage("make_ensemble: unknown ensemble kind");
  }
  return sh;
}

}  // namespace xtsg
