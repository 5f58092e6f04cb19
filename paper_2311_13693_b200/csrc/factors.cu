// K4 — compression of a tensor given by its CP factors, with the tensor
// blocks generated on the device (reference: comp_from_factors /
// make_memory_block_source over reconstruct(), compression.cpp:215-278,
// tensor.cpp:133-150).
//
// The 10^12-element configs must never exist in memory: mode-3 slabs of
// X = sum_r a_r (x) b_r (x) c_r are produced in bf16 by a register-tiled
// rank-R micro-GEMM (X_k = A diag(c_k) B^T, R FMAs per element) straight into
// the staging layout the fused tcgen05 TTM consumes, one slab at a time.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"
#include "sm100_ptx.cuh"

namespace xtsg {

namespace {

constexpr int TI = 128, TJ = 64, NT = 256;

// X[kk][j][i] (ld_i) = sum_r A[i,r] B[j,r] C[k0+kk,r]; A/B/C fp32 column-major.
// Compensated plans (X_lo != null): x scaled by 2^comp_x_shift(amax) (amax: an
// upper bound of |x| over the call, factor_bound_kernel), fp16 hi into X and
// lo = x - hi into X_lo.
__global__ void __launch_bounds__(NT) gen_slab_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                      const float* __restrict__ Cm, int64_t I, int64_t J, int64_t K,
                                                      int R, int64_t k0, int64_t ldi,
                                                      __nv_bfloat16* __restrict__ X, bool f16,
                                                      __nv_bfloat16* __restrict__ X_lo, const unsigned* __restrict__ amax) {
  extern __shared__ float sm[];
  float* As = sm;            // R x TI
  float* Bs = sm + R * TI;   // R x TJ (already scaled by c_k)
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TI, j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t kk = blockIdx.z, k = k0 + kk;
  for (int e = threadIdx.x; e < R * TI; e += NT) {
    const int r = e / TI, ii = e % TI;
    As[e] = (i0 + ii < I) ? A[(i0 + ii) + I * r] : 0.f;
  }
  for (int e = threadIdx.x; e < R * TJ; e += NT) {
    const int r = e / TJ, jj = e % TJ;
    Bs[e] = (j0 + jj < J) ? B[(j0 + jj) + J * r] * Cm[k + K * r] : 0.f;
  }
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 x 16 threads, 8 x 4 outputs each
  float acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (int r = 0; r < R; ++r) {
    float av[8], bv[4];
#pragma unroll
    for (int a = 0; a < 8; ++a) av[a] = As[r * TI + tx * 8 + a];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = Bs[r * TJ + ty + 16 * b];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
  }
  if (X_lo) {
    const float sc = ldexpf(1.f, comp_x_shift(amax));
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t j = j0 + ty + 16 * b;
      if (j >= J) continue;
      const int64_t o = (kk * J + j) * ldi + i0 + tx * 8;
      float v8[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) v8[a] = i0 + tx * 8 + a < I ? acc[a][b] * sc : 0.f;
      if (i0 + tx * 8 + 8 <= ldi) {
        uint32_t wh[4], wl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const __half2 h = __floats2half2_rn(v8[2 * q], v8[2 * q + 1]);
          const float2 hf = __half22float2(h);
          const __half2 l = __floats2half2_rn(v8[2 * q] - hf.x, v8[2 * q + 1] - hf.y);
          wh[q] = *reinterpret_cast<const uint32_t*>(&h);
          wl[q] = *reinterpret_cast<const uint32_t*>(&l);
        }
        *reinterpret_cast<uint4*>(X + o) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        *reinterpret_cast<uint4*>(X_lo + o) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
      } else {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          if (i0 + tx * 8 + a >= ldi) continue;
          const __half h = __float2half_rn(v8[a]);
          const __half l = __float2half_rn(v8[a] - __half2float(h));
          X[o + a] = __ushort_as_bfloat16(__half_as_ushort(h));
          X_lo[o + a] = __ushort_as_bfloat16(__half_as_ushort(l));
        }
      }
    }
    return;
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t j = j0 + ty + 16 * b;
    if (j >= J) continue;
    __nv_bfloat16* row = X + (kk * J + j) * ldi + i0 + tx * 8;
    if (i0 + tx * 8 + 8 <= I) {
      float v8[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) v8[a] = acc[a][b];
      *reinterpret_cast<uint4*>(row) = ptx::pack8(v8, f16);
    } else {
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (i0 + tx * 8 + a < ldi) {
          const float v = i0 + tx * 8 + a < I ? acc[a][b] : 0.f;
          row[a] = f16 ? __ushort_as_bfloat16(__half_as_ushort(__float2half_rn(v))) : __float2bfloat16(v);
        }
    }
  }
}

// |x_ijk| <= sum_r max_i |a_ir| max_j |b_jr| max_(k0 <= k < k1) |c_kr| (fp32
// factors), stored as float bits in both amax slots: the compensated split's
// scale for every slab of the call (one block)
__global__ void factor_bound_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                    const float* __restrict__ Cm, int64_t I, int64_t J, int64_t K, int R, int64_t k0,
                                    int64_t k1, unsigned* __restrict__ amax) {
  __shared__ float red[3][32];
  float total = 0.f;
  for (int r = 0; r < R; ++r) {
    float m[3] = {0.f, 0.f, 0.f};
    for (int64_t i = threadIdx.x; i < I; i += blockDim.x) m[0] = fmaxf(m[0], fabsf(A[i + I * r]));
    for (int64_t j = threadIdx.x; j < J; j += blockDim.x) m[1] = fmaxf(m[1], fabsf(B[j + J * r]));
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) m[2] = fmaxf(m[2], fabsf(Cm[k + K * r]));
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m[q] = fmaxf(m[q], __shfl_xor_sync(0xffffffffu, m[q], o));
      if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = m[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm[3] = {0.f, 0.f, 0.f};
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
        for (int q = 0; q < 3; ++q) mm[q] = fmaxf(mm[q], red[q][w]);
      total += mm[0] * mm[1] * mm[2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const unsigned bits = __float_as_uint(total * 1.0001f);  // the generator's fp32 sums round
    amax[0] = bits;
    amax[1] = bits;
  }
}

__global__ void to_f32_kernel(const double* __restrict__ s, int64_t n, float* __restrict__ d) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[e] = static_cast<float>(s[e]);
}

int g1(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 16))); }

}  // namespace

void Plan::compress_factors(const double* a, const double* b, const double* c, int64_t rank, int64_t k0, int64_t k1,
                            float* y, bool accumulate, cudaStream_t s) {
  if (!tensor_core()) usage("plan_compress_factors: needs a bf16/fp16 (tensor-core) plan");
  if (stage1) {
    const int64_t ysz = desc.count * desc.reduced[0] * desc.reduced[1] * desc.reduced[2];
    OutView<float> yo(y, static_cast<size_t>(ysz), s);
    if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
    DevBuf<float> zin(static_cast<size_t>(inner_dims[0] * inner_dims[1] * inner_dims[2]), s);
    stage1->compress_factors(a, b, c, rank, k0, k1, zin.ptr, false, s);
    stage2(zin.ptr, yo.dev, accumulate, s);
    if (yo.host) yo.finish();
    return;
  }
  const int64_t I = desc.dims[0], J = desc.dims[1], K = desc.dims[2];
  if (rank < 1 || rank > 64) usage("plan_compress_factors: rank must be in [1, 64]");
  if (k0 < 0 || k1 > K || k0 >= k1) usage("plan_compress_factors: k range outside the tensor");
  const int64_t L = desc.reduced[0], M = desc.reduced[1], N = desc.reduced[2], P = desc.count;
  const int64_t ysz = P * L * M * N;
  const bool padded = virt_padded();
  OutView<float> yo(y, static_cast<size_t>(ysz), s);
  if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
  InView<double> da(a, static_cast<size_t>(I * rank), s), db(b, static_cast<size_t>(J * rank), s),
      dc(c, static_cast<size_t>(K * rank), s);
  DevBuf<float> fa(static_cast<size_t>(I * rank), s), fb(static_cast<size_t>(J * rank), s),
      fc(static_cast<size_t>(K * rank), s);
  to_f32_kernel<<<g1(I * rank), 256, 0, s>>>(da.dev, I * rank, fa.ptr);
  to_f32_kernel<<<g1(J * rank), 256, 0, s>>>(db.dev, J * rank, fb.ptr);
  to_f32_kernel<<<g1(K * rank), 256, 0, s>>>(dc.dev, K * rank, fc.ptr);
  count_launch(2);
  XLAUNCH_CHECK();
  DevBuf<float> ypad;
  DevBuf<double> y64;
  float* ydst = yo.dev;
  bool acc = accumulate;
  if (comp()) {
    y64 = DevBuf<double>(static_cast<size_t>(vP * mpad * lpad * N), s);
    comp_y = y64.ptr;
    acc = false;
  } else if (padded) {
    ypad = DevBuf<float>(static_cast<size_t>(vP * mpad * lpad * N), s);
    ydst = ypad.ptr;
    acc = false;
  }
  const int64_t ldi = ceil_div(I, 8) * 8;
  // slab size: enough slices per TTM launch for many persistent waves (the
  // last wave's idle SMs amortized), within a quarter of the free HBM
  size_t free_b = 0, total_b = 0;
  XCUDA(cudaMemGetInfo(&free_b, &total_b));
  static const int64_t slab_gb = [] {
    const char* e = std::getenv("XTSG_SLAB_GB");
    return e && std::atoi(e) > 0 ? static_cast<int64_t>(std::atoi(e)) : int64_t(8);
  }();
  const int64_t budget = std::min<int64_t>(slab_gb << 30, static_cast<int64_t>(free_b / 4));
  const int64_t planes = comp() ? 2 : 1;
  const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(k1 - k0, budget / (planes * ldi * J * 2)));
  const size_t smem = static_cast<size_t>(rank) * (TI + TJ) * sizeof(float);
  XCUDA(cudaFuncSetAttribute(gen_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t nslabs = ceil_div(k1 - k0, ks);
  if (comp()) {
    factor_bound_kernel<<<1, 1024, 0, s>>>(fa.ptr, fb.ptr, fc.ptr, I, J, K, static_cast<int>(rank), k0, k1, amax.ptr);
    XLAUNCH_CHECK();
  }
  // Two slab buffers: the generator fills slab s+1 on the side stream while
  // the tensor cores consume slab s (the compensated mode's |x| bound sits in
  // both amax slots). XTSG_GEN_OVERLAP=0 disables.
  static const bool overlap_env = [] {
    const char* e = std::getenv("XTSG_GEN_OVERLAP");
    return !(e && std::atoi(e) == 0);
  }();
  const bool overlap = overlap_env && nslabs > 1;
  DevBuf<__nv_bfloat16> stage[2], stage_lo[2];
  for (int b = 0; b < (overlap ? 2 : 1); ++b) {
    stage[b] = DevBuf<__nv_bfloat16>(static_cast<size_t>(ks * J * ldi), s);
    if (comp()) stage_lo[b] = DevBuf<__nv_bfloat16>(static_cast<size_t>(ks * J * ldi), s);
  }
  auto gen = [&](int64_t sl, int b, cudaStream_t gs) {
    const int64_t kb = k0 + sl * ks, kn = std::min(ks, k1 - kb);
    dim3 grid(static_cast<unsigned>(ceil_div(I, TI)), static_cast<unsigned>(ceil_div(J, TJ)),
              static_cast<unsigned>(kn));
    gen_slab_kernel<<<grid, NT, smem, gs>>>(fa.ptr, fb.ptr, fc.ptr, I, J, K, static_cast<int>(rank), kb, ldi,
                                            stage[b].ptr, fp16(), comp() ? stage_lo[b].ptr : nullptr,
                                            comp() ? amax.ptr + b : nullptr);
    XLAUNCH_CHECK();
  };
  auto ttm = [&](int64_t sl, int b) {
    const int64_t kb = k0 + sl * ks, kn = std::min(ks, k1 - kb);
    const int64_t off[3] = {0, 0, kb}, ext[3] = {I, J, kn};
    cur_amax = comp() ? amax.ptr + b : nullptr;
    run_bf16_block(stage[b].ptr, ldi, ldi * J, off, ext, ydst, acc, s, comp() ? stage_lo[b].ptr : nullptr);
    cur_amax = nullptr;
    acc = true;
  };
  if (!overlap) {
    for (int64_t sl = 0; sl < nslabs; ++sl) {
      gen(sl, 0, s);
      ttm(sl, 0);
    }
  } else {
    for (int b = 0; b < 2; ++b) {
      if (!ev_copied[b]) XCUDA(cudaEventCreateWithFlags(&ev_copied[b], cudaEventDisableTiming));
      if (!ev_consumed[b]) XCUDA(cudaEventCreateWithFlags(&ev_consumed[b], cudaEventDisableTiming));
      XCUDA(cudaEventRecord(ev_consumed[b], s));  // both buffers free; the factors are on s
    }
    XCUDA(cudaStreamWaitEvent(copy_st, ev_consumed[0], 0));
    gen(0, 0, copy_st);
    XCUDA(cudaEventRecord(ev_copied[0], copy_st));
    for (int64_t sl = 0; sl < nslabs; ++sl) {
      const int b = static_cast<int>(sl & 1);
      if (sl + 1 < nslabs) {
        XCUDA(cudaStreamWaitEvent(copy_st, ev_consumed[1 - b], 0));
        gen(sl + 1, 1 - b, copy_st);
        XCUDA(cudaEventRecord(ev_copied[1 - b], copy_st));
      }
      XCUDA(cudaStreamWaitEvent(s, ev_copied[b], 0));
      ttm(sl, b);
      XCUDA(cudaEventRecord(ev_consumed[b], s));
    }
  }
  if (comp()) {
    comp_finish(y64.ptr, yo.dev, accumulate, s);
    comp_y = nullptr;
  } else if (padded) {
    compact(ypad.ptr, yo.dev, accumulate, s);
  }
  if (fp16() || comp()) check_finite16(yo.dev, ysz, s);
  if (yo.host) yo.finish();
}

}  // namespace xtsg

using namespace xtsg;

extern "C" int32_t xtsg_plan_compress_factors(xtsg_plan* plan, const double* a, const double* b, const double* c,
                                              int64_t rank, int64_t k0, int64_t k1, void* y, int32_t accumulate,
                                              void* stream) {
  return guard([&] {
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : thread_stream();
    PlanUse use(p, s);
    p->compress_factors(a, b, c, rank, k0, k1, static_cast<float*>(y), accumulate != 0, s);
  });
}
