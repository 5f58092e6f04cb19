// K7 — sparse COO compression (no reference counterpart).
//
// Eq. 3 restricted to the nonzeros, duplicates summing:
//   Y_p = sum_nz x * U_p[:, i] (x) V_p[:, j] (x) W_p[:, k].
// Evaluated in the dense path's mode order on fibers:
//   1. sort the nonzeros by (k, j) (skipped when already sorted), run-length
//      encode the mode-3 slices;
//   2. one CTA per slice k: mode-1 per fiber (j, k) accumulates
//      y1 = sum_i x * Ustack[:, i] in fp32 registers — every warp owns a
//      disjoint range of stacked rows (p, l), so the gathers of the bf16 U
//      columns (i-major copy Ut[i][p*Lpad + l], 16-byte coalesced) are shared
//      by nothing and need no atomics — then folds mode 2 into a shared-memory
//      Z_p(k) += y1 (x) V_p[:, j] at every fiber change;
//   3. mode 3 over the distinct slices as one batched GEMM with the gathered
//      W columns, exactly like the dense path.
// The per-nonzero cost is one P*L gather + P*L FMAs, independent of the index
// space (10^6^3 in config C4), so the working set is the touched U columns.
#include <cub/cub.cuh>
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "plan.cuh"

namespace xtsg {

namespace {

constexpr int NT = 256;
constexpr int CHUNK = 256;

__global__ void coo_keys_kernel(const int32_t* __restrict__ jj, const int32_t* __restrict__ kk, int64_t nnz,
                                int64_t J, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                                int* __restrict__ bad, int64_t I, int64_t K, const int32_t* __restrict__ ii) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = ii[e], j = jj[e], k = kk[e];
    if (i < 0 || i >= I || j < 0 || j >= J || k < 0 || k >= K) *bad = 1;
    keys[e] = static_cast<uint64_t>(k) * static_cast<uint64_t>(J) + static_cast<uint64_t>(j);
    idx[e] = static_cast<uint32_t>(e);
  }
}

__global__ void unsorted_kernel(const uint64_t* keys, int64_t nnz, int* flag) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e + 1 < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (keys[e] > keys[e + 1]) *flag = 1;
}

__global__ void coo_gather_kernel(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                                  const int32_t* __restrict__ ii, const float* __restrict__ vv, int64_t nnz, int64_t J,
                                  int32_t* __restrict__ oi, int32_t* __restrict__ oj, int32_t* __restrict__ ok,
                                  float* __restrict__ ov) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = skeys[e];
    const uint32_t src = sidx[e];
    oi[e] = ii[src];
    ov[e] = vv[src];
    oj[e] = static_cast<int32_t>(key % static_cast<uint64_t>(J));
    ok[e] = static_cast<int32_t>(key / static_cast<uint64_t>(J));
  }
}

// Ustack [rows_u][ld_u] (row (p,l), i contiguous) -> Ut [I][plpad] (i-major)
__global__ void transpose_u_kernel(const __nv_bfloat16* __restrict__ u, int64_t rows, int64_t ld, int64_t I,
                                   __nv_bfloat16* __restrict__ ut) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    tile[dy][threadIdx.x] = (r < rows && c < I) ? u[r * ld + c] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < I) ut[c * rows + r] = tile[threadIdx.x][dy];
  }
}

// One CTA per slice (persistent). G stacked rows per pass (RPL per lane).
template <int RPL>
__global__ void __launch_bounds__(NT) coo_slice_kernel(
    const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, const float* __restrict__ cv,
    const int64_t* __restrict__ slice_off, const int32_t* __restrict__ slice_cnt, int64_t n_slices,
    const __nv_bfloat16* __restrict__ ut, int64_t plrows, const __nv_bfloat16* __restrict__ vt, int64_t ld_v,
    int mpad, int lpad, int64_t count, float* __restrict__ z) {
  constexpr int G = NT * RPL;  // stacked rows handled per pass
  extern __shared__ float zs[];  // G x mpad
  __shared__ int32_t s_i[CHUNK], s_j[CHUNK];
  __shared__ float s_v[CHUNK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = warp * (G / 8) + lane * RPL;  // rows of this lane within the pass
  for (int64_t s = blockIdx.x; s < n_slices; s += gridDim.x) {
    const int64_t b0 = slice_off[s], b1 = b0 + slice_cnt[s];
    for (int64_t g0 = 0; g0 < plrows; g0 += G) {
      for (int e = threadIdx.x; e < G * mpad; e += NT) zs[e] = 0.f;
      float y1[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) y1[q] = 0.f;
      int32_t cur_j = -1;
      auto flush = [&]() {
        if (cur_j < 0) return;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int64_t gr = g0 + row0 + q;
          if (gr < plrows && y1[q] != 0.f) {
            const int64_t p = gr / lpad;
            const __nv_bfloat16* vcol = vt + (p * mpad) * ld_v + cur_j;
            float* zr = zs + (row0 + q) * mpad;
            for (int m = 0; m < mpad; ++m) zr[m] = fmaf(y1[q], __bfloat162float(vcol[m * ld_v]), zr[m]);
          }
          y1[q] = 0.f;
        }
      };
      __syncthreads();
      for (int64_t c0 = b0; c0 < b1; c0 += CHUNK) {
        const int n = static_cast<int>(b1 - c0 < CHUNK ? b1 - c0 : CHUNK);
        if (threadIdx.x < n) {
          s_i[threadIdx.x] = ci[c0 + threadIdx.x];
          s_j[threadIdx.x] = cj[c0 + threadIdx.x];
          s_v[threadIdx.x] = cv[c0 + threadIdx.x];
        }
        __syncthreads();
        for (int e = 0; e < n; ++e) {
          const int32_t j = s_j[e];
          if (j != cur_j) {
            flush();
            cur_j = j;
          }
          const float x = s_v[e];
          const __nv_bfloat16* ucol = ut + static_cast<int64_t>(s_i[e]) * plrows + g0 + row0;
          if (g0 + row0 + RPL <= plrows) {
            if constexpr (RPL == 4) {
              const uint2 raw = *reinterpret_cast<const uint2*>(ucol);
              const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
              const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
              y1[0] = fmaf(x, __low2float(a), y1[0]);
              y1[1] = fmaf(x, __high2float(a), y1[1]);
              y1[2] = fmaf(x, __low2float(b), y1[2]);
              y1[3] = fmaf(x, __high2float(b), y1[3]);
            } else {
#pragma unroll
              for (int q = 0; q < RPL; ++q) y1[q] = fmaf(x, __bfloat162float(ucol[q]), y1[q]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < RPL; ++q)
              if (g0 + row0 + q < plrows) y1[q] = fmaf(x, __bfloat162float(ucol[q]), y1[q]);
          }
        }
        __syncthreads();
      }
      flush();
      __syncthreads();
      // Z[p][s][m][l] for the rows of this pass
      for (int e = threadIdx.x; e < G * mpad; e += NT) {
        const int r = e / mpad, m = e % mpad;
        const int64_t gr = g0 + r;
        if (gr >= plrows) continue;
        const int64_t p = gr / lpad, l = gr % lpad;
        if (p >= count) continue;
        z[((p * n_slices + s) * mpad + m) * lpad + l] = zs[e];
      }
      __syncthreads();
    }
  }
}

__global__ void gather_w_kernel(const float* __restrict__ wf, int64_t count, int64_t N, int64_t K,
                                const int32_t* __restrict__ uk, int64_t kd, float* __restrict__ wg) {
  const int64_t total = count * N * kd;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e % kd, pn = e / kd;
    wg[e] = wf[pn * K + uk[q]];
  }
}

__global__ void compact_y2_kernel(const float* __restrict__ ypad, int64_t count, int64_t L, int64_t M, int64_t N,
                                  int64_t lpad, int64_t mpad, int32_t accumulate, float* __restrict__ y) {
  const int64_t per = L * M * N, total = count * per;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / per, r = e % per;
    const int64_t l = r % L, mn = r / L, m = mn % M, n = mn / M;
    const float v = ypad[p * mpad * lpad * N + (m * lpad + l) + mpad * lpad * n];
    y[e] = accumulate ? y[e] + v : v;
  }
}

int gridn(int64_t work) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 16))); }

}  // namespace

void Plan::compress_coo(const int32_t* i, const int32_t* j, const int32_t* k, const float* val, int64_t nnz, float* y,
                        bool accumulate, cudaStream_t s) {
  if (desc.precision != XTSG_PREC_BF16) usage("plan_compress_coo: needs a bf16 (tensor-core) plan");
  if (nnz < 0) usage("plan_compress_coo: negative nnz");
  if (nnz >= (int64_t(1) << 32)) usage("plan_compress_coo: at most 2^32-1 nonzeros per call");
  if (stage1) {
    const int64_t ysz = desc.count * desc.reduced[0] * desc.reduced[1] * desc.reduced[2];
    OutView<float> yo(y, static_cast<size_t>(ysz), s);
    if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
    DevBuf<float> zin(static_cast<size_t>(inner_dims[0] * inner_dims[1] * inner_dims[2]), s);
    stage1->compress_coo(i, j, k, val, nnz, zin.ptr, false, s);
    stage2(zin.ptr, yo.dev, accumulate, s);
    if (yo.host) yo.finish();
    return;
  }
  const int64_t I = desc.dims[0], J = desc.dims[1], K = desc.dims[2];
  const int64_t L = desc.reduced[0], M = desc.reduced[1], N = desc.reduced[2], P = desc.count;
  const int64_t ysz = P * L * M * N;
  const bool padded = (lpad != L) || (mpad != M);
  OutView<float> yo(y, static_cast<size_t>(ysz), s);
  if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
  if (nnz == 0) {
    if (!accumulate) XCUDA(cudaMemsetAsync(yo.dev, 0, ysz * 4, s));
    if (yo.host) yo.finish();
    return;
  }
  const int64_t plrows = P * lpad;
  if (!ut.ptr) {
    ut = DevBuf<__nv_bfloat16>(static_cast<size_t>(I * plrows), s);
    dim3 grid(static_cast<unsigned>(ceil_div(I, 32)), static_cast<unsigned>(ceil_div(plrows, 32)));
    transpose_u_kernel<<<grid, dim3(32, 8), 0, s>>>(ustack.ptr, plrows, ld_u, I, ut.ptr);
    XLAUNCH_CHECK();
  }
  InView<int32_t> di(i, static_cast<size_t>(nnz), s), dj(j, static_cast<size_t>(nnz), s), dk(k, static_cast<size_t>(nnz), s);
  InView<float> dv(val, static_cast<size_t>(nnz), s);
  // 1. keys, validation, sortedness
  DevBuf<uint64_t> keys(static_cast<size_t>(nnz), s);
  DevBuf<uint32_t> idx(static_cast<size_t>(nnz), s);
  DevBuf<int> flags(2, s);
  flags.zero();
  coo_keys_kernel<<<gridn(nnz), 256, 0, s>>>(dj.dev, dk.dev, nnz, J, keys.ptr, idx.ptr, flags.ptr, I, K, di.dev);
  XLAUNCH_CHECK();
  unsorted_kernel<<<gridn(nnz), 256, 0, s>>>(keys.ptr, nnz, flags.ptr + 1);
  XLAUNCH_CHECK();
  int hf[2] = {0, 0};
  XCUDA(cudaMemcpyAsync(hf, flags.ptr, sizeof(hf), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  if (hf[0]) data_error("plan_compress_coo: coordinate outside the tensor");
  const int32_t *si = di.dev, *sj = dj.dev, *sk = dk.dev;
  const float* sv = dv.dev;
  DevBuf<int32_t> bi, bj, bk;
  DevBuf<float> bv;
  if (hf[1]) {
    DevBuf<uint64_t> keys2(static_cast<size_t>(nnz), s);
    DevBuf<uint32_t> idx2(static_cast<size_t>(nnz), s);
    size_t tmp_bytes = 0;
    int end_bit = 1;
    while (end_bit < 64 && (uint64_t(1) << end_bit) < static_cast<uint64_t>(K) * static_cast<uint64_t>(J)) ++end_bit;
    XCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.ptr, keys2.ptr, idx.ptr, idx2.ptr, nnz, 0, end_bit, s));
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    XCUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, keys.ptr, keys2.ptr, idx.ptr, idx2.ptr, nnz, 0, end_bit, s));
    count_launch();
    bi = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bj = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bk = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bv = DevBuf<float>(static_cast<size_t>(nnz), s);
    coo_gather_kernel<<<gridn(nnz), 256, 0, s>>>(keys2.ptr, idx2.ptr, di.dev, dv.dev, nnz, J, bi.ptr, bj.ptr, bk.ptr,
                                                  bv.ptr);
    XLAUNCH_CHECK();
    si = bi.ptr; sj = bj.ptr; sk = bk.ptr; sv = bv.ptr;
  }
  keys.release();
  idx.release();
  // 2. mode-3 slices: unique k + counts + offsets
  DevBuf<int32_t> uk(static_cast<size_t>(nnz), s), cnt(static_cast<size_t>(nnz), s);
  DevBuf<int64_t> nruns(1, s), off(static_cast<size_t>(nnz), s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, sk, uk.ptr, cnt.ptr, nruns.ptr, nnz, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, sk, uk.ptr, cnt.ptr, nruns.ptr, nnz, s));
    count_launch();
  }
  int64_t kd = 0;
  XCUDA(cudaMemcpyAsync(&kd, nruns.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  {
    size_t tb = 0;
    XCUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.ptr, off.ptr, kd, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, cnt.ptr, off.ptr, kd, s));
    count_launch();
  }
  // 3. fibers -> Z[p][kd][m][l]
  DevBuf<float> z(static_cast<size_t>(P * kd * mpad * lpad), s);
  const int rpl_max = mpad <= 32 ? 4 : mpad <= 64 ? 2 : 1;
  int rpl = 1;
  while (rpl < rpl_max && NT * rpl < plrows) rpl *= 2;
  const size_t smem = static_cast<size_t>(NT * rpl * mpad) * sizeof(float);
  const int grid = static_cast<int>(std::min<int64_t>(kd, sm_count() * 2));
  if (rpl == 4) {
    XCUDA(cudaFuncSetAttribute(coo_slice_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    coo_slice_kernel<4><<<grid, NT, smem, s>>>(si, sj, sv, off.ptr, cnt.ptr, kd, ut.ptr, plrows, vt.ptr, ld_v,
                                               static_cast<int>(mpad), static_cast<int>(lpad), P, z.ptr);
  } else if (rpl == 2) {
    XCUDA(cudaFuncSetAttribute(coo_slice_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    coo_slice_kernel<2><<<grid, NT, smem, s>>>(si, sj, sv, off.ptr, cnt.ptr, kd, ut.ptr, plrows, vt.ptr, ld_v,
                                               static_cast<int>(mpad), static_cast<int>(lpad), P, z.ptr);
  } else {
    XCUDA(cudaFuncSetAttribute(coo_slice_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    coo_slice_kernel<1><<<grid, NT, smem, s>>>(si, sj, sv, off.ptr, cnt.ptr, kd, ut.ptr, plrows, vt.ptr, ld_v,
                                               static_cast<int>(mpad), static_cast<int>(lpad), P, z.ptr);
  }
  XLAUNCH_CHECK();
  // 4. mode 3 over the distinct slices
  DevBuf<float> wg(static_cast<size_t>(P * N * kd), s);
  gather_w_kernel<<<gridn(P * N * kd), 256, 0, s>>>(wf.ptr, P, N, K, uk.ptr, kd, wg.ptr);
  XLAUNCH_CHECK();
  DevBuf<float> ypad;
  float* ydst = yo.dev;
  if (padded) {
    ypad = DevBuf<float>(static_cast<size_t>(P * mpad * lpad * N), s);
    ydst = ypad.ptr;
  }
  GemmArgs<float> g;
  g.m = mpad * lpad; g.n = N; g.k = kd; g.batch = P;
  g.a = z.ptr; g.lda = mpad * lpad; g.stride_a = kd * mpad * lpad;
  g.b = wg.ptr; g.ldb = kd; g.stride_b = N * kd;
  g.c = ydst; g.ldc = mpad * lpad; g.stride_c = mpad * lpad * N;
  g.beta = (accumulate && !padded) ? 1.f : 0.f;
  gemm_simt(g, s);
  if (padded) {
    compact_y2_kernel<<<gridn(ysz), 256, 0, s>>>(ypad.ptr, P, L, M, N, lpad, mpad, accumulate ? 1 : 0, yo.dev);
    XLAUNCH_CHECK();
  }
  if (yo.host) yo.finish();
}

}  // namespace xtsg

using namespace xtsg;

extern "C" int32_t xtsg_plan_compress_coo(xtsg_plan* plan, const int32_t* i, const int32_t* j, const int32_t* k,
                                          const float* val, int64_t nnz, void* y, int32_t accumulate, void* stream) {
  return guard([&] {
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : thread_stream();
    p->compress_coo(i, j, k, val, nnz, static_cast<float*>(y), accumulate != 0, s);
  });
}
