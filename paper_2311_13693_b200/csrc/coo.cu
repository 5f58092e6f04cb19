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
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "plan.cuh"

namespace xtsg {

namespace {

constexpr int NT = 256;

__global__ void coo_keys_kernel(const int32_t* __restrict__ jj, const int32_t* __restrict__ kk, int64_t nnz,
                                int64_t J, uint64_t* __restrict__ keys, uint64_t* __restrict__ payload,
                                int* __restrict__ bad, int64_t I, int64_t K, const int32_t* __restrict__ ii,
                                const float* __restrict__ vv) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = ii[e], j = jj[e], k = kk[e];
    if (i < 0 || i >= I || j < 0 || j >= J || k < 0 || k >= K) *bad = 1;
    keys[e] = static_cast<uint64_t>(k) * static_cast<uint64_t>(J) + static_cast<uint64_t>(j);
    // the sort carries (i, value) with the key: no random gather afterwards
    payload[e] = (static_cast<uint64_t>(static_cast<uint32_t>(i)) << 32) | __float_as_uint(vv[e]);
  }
}

__global__ void unsorted_kernel(const uint64_t* keys, int64_t nnz, int* flag) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e + 1 < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (keys[e] > keys[e + 1]) *flag = 1;
}

// sorted (key, payload) -> SoA i, j, k, value (one streaming pass)
__global__ void coo_unpack_kernel(const uint64_t* __restrict__ skeys, const uint64_t* __restrict__ spay, int64_t nnz,
                                  int64_t J, int32_t* __restrict__ oi, int32_t* __restrict__ oj,
                                  int32_t* __restrict__ ok, float* __restrict__ ov) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = skeys[e], pl = spay[e];
    oi[e] = static_cast<int32_t>(pl >> 32);
    ov[e] = __uint_as_float(static_cast<uint32_t>(pl));
    oj[e] = static_cast<int32_t>(key % static_cast<uint64_t>(J));
    ok[e] = static_cast<int32_t>(key / static_cast<uint64_t>(J));
  }
}

// bf16 [rows][ld] (row-major, cols contiguous) -> [cols][ld_out] (transposed;
// rows <= ld_out, the caller zero-fills the padding). Builds the i-major U
// copy Ut[i][(p, l)] and the j-major V copy Vtj[j][(p, m)] of the sparse path.
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ u, int64_t rows, int64_t ld, int64_t cols,
                                      int64_t ld_out, __nv_bfloat16* __restrict__ ut) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    tile[dy][threadIdx.x] = (r < rows && c < cols) ? u[r * ld + c] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) ut[c * ld_out + r] = tile[threadIdx.x][dy];
  }
}

__device__ __forceinline__ void half8(const uint4& raw, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __half22float2(h[q]);
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
}

__device__ __forceinline__ void bf16x8(const uint4& raw, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __bfloat1622float2(h[q]);
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
}

// y[q] += x * u[q] for the 8 bf16 of u: sm_100's mixed-precision FMA
// (fma.rn.f32.bf16 -> FHFMA.BF16, half-select operands), no unpacking.
template <bool F16>
__device__ __forceinline__ void fma8(float* y, const uint4& u, uint16_t x) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if constexpr (F16)
      asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %2;\n fma.rn.f32.f16 %0, %3, lo, %0;\n"
          " fma.rn.f32.f16 %1, %3, hi, %1;\n}"
          : "+f"(y[2 * q]), "+f"(y[2 * q + 1])
          : "r"(w[q]), "h"(x));
    else
      asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %2;\n fma.rn.f32.bf16 %0, %3, lo, %0;\n"
          " fma.rn.f32.bf16 %1, %3, hi, %1;\n}"
          : "+f"(y[2 * q]), "+f"(y[2 * q + 1])
          : "r"(w[q]), "h"(x));
  }
}

// Warp-level segmented accumulation over the (k, j)-sorted nonzeros of a
// slice. A pass covers G = 256*C stacked rows (p, l); lane `lane` owns rows
// c*256 + lane*8 + t (t < 8) of it, so one nonzero is one 16-byte gather per
// row group from Ut[i] (the warp reads 512 contiguous bytes) and 8*C fp32
// FMAs. The 8 warps of a CTA take contiguous eighths of the slice's nonzeros
// (fibers may straddle: partial fibers simply fold separately) and run
// UNROLL nonzeros ahead with all gathers in flight before the FMAs. At each
// fiber change (j) the lane folds its y1 into the slice's Z (Mpad x G, shared
// memory) with V_p[:, j] from the j-major copy: Z[m][r] += y1[r] * V_p[m, j],
// shared-memory atomics (warps of the CTA share Z rows), rows skewed by r/8 so
// the 32 lanes hit 32 banks.
template <int C, bool F16, int UNROLL>
__global__ void __launch_bounds__(NT, (UNROLL <= 4 ? 3 : 2)) coo_fiber_kernel(
    const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, const float* __restrict__ cv,
    const int64_t* __restrict__ slice_off, const int32_t* __restrict__ slice_cnt, int64_t n_slices,
    const __nv_bfloat16* __restrict__ ut, int64_t ld_ut, int64_t plrows, const __nv_bfloat16* __restrict__ vtj,
    int64_t ld_vtj, int mpad, int lpad, int64_t count, float* __restrict__ z) {
  constexpr int G = 256 * C, GS = G + G / 8;
  extern __shared__ float zs[];  // [mpad][GS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t s = blockIdx.x; s < n_slices; s += gridDim.x) {
    const int64_t b0 = slice_off[s], n = slice_cnt[s];
    const int64_t per = (n + 7) / 8;
    const int64_t w0 = b0 + (warp * per < n ? warp * per : n), w1 = b0 + ((warp + 1) * per < n ? (warp + 1) * per : n);
    for (int64_t g0 = 0; g0 < plrows; g0 += G) {
      for (int e = threadIdx.x; e < mpad * GS; e += NT) zs[e] = 0.f;
      __syncthreads();
      float y1[C][8];
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int t = 0; t < 8; ++t) y1[c][t] = 0.f;
      int32_t cur_j = -1;
      auto flush = [&]() {
        if (cur_j >= 0) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int rl = c * 256 + lane * 8;  // local row of t = 0
            const int64_t rg = g0 + rl;
            if (rg < plrows) {
              const int64_t p = rg / lpad;
              const __nv_bfloat16* vrow = vtj + static_cast<int64_t>(cur_j) * ld_vtj + p * mpad;
              float* zr = zs + rl + rl / 8;
              for (int m0 = 0; m0 < mpad; m0 += 8) {
                float v[8];
                if constexpr (F16) half8(*reinterpret_cast<const uint4*>(vrow + m0), v);
                else bf16x8(*reinterpret_cast<const uint4*>(vrow + m0), v);
#pragma unroll
                for (int mm = 0; mm < 8; ++mm)
#pragma unroll
                  for (int t = 0; t < 8; ++t) atomicAdd(zr + (m0 + mm) * GS + t, y1[c][t] * v[mm]);
              }
            }
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
          for (int t = 0; t < 8; ++t) y1[c][t] = 0.f;
      };
      const __nv_bfloat16* ubase = ut + g0 + lane * 8;
      for (int64_t e0 = w0; e0 < w1; e0 += UNROLL) {
        // lanes < UNROLL fetch one nonzero each; the value is rounded to bf16
        // (the dense path's X precision) for the mixed bf16 x bf16 + f32 FMA
        int32_t li = 0, lj = -2;
        uint32_t lx = 0;
        if (lane < UNROLL && e0 + lane < w1) {
          li = __ldg(ci + e0 + lane);
          lj = __ldg(cj + e0 + lane);
          const float v = __ldg(cv + e0 + lane);
          lx = F16 ? __half_as_ushort(__float2half_rn(v)) : __bfloat16_as_ushort(__float2bfloat16_rn(v));
        }
        uint4 u[UNROLL][C];
#pragma unroll
        for (int t = 0; t < UNROLL; ++t) {
          const int32_t it = __shfl_sync(0xffffffffu, li, t);
          const __nv_bfloat16* col = ubase + static_cast<int64_t>(it) * ld_ut;
#pragma unroll
          for (int c = 0; c < C; ++c) u[t][c] = __ldg(reinterpret_cast<const uint4*>(col + c * 256));
        }
        // common case: the whole batch continues the current fiber
        const bool same = __all_sync(0xffffffffu, lane >= UNROLL || lj == cur_j || lj == -2);
        if (same) {
#pragma unroll
          for (int t = 0; t < UNROLL; ++t) {
            const uint16_t xt = static_cast<uint16_t>(__shfl_sync(0xffffffffu, lx, t));
#pragma unroll
            for (int c = 0; c < C; ++c) fma8<F16>(y1[c], u[t][c], xt);
          }
        } else {
#pragma unroll
          for (int t = 0; t < UNROLL; ++t) {
            const int32_t jt = __shfl_sync(0xffffffffu, lj, t);
            const uint16_t xt = static_cast<uint16_t>(__shfl_sync(0xffffffffu, lx, t));
            if (jt != -2) {
              if (jt != cur_j) {
                flush();
                cur_j = jt;
              }
#pragma unroll
              for (int c = 0; c < C; ++c) fma8<F16>(y1[c], u[t][c], xt);
            }
          }
        }
      }
      flush();
      __syncthreads();
      // Z[p][s][m][l] for the rows of this pass
      for (int e = threadIdx.x; e < G * mpad; e += NT) {
        const int m = e / G, r = e % G;
        const int64_t gr = g0 + r;
        if (gr >= plrows) continue;
        const int64_t p = gr / lpad, l = gr % lpad;
        if (p >= count) continue;
        z[((p * n_slices + s) * mpad + m) * lpad + l] = zs[m * GS + r + r / 8];
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


// CSF input (slices -> fibers -> nonzeros): per-nonzero fiber index j (one
// warp per fiber), slice offsets/counts in nonzeros, and range/monotonicity
// validation (bad[0]: coordinate outside the tensor, bad[1]: pointers not
// monotone or not matching the array lengths)
__global__ void csf_expand_kernel(const int64_t* __restrict__ fiber_ptr, const int32_t* __restrict__ fiber_j,
                                  int64_t n_fibers, int64_t J, int64_t nnz, int32_t* __restrict__ sj,
                                  int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t f = w0; f < n_fibers; f += nw) {
    const int64_t b = fiber_ptr[f], e = fiber_ptr[f + 1];
    const int32_t j = fiber_j[f];
    if (lane == 0) {
      if (j < 0 || j >= J) bad[0] = 1;
      if (b > e || b < 0 || e > nnz) bad[1] = 1;
    }
    if (b > e || b < 0 || e > nnz || !sj) continue;
    for (int64_t q = b + lane; q < e; q += 32) sj[q] = j;
  }
}

__global__ void csf_slices_kernel(const int64_t* __restrict__ slice_ptr, const int64_t* __restrict__ fiber_ptr,
                                  const int32_t* __restrict__ slice_k, int64_t n_slices, int64_t n_fibers,
                                  int64_t K, int64_t* __restrict__ off, int32_t* __restrict__ cnt,
                                  int* __restrict__ bad) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n_slices;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t f0 = slice_ptr[q], f1 = slice_ptr[q + 1];
    if (f0 > f1 || f0 < 0 || f1 > n_fibers) {
      bad[1] = 1;
      off[q] = 0;
      cnt[q] = 0;
      continue;
    }
    if (slice_k[q] < 0 || slice_k[q] >= K) bad[0] = 1;
    off[q] = fiber_ptr[f0];
    const int64_t c = fiber_ptr[f1] - fiber_ptr[f0];
    if (c < 0 || c > 0x7fffffff) bad[1] = 1;
    cnt[q] = static_cast<int32_t>(c);
  }
}

__global__ void range_i_kernel(const int32_t* __restrict__ ii, int64_t n, int64_t I, int* __restrict__ bad) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (ii[e] < 0 || ii[e] >= I) bad[0] = 1;
}

int64_t round_up256(int64_t a) { return (a + 255) / 256 * 256; }

int gridn(int64_t work) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 16))); }

}  // namespace

void Plan::compress_coo(const int32_t* i, const int32_t* j, const int32_t* k, const float* val, int64_t nnz, float* y,
                        bool accumulate, cudaStream_t s) {
  if (!tensor_core()) usage("plan_compress_coo: needs a bf16/fp16 (tensor-core) plan");
  if (comp()) usage("plan_compress_coo: the compensated mode covers dense input only (use a bf16/fp16 plan)");
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
  const bool padded = virt_padded();
  OutView<float> yo(y, static_cast<size_t>(ysz), s);
  if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
  if (nnz == 0) {
    if (!accumulate) XCUDA(cudaMemsetAsync(yo.dev, 0, ysz * 4, s));
    if (yo.host) yo.finish();
    return;
  }
  PhaseTrace tr("compress_coo", s);
  ensure_sparse_operands(s);
  InView<int32_t> di(i, static_cast<size_t>(nnz), s), dj(j, static_cast<size_t>(nnz), s), dk(k, static_cast<size_t>(nnz), s);
  InView<float> dv(val, static_cast<size_t>(nnz), s);
  tr.mark("inputs");
  // tile path with compact (rank k, rank j) keys: 4-byte keys make the sort
  // half the traffic of the 8-byte (k*J + j) keys; falls back to those when
  // the used k and j values do not fit 32 bits together (XTSG_COO_KEY64=1 forces)
  const char* k64 = std::getenv("XTSG_COO_KEY64");
  if (sparse_tc_ok() && !(k64 && std::atoi(k64) != 0) &&
      sparse_tc_coo32(di.dev, dj.dev, dk.dev, dv.dev, nnz, yo.dev, accumulate, s)) {
    if (fp16()) check_finite16(yo.dev, ysz, s);
    if (yo.host) yo.finish();
    return;
  }
  // 1. keys, validation, sortedness
  DevBuf<uint64_t> keys(static_cast<size_t>(nnz), s);
  DevBuf<uint64_t> idx(static_cast<size_t>(nnz), s);  // packed (i, value)
  DevBuf<int> flags(2, s);
  flags.zero();
  coo_keys_kernel<<<gridn(nnz), 256, 0, s>>>(dj.dev, dk.dev, nnz, J, keys.ptr, idx.ptr, flags.ptr, I, K, di.dev,
                                             dv.dev);
  XLAUNCH_CHECK();
  unsorted_kernel<<<gridn(nnz), 256, 0, s>>>(keys.ptr, nnz, flags.ptr + 1);
  XLAUNCH_CHECK();
  int hf[2] = {0, 0};
  XCUDA(cudaMemcpyAsync(hf, flags.ptr, sizeof(hf), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  tr.mark("keys");
  if (hf[0]) data_error("plan_compress_coo: coordinate outside the tensor");
  const int32_t *si = di.dev, *sj = dj.dev, *sk = dk.dev;
  const float* sv = dv.dev;
  DevBuf<int32_t> bi, bj, bk;
  DevBuf<float> bv;
  if (hf[1]) {
    DevBuf<uint64_t> keys2(static_cast<size_t>(nnz), s);
    DevBuf<uint64_t> idx2(static_cast<size_t>(nnz), s);
    int end_bit = 1;
    while (end_bit < 64 && (uint64_t(1) << end_bit) < static_cast<uint64_t>(K) * static_cast<uint64_t>(J)) ++end_bit;
    {
      // double-buffered sort: the two key/payload buffers are its ping-pong
      // storage (small temporary instead of another 16 B per nonzero)
      cub::DoubleBuffer<uint64_t> dkeys(keys.ptr, keys2.ptr), dpay(idx.ptr, idx2.ptr);
      size_t tmp_bytes = 0;
      XCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dkeys, dpay, nnz, 0, end_bit, s));
      DevBuf<uint8_t> tmp(tmp_bytes, s);
      XCUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, dkeys, dpay, nnz, 0, end_bit, s));
      count_launch();
      if (dkeys.Current() != keys2.ptr) std::swap(keys, keys2);
      if (dpay.Current() != idx2.ptr) std::swap(idx, idx2);
    }
    tr.mark("sort");
    keys.release();
    idx.release();
    if (sparse_tc_ok()) {
      sparse_tc_sorted(keys2, &idx2, nullptr, nullptr, nnz, yo.dev, accumulate, s);
      if (fp16()) check_finite16(yo.dev, ysz, s);
      if (yo.host) yo.finish();
      return;
    }
    bi = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bj = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bk = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bv = DevBuf<float>(static_cast<size_t>(nnz), s);
    coo_unpack_kernel<<<gridn(nnz), 256, 0, s>>>(keys2.ptr, idx2.ptr, nnz, J, bi.ptr, bj.ptr, bk.ptr, bv.ptr);
    XLAUNCH_CHECK();
    si = bi.ptr; sj = bj.ptr; sk = bk.ptr; sv = bv.ptr;
  }
  if (!hf[1] && sparse_tc_ok()) {
    idx.release();
    sparse_tc_sorted(keys, nullptr, di.dev, dv.dev, nnz, yo.dev, accumulate, s);
    if (fp16()) check_finite16(yo.dev, ysz, s);
    if (yo.host) yo.finish();
    return;
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
  coo_slices(si, sj, sv, off.ptr, cnt.ptr, uk.ptr, kd, yo.dev, accumulate, s);
  if (fp16()) check_finite16(yo.dev, ysz, s);
  if (yo.host) yo.finish();
}


// Sparse input already in CSF form (mode order k -> j -> i): no sort, no
// run-length encoding — the fibers feed the warp-level fiber kernel directly.
void Plan::compress_csf(int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr, int64_t n_fibers,
                        const int32_t* fiber_j, const int64_t* fiber_ptr, int64_t nnz, const int32_t* nz_i,
                        const float* val, float* y, bool accumulate, cudaStream_t s) {
  if (!tensor_core()) usage("plan_compress_csf: needs a bf16/fp16 (tensor-core) plan");
  if (comp()) usage("plan_compress_csf: the compensated mode covers dense input only (use a bf16/fp16 plan)");
  if (stage1) usage("plan_compress_csf: two-stage plans take COO input");
  if (n_slices < 0 || n_fibers < 0 || nnz < 0) usage("plan_compress_csf: negative size");
  const int64_t I = desc.dims[0], J = desc.dims[1], K = desc.dims[2];
  const int64_t ysz = desc.count * desc.reduced[0] * desc.reduced[1] * desc.reduced[2];
  OutView<float> yo(y, static_cast<size_t>(ysz), s);
  if (accumulate && yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, ysz * 4, cudaMemcpyHostToDevice, s));
  if (nnz == 0 || n_slices == 0) {
    if (!accumulate) XCUDA(cudaMemsetAsync(yo.dev, 0, ysz * 4, s));
    if (yo.host) yo.finish();
    return;
  }
  ensure_sparse_operands(s);
  InView<int32_t> dk(slice_k, static_cast<size_t>(n_slices), s), dj(fiber_j, static_cast<size_t>(n_fibers), s),
      di(nz_i, static_cast<size_t>(nnz), s);
  InView<int64_t> dsp(slice_ptr, static_cast<size_t>(n_slices + 1), s),
      dfp(fiber_ptr, static_cast<size_t>(n_fibers + 1), s);
  InView<float> dv(val, static_cast<size_t>(nnz), s);
  const bool tc = sparse_tc_ok();
  DevBuf<int32_t> sj(tc ? 0 : static_cast<size_t>(nnz), s), cnt(static_cast<size_t>(n_slices), s);
  DevBuf<int64_t> off(static_cast<size_t>(n_slices), s);
  DevBuf<int> bad(2, s);
  bad.zero();
  if (!tc) XCUDA(cudaMemsetAsync(sj.ptr, 0, sizeof(int32_t) * nnz, s));
  csf_expand_kernel<<<gridn(n_fibers * 32), 256, 0, s>>>(dfp.dev, dj.dev, n_fibers, J, nnz, sj.ptr, bad.ptr);
  XLAUNCH_CHECK();
  csf_slices_kernel<<<gridn(n_slices), 256, 0, s>>>(dsp.dev, dfp.dev, dk.dev, n_slices, n_fibers, K, off.ptr, cnt.ptr,
                                                    bad.ptr);
  XLAUNCH_CHECK();
  range_i_kernel<<<gridn(nnz), 256, 0, s>>>(di.dev, nnz, I, bad.ptr);
  XLAUNCH_CHECK();
  int hb[2] = {0, 0};
  XCUDA(cudaMemcpyAsync(hb, bad.ptr, sizeof(hb), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  if (hb[0]) data_error("plan_compress_csf: coordinate outside the tensor");
  if (hb[1]) data_error("plan_compress_csf: slice/fiber pointers not monotone or inconsistent with the sizes");
  if (tc) {
    sparse_tc(n_slices, dk.dev, dsp.dev, n_fibers, dfp.dev, dj.dev, nnz, di.dev, dv.dev, yo.dev, accumulate, s);
    if (fp16()) check_finite16(yo.dev, ysz, s);
    if (yo.host) yo.finish();
    return;
  }
  coo_slices(di.dev, sj.ptr, dv.dev, off.ptr, cnt.ptr, dk.dev, n_slices, yo.dev, accumulate, s);
  if (fp16()) check_finite16(yo.dev, ysz, s);
  if (yo.host) yo.finish();
}

// i-major U (rows padded to 256 with zeros) and j-major V copies of the
// sparse path, built on first use
void Plan::ensure_sparse_operands(cudaStream_t s) {
  const int64_t I = desc.dims[0], J = desc.dims[1];
  const int64_t plrows = vP * lpad;
  const int64_t ld_ut = round_up256(plrows), ld_vtj = vP * mpad;
  if (!ut.ptr) {
    // i-major U (rows padded to 256 with zeros) and j-major V copies
    ut = DevBuf<__nv_bfloat16>(static_cast<size_t>(I * ld_ut), s);
    ut.zero();
    dim3 grid(static_cast<unsigned>(ceil_div(I, 32)), static_cast<unsigned>(ceil_div(plrows, 32)));
    transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(ustack.ptr, plrows, ld_u, I, ld_ut, ut.ptr);
    XLAUNCH_CHECK();
    vtj = DevBuf<__nv_bfloat16>(static_cast<size_t>(J * ld_vtj), s);
    dim3 gv(static_cast<unsigned>(ceil_div(J, 32)), static_cast<unsigned>(ceil_div(ld_vtj, 32)));
    transpose_bf16_kernel<<<gv, dim3(32, 8), 0, s>>>(vt.ptr, ld_vtj, ld_v, J, ld_vtj, vtj.ptr);
    XLAUNCH_CHECK();
  }
}

// Steps 3-5 of the sparse path on (k, j)-grouped nonzeros: kd slices, slice s
// holding nonzeros [off[s], off[s] + cnt[s]) of mode-3 index uk[s], fibers
// (runs of equal j) contiguous inside a slice -> y (+)= the replicas.
void Plan::coo_slices(const int32_t* si, const int32_t* sj, const float* sv, const int64_t* off_p,
                      const int32_t* cnt_p, const int32_t* uk_p, int64_t kd, float* ydev, bool accumulate,
                      cudaStream_t s) {
  const int64_t plrows = vP * lpad;
  const int64_t ld_ut = round_up256(plrows), ld_vtj = vP * mpad;
  // 3. fibers -> Z[p][kd][m][l]
  DevBuf<float> z(static_cast<size_t>(vP * kd * mpad * lpad), s);
  // C groups of 256 rows per pass, Z pass in shared memory (mpad x 1.125*G fp32)
  static const int cenv = [] {
    const char* e = std::getenv("XTSG_COO_C");
    return e ? std::atoi(e) : 0;
  }();
  const int cmax = (mpad <= 64 ? 2 : 1) < (cenv > 0 ? cenv : 2) ? (mpad <= 64 ? 2 : 1) : (cenv > 0 ? cenv : 2);
  const int cg = plrows > 256 ? cmax : 1;
  const size_t smem = static_cast<size_t>(mpad) * (256 * cg + 32 * cg) * sizeof(float);
  auto launch = [&](auto kern) {
    XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 1;
    XCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    const int grid = static_cast<int>(std::min<int64_t>(kd, static_cast<int64_t>(sm_count()) * std::max(1, per_sm)));
    kern<<<grid, NT, smem, s>>>(si, sj, sv, off_p, cnt_p, kd, ut.ptr, ld_ut, plrows, vtj.ptr, ld_vtj,
                                static_cast<int>(mpad), static_cast<int>(lpad), vP, z.ptr);
  };
  // nonzeros in flight per warp: 4 keeps the kernel at <= 85 registers
  // (3 CTAs per SM), 8 at 2 CTAs per SM (XTSG_COO_UNROLL)
  static const int unroll = [] {
    const char* e = std::getenv("XTSG_COO_UNROLL");
    return e && std::atoi(e) == 8 ? 8 : 4;
  }();
  if (fp16()) {
    if (cg == 2) unroll == 8 ? launch(coo_fiber_kernel<2, true, 8>) : launch(coo_fiber_kernel<2, true, 4>);
    else unroll == 8 ? launch(coo_fiber_kernel<1, true, 8>) : launch(coo_fiber_kernel<1, true, 4>);
  } else {
    if (cg == 2) unroll == 8 ? launch(coo_fiber_kernel<2, false, 8>) : launch(coo_fiber_kernel<2, false, 4>);
    else unroll == 8 ? launch(coo_fiber_kernel<1, false, 8>) : launch(coo_fiber_kernel<1, false, 4>);
  }
  XLAUNCH_CHECK();
  sparse_mode3(z.ptr, uk_p, kd, ydev, accumulate, s);
}

// 4-5. mode 3 over the distinct slices: y (+)= Z_p W_p[:, uk]^T
void Plan::sparse_mode3(const float* z, const int32_t* uk_p, int64_t kd, float* ydev, bool accumulate,
                        cudaStream_t s) {
  const int64_t N = desc.reduced[2], K = desc.dims[2];
  const bool padded = virt_padded();
  DevBuf<float> wg(static_cast<size_t>(vP * N * kd), s);
  gather_w_kernel<<<gridn(vP * N * kd), 256, 0, s>>>(wf.ptr, vP, N, K, uk_p, kd, wg.ptr);
  XLAUNCH_CHECK();
  DevBuf<float> ypad;
  float* ydst = ydev;
  if (padded) {
    ypad = DevBuf<float>(static_cast<size_t>(vP * mpad * lpad * N), s);
    ydst = ypad.ptr;
  }
  GemmArgs<float> g;
  g.m = mpad * lpad; g.n = N; g.k = kd; g.batch = vP;
  g.a = z; g.lda = mpad * lpad; g.stride_a = kd * mpad * lpad;
  g.b = wg.ptr; g.ldb = kd; g.stride_b = N * kd;
  g.c = ydst; g.ldc = mpad * lpad; g.stride_c = mpad * lpad * N;
  g.beta = (accumulate && !padded) ? 1.f : 0.f;
  gemm_simt(g, s);
  if (padded) {
    compact(ypad.ptr, ydev, accumulate, s);
  }
}

}  // namespace xtsg

using namespace xtsg;

extern "C" int32_t xtsg_plan_compress_coo(xtsg_plan* plan, const int32_t* i, const int32_t* j, const int32_t* k,
                                          const float* val, int64_t nnz, void* y, int32_t accumulate, void* stream) {
  return guard([&] {
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : thread_stream();
    PlanUse use(p, s);
    p->compress_coo(i, j, k, val, nnz, static_cast<float*>(y), accumulate != 0, s);
  });
}

extern "C" int32_t xtsg_plan_compress_csf(xtsg_plan* plan, int64_t n_slices, const int32_t* slice_k,
                                          const int64_t* slice_ptr, int64_t n_fibers, const int32_t* fiber_j,
                                          const int64_t* fiber_ptr, int64_t nnz, const int32_t* nz_i,
                                          const float* val, void* y, int32_t accumulate, void* stream) {
  return guard([&] {
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : thread_stream();
    PlanUse use(p, s);
    p->compress_csf(n_slices, slice_k, slice_ptr, n_fibers, fiber_j, fiber_ptr, nnz, nz_i, val,
                    static_cast<float*>(y), accumulate != 0, s);
  });
}
