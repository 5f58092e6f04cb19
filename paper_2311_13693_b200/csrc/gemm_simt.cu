#include <type_traits>
#include "common.cuh"
#include "gemm_simt.cuh"

namespace xtsg {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

template <class T>
__global__ void __launch_bounds__(256) gemm_kernel(GemmArgs<T> g) {
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int64_t bz = blockIdx.z;
  const T* A = g.a + bz * g.stride_a;
  const T* B = g.b + bz * g.stride_b;
  T* C = g.c + bz * g.stride_c;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int64_t k0 = 0; k0 < g.k; k0 += BK) {
    // 64x16 tiles, 4 elements per thread each
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = threadIdx.x + e * 256;
      // A tile: element (mi, ki); when A is not transposed walk mi fastest
      int mi, ki;
      if (!g.trans_a) { mi = idx % BM; ki = idx / BM; } else { ki = idx % BK; mi = idx / BK; }
      const int64_t gm = m0 + mi, gk = k0 + ki;
      T va = T(0);
      if (gm < g.m && gk < g.k) va = g.trans_a ? A[gk + gm * g.lda] : A[gm + gk * g.lda];
      As[ki][mi] = va;
      int ni, kj;
      if (g.trans_b) { ni = idx % BN; kj = idx / BN; } else { kj = idx % BK; ni = idx / BK; }
      const int64_t gn = n0 + ni, gk2 = k0 + kj;
      T vb = T(0);
      if (gn < g.n && gk2 < g.k) vb = g.trans_b ? B[gn + gk2 * g.ldb] : B[gk2 + gn * g.ldb];
      Bs[kj][ni] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T ra[TM], rb[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) ra[i] = As[kk][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) rb[j] = Bs[kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(ra[i], rb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int64_t gn = n0 + ty + 16 * j;
    if (gn >= g.n) continue;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t gm = m0 + tx + 16 * i;
      if (gm >= g.m) continue;
      T* dst = C + gm + gn * g.ldc;
      const T v = g.alpha * acc[i][j];
      *dst = g.beta == T(0) ? v : v + g.beta * *dst;
    }
  }
}

// fp32 NN fast path: C[b] = alpha A[b] B[b] + beta C[b] with A (m x k, lda),
// B (k x n, ldb) column-major, no transposes. 128 x 64 block tile, 32-deep K
// chunks, 8 x 4 outputs per thread from float4 shared-memory reads, register
// double buffering of the next chunk. Used for the mode-3 contraction
// (Y_p += Z_p W_p^T) of the tensor-core path, where m = Lpad*Mpad, n = N.
constexpr int FM = 128, FN = 64, FK = 32;

__global__ void __launch_bounds__(256) gemm_f32_nn_kernel(GemmArgs<float> g) {
  __shared__ __align__(16) float As[FK][FM];
  __shared__ __align__(16) float Bs[FK][FN + 4];
  const int64_t bz = blockIdx.z;
  const float* A = g.a + bz * g.stride_a;
  const float* B = g.b + bz * g.stride_b;
  float* C = g.c + bz * g.stride_c;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * FM, n0 = static_cast<int64_t>(blockIdx.y) * FN;
  const int tid = threadIdx.x, tr = tid % 16, tc = tid / 16;
  // loader mapping: A chunk FK x FM (m fastest): 4 float4 per thread; B chunk FN x FK (k fastest): 2 float4
  float4 ra[4], rb[2];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;       // 0..1023 float4 slots
      const int kk = idx / (FM / 4), mm = (idx % (FM / 4)) * 4;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < g.k) {
        const float* src = A + gm + g.lda * gk;
        if (gm + 3 < g.m && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) v = *reinterpret_cast<const float4*>(src);
        else {
          if (gm < g.m) v.x = src[0];
          if (gm + 1 < g.m) v.y = src[1];
          if (gm + 2 < g.m) v.z = src[2];
          if (gm + 3 < g.m) v.w = src[3];
        }
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int idx = tid + e * 256;       // 0..511
      const int nn = idx / (FK / 4), kk = (idx % (FK / 4)) * 4;
      const int64_t gn = n0 + nn, gk = k0 + kk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gn < g.n) {
        const float* src = B + gk + g.ldb * gn;
        if (gk + 3 < g.k && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) v = *reinterpret_cast<const float4*>(src);
        else {
          if (gk < g.k) v.x = src[0];
          if (gk + 1 < g.k) v.y = src[1];
          if (gk + 2 < g.k) v.z = src[2];
          if (gk + 3 < g.k) v.w = src[3];
        }
      }
      rb[e] = v;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      const int kk = idx / (FM / 4), mm = (idx % (FM / 4)) * 4;
      *reinterpret_cast<float4*>(&As[kk][mm]) = ra[e];
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int idx = tid + e * 256;
      const int nn = idx / (FK / 4), kk = (idx % (FK / 4)) * 4;
      Bs[kk + 0][nn] = rb[e].x;
      Bs[kk + 1][nn] = rb[e].y;
      Bs[kk + 2][nn] = rb[e].z;
      Bs[kk + 3][nn] = rb[e].w;
    }
  };
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  load(0);
  for (int64_t k0 = 0; k0 < g.k; k0 += FK) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + FK < g.k) load(k0 + FK);
#pragma unroll 8
    for (int kk = 0; kk < FK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][tr * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + tr * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tc * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[4] = {b0.x, b0.y, b0.z, b0.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t gn = n0 + tc * 4 + j;
    if (gn >= g.n) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t gm = m0 + (i < 4 ? tr * 4 + i : 64 + tr * 4 + (i - 4));
      if (gm >= g.m) continue;
      float* dst = C + gm + g.ldc * gn;
      const float v = g.alpha * acc[i][j];
      *dst = g.beta == 0.f ? v : v + g.beta * *dst;
    }
  }
}

// fp64 on the tensor cores (DMMA m8n8k4): 64 x 64 block tile, 16-deep K
// chunks staged k-major in shared memory with a 68-double row stride (every
// fragment load bank-conflict free), 8 warps of 32 x 16, register-staged
// prefetch of the next chunk. Fixed K order per output (deterministic).
constexpr int DM = 64, DN = 64, DK = 16, DLD = 68;

__global__ void __launch_bounds__(256) gemm_f64_dmma_kernel(GemmArgs<double> g) {
  __shared__ __align__(16) double As[DK][DLD];
  __shared__ __align__(16) double Bs[DK][DLD];
  const int64_t bz = blockIdx.z;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * DM, n0 = static_cast<int64_t>(blockIdx.y) * DN;
  if (g.lower_only && m0 + DM <= n0) return;
  const double* A = g.a + bz * g.stride_a;
  const double* B = g.b + bz * g.stride_b;
  double* C = g.c + bz * g.stride_c;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warps of 32 x 16
  double ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int mi, ki;
      if (!g.trans_a) { mi = idx % DM; ki = idx / DM; } else { ki = idx % DK; mi = idx / DK; }
      const int64_t gm = m0 + mi, gk = k0 + ki;
      ra[e] = (gm < g.m && gk < g.k) ? (g.trans_a ? A[gk + gm * g.lda] : A[gm + gk * g.lda]) : 0.0;
      int ni, kj;
      if (g.trans_b) { ni = idx % DN; kj = idx / DN; } else { kj = idx % DK; ni = idx / DK; }
      const int64_t gn = n0 + ni, gk2 = k0 + kj;
      rb[e] = (gn < g.n && gk2 < g.k) ? (g.trans_b ? B[gn + gk2 * g.ldb] : B[gk2 + gn * g.ldb]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int mi, ki;
      if (!g.trans_a) { mi = idx % DM; ki = idx / DM; } else { ki = idx % DK; mi = idx / DK; }
      As[ki][mi] = ra[e];
      int ni, kj;
      if (g.trans_b) { ni = idx % DN; kj = idx / DN; } else { kj = idx % DK; ni = idx / DK; }
      Bs[kj][ni] = rb[e];
    }
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  load(0);
  for (int64_t k0 = 0; k0 < g.k; k0 += DK) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + DK < g.k) load(k0 + DK);
#pragma unroll
    for (int ks = 0; ks < DK / 4; ++ks) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[ks * 4 + lc][wm * 32 + i * 8 + lr];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[ks * 4 + lc][wn * 16 + j * 8 + lr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(a[i]), "d"(b[j]));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t gm = m0 + wm * 32 + i * 8 + lr, gn = n0 + wn * 16 + j * 8 + 2 * lc + e;
        if (gm >= g.m || gn >= g.n) continue;
        double* dst = C + gm + gn * g.ldc;
        const double v = g.alpha * acc[i][j][e];
        *dst = g.beta == 0.0 ? v : v + g.beta * *dst;
      }
}

}  // namespace

template <class T>
void gemm_simt(const GemmArgs<T>& g, cudaStream_t st) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
  if constexpr (std::is_same<T, float>::value) {
    if (!g.trans_a && !g.trans_b && g.k > 0) {
      int64_t left = g.batch;
      GemmArgs<float> part = g;
      while (left > 0) {
        const int64_t nb = std::min<int64_t>(left, 65535);
        part.batch = nb;
        dim3 grid(static_cast<unsigned>(ceil_div(g.m, FM)), static_cast<unsigned>(ceil_div(g.n, FN)),
                  static_cast<unsigned>(nb));
        gemm_f32_nn_kernel<<<grid, 256, 0, st>>>(part);
        XLAUNCH_CHECK();
        part.a += nb * g.stride_a;
        part.b += nb * g.stride_b;
        part.c += nb * g.stride_c;
        left -= nb;
      }
      return;
    }
  }
  if constexpr (std::is_same<T, double>::value) {
    if (g.k > 0) {
      int64_t left = g.batch;
      GemmArgs<double> part = g;
      while (left > 0) {
        const int64_t nb = std::min<int64_t>(left, 65535);
        part.batch = nb;
        dim3 grid(static_cast<unsigned>(ceil_div(g.m, DM)), static_cast<unsigned>(ceil_div(g.n, DN)),
                  static_cast<unsigned>(nb));
        if (grid.y > 65535) throw Status(XTSG_E_USAGE, "gemm: n too large for one launch");
        gemm_f64_dmma_kernel<<<grid, 256, 0, st>>>(part);
        XLAUNCH_CHECK();
        part.a += nb * g.stride_a;
        part.b += nb * g.stride_b;
        part.c += nb * g.stride_c;
        left -= nb;
      }
      return;
    }
  }
  int64_t batch_left = g.batch;
  GemmArgs<T> part = g;
  while (batch_left > 0) {
    const int64_t nb = std::min<int64_t>(batch_left, 65535);
    part.batch = nb;
    dim3 grid(static_cast<unsigned>(ceil_div(g.n, BN)), static_cast<unsigned>(ceil_div(g.m, BM)),
              static_cast<unsigned>(nb));
    if (grid.y > 65535) throw Status(XTSG_E_USAGE, "gemm: m too large for one launch");
    gemm_kernel<T><<<grid, 256, 0, st>>>(part);
    XLAUNCH_CHECK();
    part.a += nb * g.stride_a;
    part.b += nb * g.stride_b;
    part.c += nb * g.stride_c;
    batch_left -= nb;
  }
}

template void gemm_simt<double>(const GemmArgs<double>&, cudaStream_t);
template void gemm_simt<float>(const GemmArgs<float>&, cudaStream_t);

}  // namespace xtsg
