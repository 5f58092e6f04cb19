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

}  // namespace

template <class T>
void gemm_simt(const GemmArgs<T>& g, cudaStream_t st) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
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
