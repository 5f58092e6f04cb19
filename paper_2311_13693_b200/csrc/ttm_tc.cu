// K2+K3 — fused stacked mode-1 / mode-2 TTM on the 5th-gen tensor cores.
//
// Reference semantics: comp_with (compression.cpp:202-209) for all P replicas
// of an ensemble at once: Y_p = X x1 U_p x2 V_p x3 W_p. This kernel computes
// the first two mode products for every replica and every mode-3 slice k,
//   Z_p[:, :, k] = U_p * X[:, :, k] * V_p^T          (L x M per (p, k)),
// and leaves mode 3 (a K-contraction of Z with W_p, 1/M of mode-2's work) to a
// follow-up GEMM. The P replicas' U_p are stacked into one (P*L) x I operand
// so each X tile is multiplied by all replicas straight out of shared memory.
//
// Tiling (one CTA per SM, persistent, static schedule):
//   unit  = (row block rb of 128 stacked U rows = 128/L replicas, slice k)
//   tile  = 256 consecutive j of that slice; a unit walks all J/256 tiles
//   mode 1: D1[128 x 256] (fp32, TMEM) = Ustack[rb] (128 x I) * X[:, jtile, k]
//           K-loop over i in 64-wide chunks, A/B staged by TMA (SWIZZLE_128B)
//   mode 2: the epilogue warps drain D1 64 columns at a time to bf16 in smem
//           (A2, K-major SW128) and a second MMA stream computes
//           D2[128 x RPB*M] = A2 (128 x 256 j) * Vt_block (RPB*M x 256 j)^T
//           into the *already drained* first columns of the same TMEM buffer,
//           so TMEM holds two 256-column mode-1 accumulators (double buffer)
//           and no extra columns. The diagonal RPB blocks of D2 (row replica
//           == column replica) are accumulated over the unit's j tiles in the
//           epilogue's registers and written once per unit as Z[p][k][m][l].
// Warp roles (256 threads): w0 TMA producer (U, X), w1 mode-1 MMA issuer +
// TMEM owner, w2 TMA producer (Vt), w3 mode-2 MMA issuer, w4-7 epilogue (one
// TMEM lane quarter each). All hand-offs are mbarriers; tcgen05.commit
// releases smem stages and signals accumulators.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "sm100_ptx.cuh"
#include "ttm_tc.cuh"

namespace xtsg {

namespace {

constexpr int BM = 128;       // stacked U rows per tile (UMMA M)
constexpr int BK = 64;        // i per stage (128 B = one SW128 atom row)
constexpr int A_BYTES = BM * BK * 2;       // 16 KB
constexpr int A2_BYTES = BM * 64 * 2;      // 16 KB (128 rows x 64 j)
constexpr int B2_BYTES = 128 * 64 * 2;     // up to 128 (p,m) rows x 64 j

// Tile shape / pipeline depth: BN j per tile (UMMA N of mode 1, <= 256 so a
// TMEM buffer fits twice in 512 columns), S1 TMA stages. 256x3 and 192x4
// both fit the 227 KB shared-memory budget next to the mode-2 rings.
template <int BN_, int S1_>
struct TileCfg {
  static constexpr int BN = BN_;
  static constexpr int S1 = S1_;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int CHUNKS = BN / 64;  // mode-2 K chunks per full tile
  static constexpr int SMEM_DATA = S1 * STAGE_BYTES + 2 * A2_BYTES + 2 * B2_BYTES;
  static constexpr int SMEM_TOTAL = SMEM_DATA + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t IDESC1 = ptx::idesc_bf16(BM, BN);
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
};

template <int S1>
struct Bars {
  uint64_t full1[S1], empty1[S1];
  uint64_t tmem_full[2], tmem_empty[2], d2_full[2];
  uint64_t a2_full[2], a2_empty[2], b2_full[2], b2_empty[2];
  uint32_t tmem_base;
};

template <int MPAD, class Cfg, int CS>
__global__ void __launch_bounds__(256, 1)
    ttm_fused_kernel(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_v, const TtmParams p) {
  constexpr int BN = Cfg::BN, S1 = Cfg::S1, STAGE_BYTES = Cfg::STAGE_BYTES, CHUNKS = Cfg::CHUNKS;
  constexpr uint32_t IDESC1 = Cfg::IDESC1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* a2_base = smem + S1 * STAGE_BYTES;
  uint8_t* b2_base = a2_base + 2 * A2_BYTES;
  Bars<S1>* bars = reinterpret_cast<Bars<S1>*>(b2_base + 2 * B2_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S1; ++s) {
      ptx::mbar_init(&bars->full1[s], 1);
      ptx::mbar_init(&bars->empty1[s], CS);  // freed by the MMA of every CTA sharing the X tile
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bars->tmem_full[b], 1);
      ptx::mbar_init(&bars->tmem_empty[b], 128);
      ptx::mbar_init(&bars->d2_full[b], 1);
      ptx::mbar_init(&bars->a2_full[b], 128);
      ptx::mbar_init(&bars->a2_empty[b], 1);
      ptx::mbar_init(&bars->b2_full[b], 1);
      ptx::mbar_init(&bars->b2_empty[b], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tm_u);
    ptx::tma_prefetch(&tm_x);
    ptx::tma_prefetch(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 512);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // CS CTAs of a cluster take CS consecutive row blocks of the same slice and
  // tile sequence; each loads BN/CS rows of every X tile and multicasts them
  // to all CS CTAs, so an X tile crosses the L2->SM fabric once per cluster.
  const int crank = CS > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int cid = blockIdx.x / CS, n_clusters = gridDim.x / CS;
  const int n_rbg = p.n_rb / CS;
  const int n_units = n_rbg * p.kc;
  const uint16_t cmask = static_cast<uint16_t>((1u << CS) - 1u);
  const int j_tiles = p.j_tiles;
  const int k_steps = p.k_steps;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: U rows and X tiles -------------------------------
      int s = 0;
      uint32_t ph = 0;
      for (int u = cid; u < n_units; u += n_clusters) {
        const int kk = u / n_rbg, rb = (u % n_rbg) * CS + crank;
        for (int jt = 0; jt < j_tiles; ++jt) {
          for (int ks = 0; ks < k_steps; ++ks) {
            ptx::mbar_wait(&bars->empty1[s], ph ^ 1);
            uint8_t* st = stage_base + s * STAGE_BYTES;
            ptx::mbar_arrive_expect_tx(&bars->full1[s], STAGE_BYTES);
            ptx::tma_load_2d(st, &tm_u, &bars->full1[s], ks * BK, rb * BM);
            if constexpr (CS == 1)
              ptx::tma_load_3d(st + A_BYTES, &tm_x, &bars->full1[s], ks * BK, jt * BN, p.k_first + kk);
            else
              ptx::tma_load_3d_mc(st + A_BYTES + crank * (Cfg::B_BYTES / CS), &tm_x, &bars->full1[s], ks * BK,
                                  jt * BN + crank * (BN / CS), p.k_first + kk, cmask);
            if (++s == S1) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- mode-1 MMA issuer ----------------------------------------------
      int s = 0;
      uint32_t ph = 0;
      uint32_t t = 0;
      for (int u = cid; u < n_units; u += n_clusters) {
        for (int jt = 0; jt < j_tiles; ++jt, ++t) {
          const uint32_t b = t & 1, use = t >> 1;
          ptx::mbar_wait(&bars->tmem_empty[b], (use & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t d = tmem + b * 256;
          // ragged edges: the last j tile narrows N, the last i step issues
          // only the K=16 slices that hold data (TMA zero-fills the rest)
          const uint32_t idesc1 =
              (jt == j_tiles - 1 ? ptx::idesc_bf16(BM, p.n_last) : IDESC1) & ptx::idesc_fmt_mask(p.f16 != 0);
          for (int ks = 0; ks < k_steps; ++ks) {
            ptx::mbar_wait(&bars->full1[s], ph);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(stage_base + s * STAGE_BYTES);
            const uint32_t b0 = a0 + A_BYTES;
            const int nk16 = ks == k_steps - 1 ? p.k16_last : BK / 16;
#pragma unroll
            for (int k4 = 0; k4 < BK / 16; ++k4)
              if (k4 < nk16)
                ptx::mma_bf16(d, ptx::sw128_desc(a0 + k4 * 32), ptx::sw128_desc(b0 + k4 * 32), idesc1,
                              (ks | k4) != 0);
            if constexpr (CS == 1)
              ptx::mma_commit(&bars->empty1[s]);
            else
              ptx::mma_commit_mc(&bars->empty1[s], cmask);
            if (++s == S1) { s = 0; ph ^= 1; }
          }
          ptx::mma_commit(&bars->tmem_full[b]);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ---- TMA producer: Vt chunks for mode 2 -----------------------------
      const uint32_t bytes = static_cast<uint32_t>(p.n2) * 128;
      uint32_t g = 0;  // running chunk counter (shared convention with w3 / epilogue)
      for (int u = cid; u < n_units; u += n_clusters) {
        const int rb = (u % n_rbg) * CS + crank;
        for (int jt = 0; jt < j_tiles; ++jt) {
          const int nch = jt == j_tiles - 1 ? p.chunks_last : CHUNKS;
          for (int c = 0; c < nch; ++c, ++g) {
            const int slot = g & 1;
            const uint32_t par = (g >> 1) & 1;
            ptx::mbar_wait(&bars->b2_empty[slot], par ^ 1);
            ptx::mbar_arrive_expect_tx(&bars->b2_full[slot], bytes);
            ptx::tma_load_2d(b2_base + slot * B2_BYTES, &tm_v, &bars->b2_full[slot], jt * BN + c * 64,
                             rb * p.n2);
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ---- mode-2 MMA issuer ----------------------------------------------
      const uint32_t idesc2 = ptx::idesc_bf16(BM, p.n2) & ptx::idesc_fmt_mask(p.f16 != 0);
      uint32_t t = 0, g = 0;
      for (int u = cid; u < n_units; u += n_clusters) {
        for (int jt = 0; jt < j_tiles; ++jt, ++t) {
          const uint32_t b = t & 1;
          const uint32_t d = tmem + b * 256;
          const bool last = jt == j_tiles - 1;
          const int nch = last ? p.chunks_last : CHUNKS;
          // D2 overwrites D1 columns [0, n2): the first two 64-col chunks
          // (when present) must have been drained before the first MMA.
          ptx::mbar_wait(&bars->a2_full[g & 1], (g >> 1) & 1);
          if (nch > 1) ptx::mbar_wait(&bars->a2_full[(g + 1) & 1], ((g + 1) >> 1) & 1);
          for (int c = 0; c < nch; ++c, ++g) {
            const int slot = g & 1;
            const uint32_t par = (g >> 1) & 1;
            if (c >= 2) ptx::mbar_wait(&bars->a2_full[slot], par);
            ptx::mbar_wait(&bars->b2_full[slot], par);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(a2_base + slot * A2_BYTES);
            const uint32_t b0 = ptx::smem_u32(b2_base + slot * B2_BYTES);
            const int nk16 = (last && c == nch - 1) ? p.k16_chunk_last : 4;
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              if (k4 < nk16)
                ptx::mma_bf16(d, ptx::sw128_desc(a0 + k4 * 32), ptx::sw128_desc(b0 + k4 * 32), idesc2,
                              (c | k4) != 0);
            ptx::mma_commit(&bars->a2_empty[slot]);
            ptx::mma_commit(&bars->b2_empty[slot]);
          }
          ptx::mma_commit(&bars->d2_full[b]);
        }
      }
    }
  } else {
    // ---- epilogue: 4 warps, one TMEM lane quarter each ---------------------
    const int q = warp & 3;
    const int r = q * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int p_local = r / p.lpad;
    const int l = r % p.lpad;
    uint32_t t = 0, g = 0;
    for (int u = cid; u < n_units; u += n_clusters) {
      const int kk = u / n_rbg, rb = (u % n_rbg) * CS + crank;
      float zacc[MPAD];
#pragma unroll
      for (int m = 0; m < MPAD; ++m) zacc[m] = 0.f;
      for (int jt = 0; jt < j_tiles; ++jt, ++t) {
        const uint32_t b = t & 1, use = t >> 1;
        const int nch = jt == j_tiles - 1 ? p.chunks_last : CHUNKS;
        ptx::mbar_wait(&bars->tmem_full[b], use & 1);
        ptx::tc_fence_after();
        for (int c = 0; c < nch; ++c, ++g) {
          const int slot = g & 1;
          const uint32_t par = (g >> 1) & 1;
          ptx::mbar_wait(&bars->a2_empty[slot], par ^ 1);
          uint8_t* row = a2_base + slot * A2_BYTES + r * 128;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            float v[32];
            ptx::tmem_ld32(lane_addr + b * 256 + c * 64 + h * 32, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int q8 = h * 4 + q4;
              const uint4 pk = ptx::pack8(v + q4 * 8, p.f16 != 0);
              *reinterpret_cast<uint4*>(row + ((q8 ^ (r & 7)) << 4)) = pk;
            }
          }
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&bars->a2_full[slot]);
        }
        ptx::mbar_wait(&bars->d2_full[b], use & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int mc = 0; mc < MPAD / 32; ++mc) {
          float v[32];
          ptx::tmem_ld32(lane_addr + b * 256 + p_local * MPAD + mc * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) zacc[mc * 32 + e] += v[e];
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->tmem_empty[b]);
      }
      const int prep = rb * p.rpb + p_local;
      if (prep < p.count) {
        float* dst = p.z + ((static_cast<int64_t>(prep) * p.kc + kk) * MPAD) * p.lpad + l;
        const int stride = p.lpad;
#pragma unroll
        for (int m = 0; m < MPAD; ++m) {
          __stcs(dst, zacc[m]);
          dst += stride;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) ptx::cluster_sync();  // no CTA leaves while a peer may still multicast to it
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      throw Status(XTSG_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

void make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box, bool f16) {
  cuuint64_t d[3], s[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  if (reinterpret_cast<uintptr_t>(base) % 16) usage("tma: base address must be 16-byte aligned");
  for (int i = 0; i < rank - 1; ++i)
    if (s[i] % 16) usage("tma: strides must be multiples of 16 bytes");
  CUresult r = encode_fn()(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, bx, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Status(XTSG_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

template <int MPAD, class Cfg, int CS>
void launch_impl(const TtmLaunch& L, cudaStream_t st) {
  constexpr int BN = Cfg::BN;
  CUtensorMap mu, mx, mv;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(L.ni), static_cast<uint64_t>(L.rows_u)};
    const uint64_t str[1] = {static_cast<uint64_t>(L.ld_u) * 2};
    const uint32_t box[2] = {BK, BM};
    make_map(&mu, L.u, 2, dims, str, box, L.prm.f16 != 0);
  }
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(L.ni), static_cast<uint64_t>(L.nj), static_cast<uint64_t>(L.nk)};
    const uint64_t str[2] = {static_cast<uint64_t>(L.ld_x0) * 2, static_cast<uint64_t>(L.ld_x1) * 2};
    const uint32_t box[3] = {BK, BN / CS, 1};
    make_map(&mx, L.x, 3, dims, str, box, L.prm.f16 != 0);
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(L.nj), static_cast<uint64_t>(L.rows_v)};
    const uint64_t str[1] = {static_cast<uint64_t>(L.ld_v) * 2};
    const uint32_t box[2] = {64, static_cast<uint32_t>(L.prm.n2)};
    make_map(&mv, L.v, 2, dims, str, box, L.prm.f16 != 0);
  }
  // per launch: the attribute is per device, and a static flag would race
  XCUDA(cudaFuncSetAttribute(ttm_fused_kernel<MPAD, Cfg, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::SMEM_TOTAL));
  if (L.prm.n_rb % CS) usage("ttm_fused: row blocks must be a multiple of the cluster size");
  const int clusters = (L.prm.n_rb / CS) * L.prm.kc;
  const int cap = (L.grid_limit > 0 ? L.grid_limit : sm_count()) / CS;
  const int grid = std::max(1, std::min(clusters, cap)) * CS;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = Cfg::SMEM_TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  XCUDA(cudaLaunchKernelEx(&cfg, ttm_fused_kernel<MPAD, Cfg, CS>, mu, mx, mv, L.prm));
  XLAUNCH_CHECK();
}

}  // namespace


void launch_ttm_fused(const TtmLaunch& L, cudaStream_t st) {
  if (L.prm.n2 > 128 || L.prm.n2 % 16 || L.prm.lpad * L.prm.rpb != BM)
    usage("ttm_fused: unsupported reduced dims for the tensor-core path");
  if (L.prm.comp) {
    // the compensated mode exists only as the CTA-pair kernel (plans round
    // their stacked rows up to whole pairs of row blocks)
    if (!ttm_pair_supported(L)) usage("ttm_fused: compensated mode needs the CTA-pair kernel shape");
    launch_ttm_pair(L, st);
    return;
  }
  if (ttm_pair_enabled() && ttm_pair_supported(L)) {
    launch_ttm_pair(L, st);  // cta_group::2 kernel (ttm_tc2.cu)
    return;
  }
  const int cs = (L.prm.n_rb % ttm_cluster_size() == 0) ? ttm_cluster_size() : 1;
  using C = TileCfg<256, 3>;
  auto go = [&](auto cs_tag) {
    constexpr int CS = decltype(cs_tag)::value;
    switch (L.mpad) {
      case 32: launch_impl<32, C, CS>(L, st); break;
      case 64: launch_impl<64, C, CS>(L, st); break;
      case 128: launch_impl<128, C, CS>(L, st); break;
      default: usage("ttm_fused: M must pad to 32, 64 or 128");
    }
  };
  if (cs == 4) go(std::integral_constant<int, 4>{});
  else if (cs == 2) go(std::integral_constant<int, 2>{});
  else go(std::integral_constant<int, 1>{});
}

// Cluster size for the X-tile multicast (XTSG_TTM_CLUSTER=1|2|4, default 2).
int ttm_cluster_size() {
  static const int cs = [] {
    const char* e = std::getenv("XTSG_TTM_CLUSTER");
    const int v = e ? std::atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  return cs;
}

int ttm_block_n() { return 256; }

// CTA-pair kernel on by default (XTSG_TTM_PAIR=0 selects the single-CTA one).
bool ttm_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("XTSG_TTM_PAIR");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

}  // namespace xtsg
