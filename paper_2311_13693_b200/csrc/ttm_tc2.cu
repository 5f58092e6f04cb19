// K2+K3 on CTA pairs — the cta_group::2 version of the fused TTM (ttm_tc.cu).
//
// Same contraction (Z_p[:, :, k] = U_p X[:, :, k] V_p^T for every replica and
// slice; reference comp_with, compression.cpp:202-209), but each tcgen05.mma
// spans the two SMs of a TPC: M = 256 stacked U rows (128 per CTA) x N = 256 j
// (each CTA stages only its 128 j of the X tile). Per SM this halves the X
// bytes TMA writes into shared memory and the B bytes the tensor core reads
// back, which is what capped the single-CTA kernel at ~2/3 tensor-pipe
// occupancy (ncu: smem shared between TMA fills and UMMA operand reads).
//
// Roles per CTA (256 threads): w0 TMA producer (own U rows + own half of the X
// tile, completing on the LEADER's full barrier), w1 TMEM owner and — leader
// only — mode-1 MMA issuer, w2 Vt producer, w3 — leader only — mode-2 MMA
// issuer, w4-7 epilogue over this CTA's 128 TMEM lanes. Commits multicast to
// both CTAs' barriers; the epilogues arrive remotely on the leader's.
//
// Mode 2 runs with the same cta_group (M = 256 rows = 2*RPB replicas,
// N = 2*RPB*Mpad <= 256 columns): D2 reuses the drained 256-column D1 buffer,
// so all D1 chunks that D2 overlaps are drained (a 4-deep A2 ring) before the
// first mode-2 MMA of a tile.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "sm100_ptx.cuh"
#include "ttm_tc.cuh"

namespace xtsg {

namespace {

constexpr int BM = 128;                 // rows per CTA (M = 256 per pair)
constexpr int BN = 256;                 // j per tile (128 staged per CTA)
constexpr int BNC = BN / 2;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;    // 16 KB
constexpr int B_BYTES = BNC * BK * 2;   // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int A2_BYTES = BM * 64 * 2;   // 16 KB
constexpr int B2_BYTES = 128 * 64 * 2;  // 16 KB (n2 <= 128 rows per CTA)
constexpr int CHUNKS = BN / 64;
// Compensated mode (XTSG_PREC_FP16X3): every operand is an fp16 pair
// (hi, lo = x - hi), each operand pre-scaled by a power of two so its largest
// value sits in [2^13, 2^14) (lo then stays a normal binary16 for every value
// within 2^16 of the maximum), and each product is hi*hi + hi*lo + lo*hi (the
// dropped lo*lo term is 2^-22 relative). One ring stage holds a whole 64-wide
// i step — (Uh, Ul, Xh, Xl), 64 KB per CTA — and the MMA issuer runs the three
// products (Uh, Xh), (Uh, Xl), (Ul, Xh) from it into the same accumulator; the
// epilogue splits the fp32 mode-1 result into an A2 (hi, lo) pair and mode 2
// issues (Th, Vh), (Th, Vl), (Tl, Vh) from a two-plane V slot.
// S ring stages, A2_SLOTS mode-1 chunks in flight to mode 2, B2_SLOTS V chunks.
constexpr int smem_total(int S, int A2_SLOTS, bool COMP = false, int B2_SLOTS = 2) {
  return S * STAGE_BYTES * (COMP ? 2 : 1) + A2_SLOTS * A2_BYTES * (COMP ? 2 : 1) +
         B2_SLOTS * B2_BYTES * (COMP ? 2 : 1) + 1024 + 512;
}
static_assert(smem_total(4, 4) <= 232448 && smem_total(5, 2) <= 232448, "shared memory budget");
static_assert(smem_total(2, 2, true, 1) <= 232448, "shared memory budget (compensated)");
constexpr uint32_t IDESC1 = ptx::idesc_bf16(2 * BM, BN);
constexpr uint16_t PAIR = 0x3;

// Unit u -> (slice kk, row-block pair rb2). Units are grouped by `group`
// row-block pairs: the ~#SM/2 units in flight at once then share `group`
// blocks of U (L2-resident however large P*L) while each X tile is read by
// `group` clusters at the same time (so from DRAM ~n_rb2/group times).
__device__ __forceinline__ void decode_unit(int u, int n_rb2, int kc, int group, int& kk, int& rb2) {
  const int g = u / (group * kc);
  const int rem = u - g * group * kc;
  const int gsz = min(group, n_rb2 - g * group);
  kk = rem / gsz;
  rb2 = g * group + (rem - kk * gsz);
}

// Persistent-cluster schedule over (slice kk, row-block pair rb2) units.
// lanes == 0: round robin over the grouped unit order (decode_unit).
// lanes > 0: static 2-D assignment — cluster c serves row block r = c % group
// of every group, on the slices kk = lane, lane + lanes, ... (lane = c /
// group), so the `group` clusters of a lane always work on the same slice and
// read each X tile together; with p.sync they also re-align at every slot.
struct UnitSched {
  int cid, n_clusters, n_rb2, kc, group, lanes, lane, r, ngroups;
  int u, g, kk, slot;
  __device__ UnitSched(int c, int nc, int nrb2, const TtmParams& p)
      : cid(c), n_clusters(nc), n_rb2(nrb2), kc(p.kc), group(p.rb_group), lanes(p.lanes) {
    lane = lanes ? cid / group : 0;
    r = lanes ? cid % group : 0;
    ngroups = (n_rb2 + group - 1) / group;
    u = cid - n_clusters;
    g = 0;
    kk = lane - lanes;
    slot = -1;
  }
  // next slot; active = this cluster has a unit in it
  __device__ bool next(bool& active, int& ukk, int& urb2) {
    if (!lanes) {
      u += n_clusters;
      if (u >= n_rb2 * kc) return false;
      decode_unit(u, n_rb2, kc, group, ukk, urb2);
      active = true;
      return true;
    }
    if (lane >= lanes) return false;
    kk += lanes;
    while (kk >= kc) {
      if (++g >= ngroups) return false;
      kk = lane;
    }
    ++slot;
    const int gsz = min(group, n_rb2 - g * group);
    active = r < gsz;
    ukk = kk;
    urb2 = g * group + r;
    return true;
  }
};

// Lane barrier between slots (performance only: bounded wait, then proceed).
__device__ __forceinline__ void lane_barrier(unsigned* ctr, unsigned target) {
  atomicAdd(ctr, 1u);
  for (int spin = 0; spin < 40000; ++spin) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(64);
  }
}

template <int S, int A2_SLOTS, int B2_SLOTS>
struct Bars2 {
  uint64_t full1[S], empty1[S];
  uint64_t tmem_full[2], tmem_empty[2], d2_full[2];
  uint64_t a2_full[A2_SLOTS], a2_empty[A2_SLOTS];
  uint64_t b2_full[B2_SLOTS], b2_empty[B2_SLOTS];
  uint32_t tmem_base;
};

// split of an fp32 value into the fp16 pair (hi, lo = v - hi)
__device__ __forceinline__ void split16x2(const float* v, uint4& hi, uint4& lo) {
  uint32_t wh[4], wl[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __half2 h = __floats2half2_rn(v[2 * q], v[2 * q + 1]);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(v[2 * q] - hf.x, v[2 * q + 1] - hf.y);
    wh[q] = *reinterpret_cast<const uint32_t*>(&h);
    wl[q] = *reinterpret_cast<const uint32_t*>(&l);
  }
  hi = make_uint4(wh[0], wh[1], wh[2], wh[3]);
  lo = make_uint4(wl[0], wl[1], wl[2], wl[3]);
}

template <int MPAD, bool LOCAL2, int S, int A2_SLOTS, bool COMP = false, int B2_SLOTS = 2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    ttm_pair_kernel(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_x,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_xl,
                    const TtmParams p) {
  static_assert(!COMP || LOCAL2, "the compensated mode runs mode 2 per CTA");
  constexpr int NC = COMP ? 3 : 1;                      // products per i step / per mode-2 chunk
  constexpr int CSTAGE = STAGE_BYTES * (COMP ? 2 : 1);  // (U[, Ul], X[, Xl]) tiles of one i step
  constexpr int A2_SLOT = A2_BYTES * (COMP ? 2 : 1);    // (Th[, Tl]) mode-2 A tiles
  constexpr int B2_SLOT = B2_BYTES * (COMP ? 2 : 1);    // (Vh[, Vl]) planes
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* a2_base = smem + S * CSTAGE;
  uint8_t* b2_base = a2_base + A2_SLOTS * A2_SLOT;
  auto* bars = reinterpret_cast<Bars2<S, A2_SLOTS, B2_SLOTS>*>(b2_base + B2_SLOTS * B2_SLOT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_ctarank();
  const bool leader = crank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&bars->full1[s], 1);
      ptx::mbar_init(&bars->empty1[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bars->tmem_full[b], 1);
      ptx::mbar_init(&bars->tmem_empty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy)
      ptx::mbar_init(&bars->d2_full[b], 1);
    }
    for (int b = 0; b < B2_SLOTS; ++b) {
      ptx::mbar_init(&bars->b2_full[b], 1);
      ptx::mbar_init(&bars->b2_empty[b], 1);
    }
    for (int q = 0; q < A2_SLOTS; ++q) {
      ptx::mbar_init(&bars->a2_full[q], LOCAL2 ? 4 : 8);
      ptx::mbar_init(&bars->a2_empty[q], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tm_u);
    ptx::tma_prefetch(&tm_x);
    ptx::tma_prefetch(&tm_v);
    if (COMP) ptx::tma_prefetch(&tm_xl);
  }
  if (warp == 1) ptx::tmem_alloc_pair(&bars->tmem_base, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  const int cid = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int n_rb2 = p.n_rb >> 1;
  const int j_tiles = p.j_tiles, k_steps = p.k_steps;
  // a tile is (j tile, i chunk): each i chunk of kpc steps gets its own
  // mode-1 accumulator and mode-2 pass (shorter fp32 TMEM sums), the mode-2
  // results of all chunks fold into the same register accumulators
  const int i_chunks = p.i_chunks > 0 ? p.i_chunks : 1, kpc = p.i_chunks > 0 ? p.kpc : k_steps;
  const int n_tiles = j_tiles * i_chunks;
  const int n2c = p.n2;            // mode-2 columns contributed by this CTA
  const int n2 = LOCAL2 ? n2c : 2 * n2c;  // mode-2 MMA N
  const int need = (n2 + 63) / 64;        // D1 chunks D2 overlaps

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own U rows, own half of the X tile -----
      int s = 0;
      uint32_t ph = 0;
      UnitSched us(cid, n_clusters, n_rb2, p);
      int kk, rb2;
      bool act;
      unsigned sync_no = 0;
      while (us.next(act, kk, rb2)) {
        const int urow = rb2 * 2 * BM + crank * BM;
        for (int t2 = 0; t2 < n_tiles; ++t2) {
          const int jt = t2 / i_chunks, ic = t2 - jt * i_chunks;
          // lane barrier every sync_j tiles (idle clusters of a partial group
          // keep arriving so the counts stay aligned)
          if (p.sync && ic == 0 && jt % p.sync_j == 0) lane_barrier(p.sync + us.lane, 2u * us.group * ++sync_no);
          if (!act) continue;
          const int ks1 = min(k_steps, (ic + 1) * kpc);
          // the last j tile runs with N = n_last: each CTA holds n_last / 2 of its j
          const int half = jt == j_tiles - 1 ? (p.n_last >> 1) : BNC;
          for (int ks = ic * kpc; ks < ks1; ++ks) {
            ptx::mbar_wait(&bars->empty1[s], ph ^ 1);
            uint8_t* st = stage_base + s * CSTAGE;
            if (leader) ptx::mbar_arrive_expect_tx(&bars->full1[s], 2 * CSTAGE);
            const uint32_t fb = ptx::mapa_shared(&bars->full1[s], 0);
#pragma unroll
            for (int c = 0; c < (COMP ? 2 : 1); ++c)
              ptx::tma_load_2d_pair_hint(st + c * A_BYTES, &tm_u, fb, ks * BK, urow + c * p.u_plane_rows, p.u_policy);
            uint8_t* xs = st + (COMP ? 2 : 1) * A_BYTES;
            ptx::tma_load_3d_pair_hint(xs, &tm_x, fb, ks * BK, jt * BN + crank * half, p.k_first + kk, p.x_policy);
            if (COMP)
              ptx::tma_load_3d_pair_hint(xs + B_BYTES, &tm_xl, fb, ks * BK, jt * BN + crank * half, p.k_first + kk,
                                         p.x_policy);
            if (++s == S) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---- mode-1 MMA issuer (leader) -----------------------------------------
      int s = 0;
      uint32_t ph = 0, t = 0;
      UnitSched us(cid, n_clusters, n_rb2, p);
      int kk, rb2;
      bool act;
      while (us.next(act, kk, rb2)) {
        if (!act) continue;
        for (int t2 = 0; t2 < n_tiles; ++t2, ++t) {
          const int jt = t2 / i_chunks, ic = t2 - jt * i_chunks;
          const uint32_t b = t & 1, use = t >> 1;
          ptx::mbar_wait(&bars->tmem_empty[b], (use & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t d = tmem + b * 256;
          const uint32_t idesc1 =
              (jt == j_tiles - 1 ? ptx::idesc_bf16(2 * BM, p.n_last) : IDESC1) & ptx::idesc_fmt_mask(p.f16 != 0);
          const int ks0 = ic * kpc, ks1 = min(k_steps, ks0 + kpc);
          for (int ks = ks0; ks < ks1; ++ks) {
            const int nk16 = ks == k_steps - 1 ? p.k16_last : BK / 16;
            ptx::mbar_wait(&bars->full1[s], ph);
            ptx::tc_fence_after();
            const uint32_t st0 = ptx::smem_u32(stage_base + s * CSTAGE);
            const uint32_t xs0 = st0 + (COMP ? 2 : 1) * A_BYTES;
            // products (U plane, X plane): (h, h)[, (h, l), (l, h)]
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const uint32_t a0 = st0 + (c == 2 ? A_BYTES : 0);
              const uint32_t b0 = xs0 + (c == 1 ? B_BYTES : 0);
#pragma unroll
              for (int k4 = 0; k4 < BK / 16; ++k4)
                if (k4 < nk16)
                  ptx::mma_bf16_pair(d, ptx::sw128_desc(a0 + k4 * 32), ptx::sw128_desc(b0 + k4 * 32), idesc1,
                                     (ks != ks0 || c != 0 || k4 != 0));
            }
            ptx::mma_commit_pair(&bars->empty1[s], PAIR);
            if (++s == S) { s = 0; ph ^= 1; }
          }
          ptx::mma_commit_pair(&bars->tmem_full[b], PAIR);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ---- Vt producer (both CTAs): this CTA's replicas' V rows ---------------
      uint32_t g = 0;
      const uint32_t bytes = static_cast<uint32_t>(n2c) * 128;
      UnitSched us(cid, n_clusters, n_rb2, p);
      int kk, rb2;
      bool act;
      while (us.next(act, kk, rb2)) {
        if (!act) continue;
        const int vrow = (rb2 * 2 + static_cast<int>(crank)) * n2c;
        for (int t2 = 0; t2 < n_tiles; ++t2) {
          const int jt = t2 / i_chunks;
          const int nch = jt == j_tiles - 1 ? p.chunks_last : CHUNKS;
          for (int c = 0; c < nch; ++c, ++g) {
            const int slot = g % B2_SLOTS;
            ptx::mbar_wait(&bars->b2_empty[slot], ((g / B2_SLOTS) & 1) ^ 1);
            if (LOCAL2) {
              ptx::mbar_arrive_expect_tx(&bars->b2_full[slot], bytes * (COMP ? 2 : 1));
#pragma unroll
              for (int pl = 0; pl < (COMP ? 2 : 1); ++pl)
                ptx::tma_load_2d(b2_base + slot * B2_SLOT + pl * B2_BYTES, &tm_v, &bars->b2_full[slot],
                                 jt * BN + c * 64, vrow + pl * p.v_plane_rows);
            } else {
              if (leader) ptx::mbar_arrive_expect_tx(&bars->b2_full[slot], 2 * bytes);
              ptx::tma_load_2d_pair(b2_base + slot * B2_SLOT, &tm_v, ptx::mapa_shared(&bars->b2_full[slot], 0),
                                    jt * BN + c * 64, vrow);
            }
          }
        }
      }
    }
  } else if (warp == 3) {
    if ((LOCAL2 || leader) && lane == 0) {
      // ---- mode-2 MMA issuer (leader; every CTA for the per-CTA variant) ------
      const uint32_t idesc2 = ptx::idesc_bf16(LOCAL2 ? BM : 2 * BM, n2) & ptx::idesc_fmt_mask(p.f16 != 0);
      uint32_t t = 0, g = 0;
      UnitSched us(cid, n_clusters, n_rb2, p);
      int kk, rb2;
      bool act;
      while (us.next(act, kk, rb2)) {
        if (!act) continue;
        for (int t2 = 0; t2 < n_tiles; ++t2, ++t) {
          const int jt = t2 / i_chunks;
          const uint32_t b = t & 1;
          const uint32_t d = tmem + b * 256;
          const bool last = jt == j_tiles - 1;
          const int nch = last ? p.chunks_last : CHUNKS;
          // D2 overwrites drained D1 columns: a region's first MMA waits until
          // the `need` chunks it overlaps are drained. Compensated tiles use
          // two D2 regions (chunks 0-1 -> columns [0, n2), chunks 2-3 ->
          // [128, 128 + n2)) so each fp32 mode-2 chain spans 24 MMAs, not 48.
          const uint32_t g0 = g;
          int waited = 0;
          for (int c = 0; c < nch; ++c, ++g) {
            const int rs = (COMP && c >= 2) ? 2 : 0;
            const int upto = c == rs ? (nch < rs + need ? nch : rs + need) : c + 1;
            for (; waited < upto; ++waited)
              ptx::mbar_wait(&bars->a2_full[(g0 + waited) % A2_SLOTS], ((g0 + waited) / A2_SLOTS) & 1);
            const uint32_t dr = d + (rs ? 128u : 0u);
            const int slot = g % A2_SLOTS, bslot = g % B2_SLOTS;
            ptx::mbar_wait(&bars->b2_full[bslot], (g / B2_SLOTS) & 1);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(a2_base + slot * A2_SLOT);
            const uint32_t b0 = ptx::smem_u32(b2_base + bslot * B2_SLOT);
            const int nk16 = (last && c == nch - 1) ? p.k16_chunk_last : 4;
            if (LOCAL2) {
              // (A2 tile, V plane) per product: (Th, Vh)[, (Th, Vl), (Tl, Vh)]
#pragma unroll
              for (int q = 0; q < NC; ++q) {
                const uint32_t aq = a0 + (q == 2 ? A2_BYTES : 0), bq = b0 + (q == 1 ? B2_BYTES : 0);
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4)
                  if (k4 < nk16)
                    ptx::mma_bf16(dr, ptx::sw128_desc(aq + k4 * 32), ptx::sw128_desc(bq + k4 * 32), idesc2,
                                  (c != rs || k4 != 0 || q != 0));
              }
              ptx::mma_commit(&bars->a2_empty[slot]);
              ptx::mma_commit(&bars->b2_empty[bslot]);
            } else {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
                if (k4 < nk16)
                  ptx::mma_bf16_pair(d, ptx::sw128_desc(a0 + k4 * 32), ptx::sw128_desc(b0 + k4 * 32), idesc2,
                                     (c | k4) != 0);
              ptx::mma_commit_pair(&bars->a2_empty[slot], PAIR);
              ptx::mma_commit_pair(&bars->b2_empty[bslot], PAIR);
            }
          }
          if (LOCAL2)
            ptx::mma_commit(&bars->d2_full[b]);
          else
            ptx::mma_commit_pair(&bars->d2_full[b], PAIR);
        }
      }
    }
  } else {
    // ---- epilogue (both CTAs): this CTA's 128 TMEM lanes ---------------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int p_local = r / p.lpad;
    const int l = r % p.lpad;
    const uint32_t d2col = (LOCAL2 ? 0u : crank * n2c) + p_local * MPAD;
    uint32_t t = 0, g = 0;
    UnitSched us(cid, n_clusters, n_rb2, p);
    int kk, rb2;
    bool act;
    // compensated: the mode-1 result (2^-(bu+sx) U X, operands scaled to
    // [2^13, 2^14)) is scaled by 2^-c0 into the binary16 range before the split
    const float t_scale = COMP ? exp2f(static_cast<float>(-p.comp_c0)) : 1.f;
    while (us.next(act, kk, rb2)) {
      if (!act) continue;
      float zacc[MPAD];
#pragma unroll
      for (int m = 0; m < MPAD; ++m) zacc[m] = 0.f;
      for (int t2 = 0; t2 < n_tiles; ++t2, ++t) {
        const int jt = t2 / i_chunks;
        const uint32_t b = t & 1, use = t >> 1;
        const int nch = jt == j_tiles - 1 ? p.chunks_last : CHUNKS;
        ptx::mbar_wait(&bars->tmem_full[b], use & 1);
        ptx::tc_fence_after();
        for (int c = 0; c < nch; ++c, ++g) {
          const int slot = g % A2_SLOTS;
          ptx::mbar_wait(&bars->a2_empty[slot], ((g / A2_SLOTS) & 1) ^ 1);
          uint8_t* row = a2_base + slot * A2_SLOT + r * 128;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            float v[32];
            ptx::tmem_ld32(lane_addr + b * 256 + c * 64 + h * 32, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int q8 = h * 4 + q4;
              if (COMP) {
                float w8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) w8[e] = v[q4 * 8 + e] * t_scale;
                uint4 hi, lo;
                split16x2(w8, hi, lo);
                *reinterpret_cast<uint4*>(row + ((q8 ^ (r & 7)) << 4)) = hi;
                *reinterpret_cast<uint4*>(row + A2_BYTES + ((q8 ^ (r & 7)) << 4)) = lo;
              } else {
                const uint4 pk = ptx::pack8(v + q4 * 8, p.f16 != 0);
                *reinterpret_cast<uint4*>(row + ((q8 ^ (r & 7)) << 4)) = pk;
              }
            }
          }
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (LOCAL2)
              ptx::mbar_arrive(&bars->a2_full[slot]);
            else
              ptx::mbar_arrive_cluster(ptx::mapa_shared(&bars->a2_full[slot], 0));
          }
        }
        ptx::mbar_wait(&bars->d2_full[b], use & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int mc = 0; mc < MPAD / 32; ++mc) {
          float v[32];
          ptx::tmem_ld32(lane_addr + b * 256 + d2col + mc * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) zacc[mc * 32 + e] += v[e];
        }
        if (COMP && nch > 2) {
#pragma unroll
          for (int mc = 0; mc < MPAD / 32; ++mc) {
            float v[32];
            ptx::tmem_ld32(lane_addr + b * 256 + 128 + d2col + mc * 32, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) zacc[mc * 32 + e] += v[e];
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa_shared(&bars->tmem_empty[b], 0));
      }
      const int prep = (rb2 * 2 + static_cast<int>(crank)) * p.rpb + p_local;
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
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(tmem, 512);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn2() {
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

void map_bf16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
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
  const CUresult r = encode_fn2()(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, bx, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Status(XTSG_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

template <int MPAD, bool LOCAL2, int S, int A2_SLOTS, bool COMP = false, int B2_SLOTS = 2>
void launch_pair(const TtmLaunch& L, cudaStream_t st) {
  CUtensorMap mu, mx, mv, mxl;
  {
    // compensated: two U planes (hi, lo) of rows_u rows each, stacked
    const uint64_t dims[2] = {static_cast<uint64_t>(L.ni), static_cast<uint64_t>(L.rows_u * (COMP ? 2 : 1))};
    const uint64_t str[1] = {static_cast<uint64_t>(L.ld_u) * 2};
    const uint32_t box[2] = {BK, BM};
    map_bf16(&mu, L.u, 2, dims, str, box, L.prm.f16 != 0);
  }
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(L.ni), static_cast<uint64_t>(L.nj), static_cast<uint64_t>(L.nk)};
    const uint64_t str[2] = {static_cast<uint64_t>(L.ld_x0) * 2, static_cast<uint64_t>(L.ld_x1) * 2};
    const uint32_t box[3] = {BK, BNC, 1};
    map_bf16(&mx, L.x, 3, dims, str, box, L.prm.f16 != 0);
    if (COMP) map_bf16(&mxl, L.x_lo, 3, dims, str, box, true);
    else mxl = mx;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(L.nj), static_cast<uint64_t>(L.rows_v * (COMP ? 2 : 1))};
    const uint64_t str[1] = {static_cast<uint64_t>(L.ld_v) * 2};
    const uint32_t box[2] = {64, static_cast<uint32_t>(L.prm.n2)};
    map_bf16(&mv, L.v, 2, dims, str, box, L.prm.f16 != 0);
  }
  constexpr int SMEM_TOTAL = smem_total(S, A2_SLOTS, COMP, B2_SLOTS);
  // per launch: the attribute is per device, and a static flag would race
  XCUDA(cudaFuncSetAttribute(ttm_pair_kernel<MPAD, LOCAL2, S, A2_SLOTS, COMP, B2_SLOTS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL));
  const int clusters = (L.prm.n_rb / 2) * L.prm.kc;
  const int cap = (L.grid_limit > 0 ? L.grid_limit : sm_count()) / 2;
  const int ncl = std::max(1, std::min(clusters, cap));
  const int grid = ncl * 2;
  TtmParams prm = L.prm;
  // schedule (UnitSched): 0 round robin, 1 static lanes, 2 static lanes with a
  // per-slot lane barrier; static lanes need at least one slice per lane
  static const int sched_env = [] {
    const char* e = std::getenv("XTSG_TTM_SCHED");
    return e ? std::atoi(e) : 2;
  }();
  const int lanes = ncl / std::max(1, prm.rb_group);
  prm.lanes = (sched_env && lanes >= 1 && lanes <= prm.kc) ? lanes : 0;
  prm.sync = nullptr;
  static const int syncj_env = [] {
    const char* e = std::getenv("XTSG_TTM_SYNCJ");
    return e ? std::atoi(e) : 0;
  }();
  // lane barrier spacing: once per slice when a slice is a few j tiles (C2:
  // 8), every 4 j tiles for large slices (C3: 40 tiles, 200 MB per slice; the
  // group's clusters drift apart within a slice and re-read X from DRAM).
  // Measured at C3 (tools/c3_syncj_ab.sh, c3_traffic_sweep.sh): DRAM reads
  // 190 -> 161 GB per 40-slice launch, 1072 -> 1091 TF/s (3 alternating reps)
  prm.sync_j = syncj_env > 0 ? syncj_env : (prm.j_tiles >= 16 ? 4 : prm.j_tiles);
  if (prm.lanes && sched_env == 2 && L.sync) {
    XCUDA(cudaMemsetAsync(L.sync, 0, sizeof(unsigned) * prm.lanes, st));
    prm.sync = L.sync;
  }
  prm.u_plane_rows = static_cast<int32_t>(L.rows_u);
  prm.v_plane_rows = static_cast<int32_t>(L.rows_v);
  ttm_pair_kernel<MPAD, LOCAL2, S, A2_SLOTS, COMP, B2_SLOTS><<<grid, 256, SMEM_TOTAL, st>>>(mu, mx, mv, mxl, prm);
  XLAUNCH_CHECK();
}

}  // namespace

bool ttm_pair_supported(const TtmLaunch& L) {
  return L.prm.n_rb % 2 == 0 && L.prm.n2 <= 128 && L.prm.lpad * L.prm.rpb == BM && (!L.prm.comp || L.x_lo);
}

void launch_ttm_pair(const TtmLaunch& L, cudaStream_t st) {
  if (!ttm_pair_supported(L)) usage("ttm_pair: unsupported shape for the CTA-pair kernel");
  // 0: mode 2 on the pair (M = 256); 1: mode 2 per CTA (cta_group::1, M = 128,
  // half the wasted columns), 4 stages; 2 (default): per-CTA mode 2, 5 stages /
  // 2 A2 slots — measured back to back on one box: C2 29.2 -> 28.4 ms/step,
  // every C5 (L, P) point +1-5 %, C3 equal (profiles/r1_pair_variants.json)
  static const int variant = [] {
    const char* e = std::getenv("XTSG_TTM_PAIR_CFG");
    return e ? std::atoi(e) : 2;
  }();
  auto go = [&](auto mpad_tag) {
    constexpr int MP = decltype(mpad_tag)::value;
    if (L.prm.comp)
      launch_pair<MP, true, 2, 2, true, 1>(L, st);
    else if (variant == 0)
      launch_pair<MP, false, 4, 4>(L, st);
    else if (variant == 1)
      launch_pair<MP, true, 4, 4>(L, st);
    else
      launch_pair<MP, true, 5, 2>(L, st);
  };
  switch (L.mpad) {
    case 32: go(std::integral_constant<int, 32>{}); break;
    case 64: go(std::integral_constant<int, 64>{}); break;
    case 128: go(std::integral_constant<int, 128>{}); break;
    default: usage("ttm_pair: M must pad to 32, 64 or 128");
  }
}

}  // namespace xtsg
