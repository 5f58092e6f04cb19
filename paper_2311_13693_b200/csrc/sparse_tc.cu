// K7 (tensor-core form) — sparse compression as dense tiles of a mode-3 slice.
//
// Eq. 3 restricted to the nonzeros (no reference counterpart):
//   Z_k = sum_{(i,j) in slice k} x_ijk * U[:, i] (x) V_p[:, j]   (per replica)
// then mode 3 over the slices exactly like the dense path (coo.cu
// sparse_mode3).
//
// The SIMT fiber kernel (coo.cu) gathers a 1 KB stacked U column per nonzero
// and spends P*L FMAs on it; nothing is reused across the fibers of a slice.
// Here a slice is cut into tiles of up to 64 fibers whose nonzeros touch at
// most 512 distinct i, and both mode products of a tile run on the tensor
// cores, so a U column is gathered once per tile instead of once per nonzero.
//
//   1. sparse_plan_kernel (several CTAs per SM, one per slice at a time): a
//      shared-memory hash i -> local id that stays warm across the slice's
//      tiles (one lookup pass per nonzero when the tile adds no new i; else
//      claim + ids in slot order + lookup), table epochs whose id -> i lists
//      go to si_g, a 16-bit code (tile fiber << 9 | id) per nonzero in li_g,
//      a descriptor per tile; duplicate coordinates inside a tile are flagged.
//   2. sparse_tc_kernel (one CTA per SM, 16 warps, planned tiles in a static
//      order with the next tile prefetched to L2): warps 0-1 and 8-15 scatter
//      the tile's values into a dense bf16 tile Xd[fiber][id] (K-major
//      SWIZZLE_128B; CAS adds only for flagged tiles) while warps 2-7 gather
//      the tile's U columns from the i-major copy Ut[i][(p, l)] (64-byte
//      cp.async tasks into MN-major SWIZZLE_128B stages, 5-slot ring) and the
//      V rows of its fibers (3 buffers); one thread issues mode 1 (M = 128
//      stacked rows, N = 64 fibers, K = ids, A MN-major) and mode 2 (N =
//      (128/Lpad)*Mpad, B MN-major) with mode 2 of block rb-1 after mode 1 of
//      block rb; warps 8-15 drain D1 to bf16 and add the diagonal replica
//      blocks of D2 into Z with fire-and-forget reductions.
// Per nonzero: 4 B (planner) + 6 B (tensor kernel) from HBM, 2 B written;
// per tile 2*PL*64*ni + 2*PL*64*N2 tensor flops and ni*PL*2 B of U over L2.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cub/cub.cuh>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "plan.cuh"
#include "sm100_ptx.cuh"

namespace xtsg {

namespace {

constexpr int SP_NT = 512;   // tensor kernel: 16 warps
constexpr int PL_NT = 256;   // planner: 8 warps, several CTAs per SM
constexpr int SP_NF = 64;    // fibers per tile (mode-1 UMMA N, mode-2 K)
constexpr int SP_NI = 512;   // distinct i per tile (mode-1 K)
constexpr int SP_HS = 2048;  // planner hash slots (<= SP_NI + PL_NT claims)
constexpr int SP_NS = 5;     // U gather ring slots
constexpr int SP_AHEAD = 4;  // cp.async groups in flight per producer
constexpr int SP_NV = 3;     // V-row buffers: the producer never waits on the mode-2 MMA it feeds
constexpr int SC_NT = 320;   // scatter team: warps 0, 1, 8-15 (the producers gather meanwhile)
constexpr int XD_CHUNK = SP_NF * 128;              // 64 fibers x 64 i, 8 KB
constexpr int XD_BYTES = (SP_NI / 64) * XD_CHUNK;  // 64 KB
constexpr int UC_BYTES = 128 * 64 * 2;             // 128 rows x 64 i, 16 KB
constexpr int A2_BYTES = 128 * 128;                // 128 rows x 64 fibers
constexpr int VG_BYTES = 128 * 64 * 2;             // 128 (p, m) x 64 fibers (x SP_NV buffers)

// one planned tile: fibers [f0, f0 + nf) of slice s, nonzeros [e0, e0 + n)
// (a piece of one fiber when nf == 1 and the fiber is longer), local ids
// 0..ni-1 standing for si_g[si0 ..), each nonzero's id at li_g[e]
struct SpTile {
  int64_t e0, f0, si0;  // first nonzero, first fiber, id -> i list at si_g[si0 ..)
  int32_t s, n, nf, ni, dup, pad;
};

struct SpMisc {
  uint64_t full[SP_NS], empty[SP_NS];  // U gather ring
  uint64_t vg_full[SP_NV], vg_empty[SP_NV];  // V rows (mode-2 B)
  uint64_t d1_full[2], d1_empty[2];    // mode-1 accumulator (TMEM, double-buffered)
  uint64_t a2_full, d2_full, d2_empty;
  uint64_t xd_full;                    // the tile's dense X is in shared memory
  uint32_t tmem_base;
  int64_t tile;
  SpTile t;
};

constexpr int OFF_RING = XD_BYTES;
constexpr int OFF_A2 = OFF_RING + SP_NS * UC_BYTES;
constexpr int OFF_VG = OFF_A2 + A2_BYTES;
constexpr int OFF_SI = OFF_VG + SP_NV * VG_BYTES;
constexpr int OFF_TFP = OFF_SI + SP_NI * 4;
constexpr int OFF_TFJ = OFF_TFP + (SP_NF + 2) * 4;
constexpr int OFF_MISC = OFF_TFJ + SP_NF * 4;
constexpr int SP_SMEM = OFF_MISC + static_cast<int>(sizeof(SpMisc)) + 1024;
static_assert(SP_SMEM <= 232448, "shared memory budget");

struct SpPlanParams {
  const int64_t* slice_ptr;  // n_slices + 1 fiber offsets
  const int64_t* fiber_ptr;  // nonzero offsets per fiber
  const int32_t* nz_i;
  int64_t n_slices;
  int32_t* si_g;    // nnz: a tile's distinct i at [e0, e0 + ni)
  uint16_t* li_g;   // nnz: local id of each nonzero
  SpTile* tiles;
  int64_t max_tiles;
  unsigned long long* counters;  // [0] slice counter, [1] tile count
};

struct SpTcParams {
  const int64_t* fiber_ptr;
  const int32_t* fiber_j;
  const float* val;
  const int32_t* si_g;
  const uint16_t* li_g;
  const SpTile* tiles;
  const unsigned long long* n_tiles;
  int64_t max_tiles;
  unsigned long long* counter;
  int64_t n_slices;
  const __nv_bfloat16* ut;  // [I][ld_ut], row (p, l) contiguous
  int64_t ld_ut;
  const __nv_bfloat16* vtj;  // [J][ld_vtj], (p, m) contiguous
  int64_t ld_vtj;
  int lpad, mpad, nrb, n2;
  int64_t vp;
  float* z;  // [vp][n_slices][mpad][lpad]
};

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// shared-space atomics (generic-pointer atomics compile to the slower ATOM.E)
__device__ __forceinline__ int atoms_cas(int* p, int cmp, int v) {
  int old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(ptx::smem_u32(p)), "r"(cmp), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int atoms_add(int* p, int v) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(ptx::smem_u32(p)), "r"(v) : "memory");
  return old;
}

// x += v on a 16-bit float at shared address a (bf16 or fp16): CAS on its
// 32-bit word (sm_100 has no native shared-memory float reduction)
template <bool F16>
__device__ __forceinline__ void atoms_add16(uint32_t a, float v) {
  const uint32_t w = a & ~3u, sh = (a & 2u) * 8u;
  uint32_t old;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(old) : "r"(w) : "memory");
  for (;;) {
    const uint16_t cur = static_cast<uint16_t>(old >> sh);
    uint16_t nv;
    if constexpr (F16) nv = __half_as_ushort(__float2half_rn(__half2float(__ushort_as_half(cur)) + v));
    else nv = __bfloat16_as_ushort(__float2bfloat16_rn(__bfloat162float(__ushort_as_bfloat16(cur)) + v));
    const uint32_t repl = (old & ~(0xFFFFu << sh)) | (static_cast<uint32_t>(nv) << sh);
    uint32_t prev;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(w), "r"(old), "r"(repl) : "memory");
    if (prev == old) return;
    old = prev;
  }
}

// volatile shared-memory loads (a generic volatile pointer becomes a slow system-scope load)
__device__ __forceinline__ int lds_volatile(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(p)));
  return v;
}
__device__ __forceinline__ uint16_t lds_volatile16(const uint16_t* p) {
  uint16_t v;
  asm volatile("ld.volatile.shared.u16 %0, [%1];" : "=h"(v) : "r"(ptx::smem_u32(p)));
  return v;
}

__device__ __forceinline__ uint32_t sp_hash(int32_t key) {
  return (static_cast<uint32_t>(key) * 2654435761u) >> (32 - 11);
}

// Batched visitor over nonzeros [e0, e1) (e1 - e0 < 2^30) with NT threads:
// f(n, xs, ks) with n <= 4*U valid entries (xs = e - e0, ascending per
// thread; ks the i), 16-byte loads, U in flight per thread; the batch lets f
// keep its shared-memory round trips in flight together.
template <int NT, int U, class F>
__device__ __forceinline__ void for_each_i(const int32_t* __restrict__ nz_i, int64_t e0, int64_t e1, F&& f) {
  constexpr int B = 4 * U;
  const int tid = threadIdx.x;
  const int64_t a0 = min(e1, (e0 + 3) & ~int64_t(3));
  const int64_t a1 = max(a0, e1 & ~int64_t(3));
  int xs[B];
  int32_t ks[B];
  if (e0 + tid < a0) {  // head: fewer than 4 entries
    xs[0] = tid;
    ks[0] = __ldg(nz_i + e0 + tid);
    f(1, xs, ks);
  }
  const int4* vi = reinterpret_cast<const int4*>(nz_i + a0);
  const int nv = static_cast<int>((a1 - a0) >> 2), xa = static_cast<int>(a0 - e0);
  for (int b = 0; b < nv; b += NT * U) {
    int n = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = b + u * NT + tid;
      if (idx < nv) {
        const int4 x = __ldg(vi + idx);
        ks[4 * u] = x.x;
        ks[4 * u + 1] = x.y;
        ks[4 * u + 2] = x.z;
        ks[4 * u + 3] = x.w;
#pragma unroll
        for (int q = 0; q < 4; ++q) xs[4 * u + q] = xa + idx * 4 + q;
        n = 4 * (u + 1);
      }
    }
    if (n) f(n, xs, ks);
  }
  if (a1 + tid < e1) {  // tail: fewer than 4 entries
    xs[0] = static_cast<int>(a1 + tid - e0);
    ks[0] = __ldg(nz_i + a1 + tid);
    f(1, xs, ks);
  }
}

// ---------------------------------------------------------------------------
// Planner: one CTA per slice (dynamic), cuts it into tiles of <= 64 fibers
// with <= 512 distinct i and writes, per tile, a descriptor and the local id
// of every nonzero (li_g). One pass per nonzero: the i -> id table persists
// across the tiles of a slice (their i supports usually coincide) and a new i
// gets the next id when it is first claimed. A table epoch (the tiles between
// two clears) writes its id -> i list once, at si_g[first nonzero of the
// epoch ...) (an epoch holds at least as many nonzeros as committed ids), and
// its tiles use a prefix of it. When a tile pushes the table past 512 ids the
// epoch is closed, the table cleared and the tile redone; if it overflows a
// fresh table it is retried with half the fibers (a long fiber is cut into
// 512-nonzero pieces). Duplicate coordinates inside a tile are flagged (the
// tensor kernel then sums them with atomics; otherwise it stores).
__global__ void __launch_bounds__(PL_NT, 4) sparse_plan_kernel(const SpPlanParams p) {
  __shared__ int keys[SP_HS];
  __shared__ uint16_t lis[SP_HS];
  __shared__ uint32_t seen[SP_NF * SP_NI / 32];  // (fiber, id) occupancy bits
  __shared__ int32_t tfp[SP_NF + 1];            // fiber starts relative to the tile
  __shared__ int32_t idkey[SP_NI];              // id -> i of the current epoch
  __shared__ int count, ovf, dup, wsum[PL_NT / 32];
  __shared__ int64_t slice;
  const int tid = threadIdx.x;
  // empty table: no keys, no ids (a claimed slot shows 0xFFFF until its id is published)
  auto clear_table = [&]() {
    for (int t = tid; t < SP_HS; t += PL_NT) {
      keys[t] = -1;
      lis[t] = 0xFFFF;
    }
    if (tid == 0) count = 0;
  };
  clear_table();
  for (;;) {
    if (tid == 0) slice = static_cast<int64_t>(atomicAdd(p.counters, 1ull));
    __syncthreads();
    const int64_t s = slice;
    if (s >= p.n_slices) break;
    const int64_t fs0 = p.slice_ptr[s], fs1 = p.slice_ptr[s + 1];
    int64_t f = fs0, e_in = fs1 > fs0 ? p.fiber_ptr[fs0] : 0;
    int64_t epoch0 = e_in;  // first nonzero of the current table epoch
    int committed = 0;      // ids used by the epoch's finished tiles
    int nt = SP_NF;
    // close the epoch: its committed ids -> si_g, then an empty table
    auto close_epoch = [&]() {
      for (int t = tid; t < committed; t += PL_NT) p.si_g[epoch0 + t] = idkey[t];
      clear_table();
      committed = 0;
      __syncthreads();
    };
    while (f < fs1) {
      int nf = static_cast<int>(imin64(nt, fs1 - f));
      const int64_t fend0 = p.fiber_ptr[f + 1];
      if (nt > 1 && p.fiber_ptr[f + nf] - e_in > (int64_t(1) << 30)) nt = nf = 1;
      const int64_t e_end = nt == 1 ? imin64(fend0, e_in + SP_NI) : p.fiber_ptr[f + nf];
      int64_t f_next = f + nf, e_next;
      if (nt == 1 && e_end < fend0) {
        f_next = f;
        e_next = e_end;
      } else {
        if (nt == 1) f_next = f + 1;
        e_next = f_next < fs1 ? p.fiber_ptr[f_next] : 0;
      }
      if (e_end == e_in) {  // empty fibers only
        f = f_next;
        e_in = e_next;
        continue;
      }
      for (int t = tid; t <= nf; t += PL_NT)
        tfp[t] = t == 0 ? 0 : static_cast<int32_t>((t == nf ? e_end : p.fiber_ptr[f + t]) - e_in);
      if (tid == 0) {  // the next tile's i (about as many as this one's) into L2
        const int64_t n = e_end - e_in, es1 = p.fiber_ptr[fs1];
        const int64_t pa = (e_end + 3) & ~int64_t(3), pb = imin64(es1, e_end + n) & ~int64_t(3);
        if (pb > pa) ptx::bulk_prefetch_l2(p.nz_i + pa, static_cast<uint32_t>(imin64((pb - pa) * 4, 1 << 20)));
      }
      // lookup pass: id of every nonzero -> li_g, (fiber, id) occupancy ->
      // dup; an i without an id sets `miss` (and the pass stops early)
      auto lookup = [&]() {
        int fl = 0;
        for_each_i<PL_NT, 2>(p.nz_i, e_in, e_end, [&](int n, const int* xs, const int32_t* ks) {
          constexpr int B = 8;
          uint32_t h[B];
          int li[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {  // first probes in flight together
            h[e] = sp_hash(ks[e]);
            li[e] = e < n ? keys[h[e]] : 0;
          }
          if (lds_volatile(&ovf)) return;
          bool m = false;
#pragma unroll
          for (int e = 0; e < B; ++e) {
            if (e >= n) continue;
            uint32_t hp = h[e];
            int k2 = li[e];
            while (k2 != ks[e] && k2 != -1) {
              hp = (hp + 1) & (SP_HS - 1);
              k2 = keys[hp];
            }
            li[e] = k2 == -1 ? 0xFFFF : lis[hp];
            m |= li[e] == 0xFFFF;
          }
          if (m) {
            ovf = 1;  // here: a miss
            return;
          }
#pragma unroll
          for (int e = 0; e < B; ++e) {
            if (e >= n) continue;
            while (tfp[fl + 1] <= xs[e]) ++fl;
            p.li_g[e_in + xs[e]] = static_cast<uint16_t>((fl << 9) | li[e]);  // fiber (6 bits) | id (9 bits)
            const int bit = fl * SP_NI + li[e];
            // occupancy of (fiber, id): fire-and-forget; duplicates show as
            // fewer set bits than nonzeros (counted after the pass)
            asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(ptx::smem_u32(&seen[bit >> 5])), "r"(1u << (bit & 31))
                         : "memory");
          }
        });
      };
      bool hit = false;
      if (committed > 0) {  // a warm table usually holds all of the tile's i
        for (int t = tid; t < SP_NF * SP_NI / 32; t += PL_NT) seen[t] = 0;
        if (tid == 0) {
          ovf = 0;
          dup = 0;
        }
        __syncthreads();
        lookup();
        __syncthreads();
        hit = lds_volatile(&ovf) == 0;
        __syncthreads();
      }
      if (!hit) {
        // claim slots for the new i (ids afterwards, in slot order)
        if (tid == 0) ovf = 0;
        __syncthreads();
        for_each_i<PL_NT, 2>(p.nz_i, e_in, e_end, [&](int n, const int*, const int32_t* ks) {
          constexpr int B = 8;
          uint32_t h[B];
          int k2[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            h[e] = sp_hash(ks[e]);
            k2[e] = e < n ? keys[h[e]] : 0;
          }
          if (lds_volatile(&ovf)) return;
#pragma unroll
          for (int e = 0; e < B; ++e) {
            if (e >= n || k2[e] == ks[e]) continue;
            const int32_t key = ks[e];
            uint32_t hp = h[e];
            int old = k2[e];
            for (;;) {
              if (old == key) break;
              if (old == -1) {
                if (lds_volatile(&count) >= SP_NI) {  // bounds the claims: <= SP_NI + PL_NT < SP_HS slots
                  ovf = 1;
                  break;
                }
                old = atoms_cas(&keys[hp], -1, key);
                if (old == -1) {
                  if (atoms_add(&count, 1) >= SP_NI) ovf = 1;
                  break;
                }
                continue;  // lost the race for this slot: look at what landed there
              }
              hp = (hp + 1) & (SP_HS - 1);
              old = keys[hp];
            }
          }
        });
        __syncthreads();
        if (lds_volatile(&ovf)) {
          const bool fresh = committed == 0;
          __syncthreads();
          if (fresh) {  // too many distinct i even alone: fewer fibers
            clear_table();
            __syncthreads();
            nt = max(1, nt >> 1);
          } else {      // close the epoch and redo this tile on an empty table
            close_epoch();
            epoch0 = e_in;
          }
          continue;
        }
        // ids for the new keys, in slot order (thread t owns SP_HS / PL_NT slots)
        {
          constexpr int SPT = SP_HS / PL_NT;
          const int lane = tid & 31, warp = tid >> 5;
          int c = 0;
#pragma unroll
          for (int k = 0; k < SPT; ++k) c += keys[tid * SPT + k] != -1 && lis[tid * SPT + k] == 0xFFFF;
          int incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane == 31) wsum[warp] = incl;
          __syncthreads();
          int base = incl - c + committed;
          for (int w = 0; w < warp; ++w) base += wsum[w];
#pragma unroll
          for (int k = 0; k < SPT; ++k) {
            const int key = keys[tid * SPT + k];
            if (key != -1 && lis[tid * SPT + k] == 0xFFFF) {
              lis[tid * SPT + k] = static_cast<uint16_t>(base);
              idkey[base] = key;
              ++base;
            }
          }
        }
        for (int t = tid; t < SP_NF * SP_NI / 32; t += PL_NT) seen[t] = 0;
        if (tid == 0) {
          ovf = 0;
          dup = 0;
        }
        __syncthreads();
        lookup();
        __syncthreads();
      }
      committed = lds_volatile(&count);
      {  // duplicate coordinates <=> fewer occupied (fiber, id) cells than nonzeros
        int c = 0;
        for (int w = tid; w < nf * (SP_NI / 32); w += PL_NT) c += __popc(seen[w]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((tid & 31) == 0) wsum[tid >> 5] = c;
        __syncthreads();
        if (tid == 0) {
          int tot = 0;
          for (int w = 0; w < PL_NT / 32; ++w) tot += wsum[w];
          dup = tot != static_cast<int>(e_end - e_in);
        }
        __syncthreads();
      }
      if (tid == 0) {
        const unsigned long long t = atomicAdd(p.counters + 1, 1ull);
        if (static_cast<int64_t>(t) < p.max_tiles) {
          SpTile d;
          d.e0 = e_in;
          d.f0 = f;
          d.si0 = epoch0;
          d.s = static_cast<int32_t>(s);
          d.n = static_cast<int32_t>(e_end - e_in);
          d.nf = nf;
          d.ni = committed;
          d.dup = dup;
          p.tiles[t] = d;
        }
      }
      f = f_next;
      e_in = e_next;
      nt = (f < fs1 && e_in != p.fiber_ptr[f]) ? 1 : min(SP_NF, nt * 2);
    }
    close_epoch();
  }
}

// ---------------------------------------------------------------------------
// Tensor kernel: one CTA per SM takes planned tiles off a counter (any order:
// the Z contributions are reductions). Per tile all warps scatter the values
// into the dense tile Xd (plain stores; shared-memory CAS adds when the
// planner saw duplicates), then the row blocks run on the roles below.
template <bool F16>
__global__ void __launch_bounds__(SP_NT, 1) sparse_tc_kernel(const SpTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xd = sm;
  uint8_t* ring = sm + OFF_RING;
  uint8_t* a2 = sm + OFF_A2;
  uint8_t* vg = sm + OFF_VG;
  int32_t* si = reinterpret_cast<int32_t*>(sm + OFF_SI);
  int32_t* tfp = reinterpret_cast<int32_t*>(sm + OFF_TFP);  // fiber starts, local offsets
  int32_t* tfj = reinterpret_cast<int32_t*>(sm + OFF_TFJ);
  SpMisc* ms = reinterpret_cast<SpMisc*>(sm + OFF_MISC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < SP_NS; ++s) {
      ptx::mbar_init(&ms->full[s], 192);
      ptx::mbar_init(&ms->empty[s], 1);
    }
    for (int b = 0; b < SP_NV; ++b) {
      ptx::mbar_init(&ms->vg_full[b], 192);
      ptx::mbar_init(&ms->vg_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&ms->d1_full[b], 1);
      ptx::mbar_init(&ms->d1_empty[b], 256);
    }
    ptx::mbar_init(&ms->a2_full, 256);
    ptx::mbar_init(&ms->d2_full, 1);
    ptx::mbar_init(&ms->d2_empty, 256);
    ptx::mbar_init(&ms->xd_full, SC_NT);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(&ms->tmem_base, 256);
  // stale operand bytes beyond a partial chunk must be finite (they multiply zeros)
  for (int e = tid; e < (SP_NS * UC_BYTES + A2_BYTES + SP_NV * VG_BYTES) / 16; e += SP_NT)
    reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = ms->tmem_base;
  const uint32_t d1 = tmem, d2 = tmem + 128;
  const uint32_t idesc1 = (ptx::idesc_bf16(128, SP_NF) | ptx::IDESC_A_MN) & ptx::idesc_fmt_mask(F16);
  const uint32_t idesc2 = (ptx::idesc_bf16(128, p.n2) | ptx::IDESC_B_MN) & ptx::idesc_fmt_mask(F16);
  const int q = warp & 3;
  const int r = q * 32 + lane;  // row of the 128-row block == TMEM lane
  const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
  const int p_local = r / p.lpad, l = r % p.lpad;
  const int rpb = 128 / p.lpad;
  const int half = p.mpad >> 1;
  const uint32_t ring_u = ptx::smem_u32(ring), xd_u = ptx::smem_u32(xd);
  const int64_t n_tiles = imin64(static_cast<int64_t>(*p.n_tiles), p.max_tiles);
  uint32_t g = 0, rbs = 0;  // U chunk and row-block sequence numbers (barrier phases)

  const bool scatterer = warp < 2 || warp >= 8;
  const int st = warp < 2 ? tid : tid - 192;  // rank in the scatter team
  for (int64_t it = 0;; ++it) {
    // static tile order (the planner's tiles are alike in size): the next
    // tile of this CTA is known, so its nonzeros are pulled into L2 now
    const int64_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= n_tiles) break;
    const SpTile T = p.tiles[tile];
    if (tid == 0 && tile + gridDim.x < n_tiles) {
      const SpTile Tn = p.tiles[tile + gridDim.x];
      const int64_t a = Tn.e0 & ~int64_t(7), b = (Tn.e0 + Tn.n + 7) & ~int64_t(7);
      ptx::bulk_prefetch_l2(p.li_g + a, static_cast<uint32_t>(imin64((b - a) * 2, 1 << 20)));
      ptx::bulk_prefetch_l2(p.val + a, static_cast<uint32_t>(imin64((b - a) * 4, 1 << 20)));
    }
    const int64_t s = T.s, e0 = T.e0;
    const int nf = T.nf, ni = T.ni, nnz = T.n;
    for (int t = tid; t <= nf; t += SP_NT)
      tfp[t] = t == 0 ? 0 : (t == nf ? nnz : static_cast<int32_t>(p.fiber_ptr[T.f0 + t] - e0));
    for (int t = tid; t < nf; t += SP_NT) tfj[t] = p.fiber_j[T.f0 + t];
    for (int t = tid; t < ni; t += SP_NT) si[t] = p.si_g[T.si0 + t];
    const int nch = (ni + 63) >> 6;
    for (int e = tid; e < nch * (XD_CHUNK / 16); e += SP_NT) reinterpret_cast<uint4*>(xd)[e] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // 1. scatter (warps 0, 1, 8-15; the producers start gathering U meanwhile):
    //    Xd[fiber][id] = value (K-major SWIZZLE_128B, 64-id chunks)
    if (scatterer) {
      // li_g packs the nonzero's tile fiber (bits 9-14) and local id (bits 0-8)
      auto put = [&](int, uint32_t code, float v) {
        const uint32_t fl = code >> 9, li = code & 511u;
        const uint32_t a = xd_u + (li >> 6) * XD_CHUNK + (fl >> 3) * 1024 + (fl & 7) * 128 +
                           ((((li & 63) >> 3) ^ (fl & 7)) << 4) + (li & 7) * 2;
        if (T.dup) {
          atoms_add16<F16>(a, v);
        } else {
          const uint16_t b = F16 ? __half_as_ushort(__float2half_rn(v)) : __bfloat16_as_ushort(__float2bfloat16_rn(v));
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(b));
        }
      };
      const int64_t a0 = imin64(e0 + nnz, (e0 + 3) & ~int64_t(3));
      const int64_t a1 = max(a0, (e0 + nnz) & ~int64_t(3));
      if (e0 + st < a0) put(st, p.li_g[e0 + st], __ldg(p.val + e0 + st));
      const uint2* vl = reinterpret_cast<const uint2*>(p.li_g + a0);
      const float4* vv = reinterpret_cast<const float4*>(p.val + a0);
      const int nv = static_cast<int>((a1 - a0) >> 2), xa = static_cast<int>(a0 - e0);
      constexpr int U = 8;
      for (int b = 0; b < nv; b += SC_NT * U) {
        uint2 li4[U];
        float4 v4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = b + u * SC_NT + st;
          if (idx < nv) {
            li4[u] = __ldg(vl + idx);
            v4[u] = __ldg(vv + idx);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = b + u * SC_NT + st;
          if (idx < nv) {
            const int x = xa + idx * 4;
            put(x, li4[u].x & 0xFFFF, v4[u].x);
            put(x + 1, li4[u].x >> 16, v4[u].y);
            put(x + 2, li4[u].y & 0xFFFF, v4[u].z);
            put(x + 3, li4[u].y >> 16, v4[u].w);
          }
        }
      }
      if (a1 + st < e0 + nnz) put(static_cast<int>(a1 + st - e0), p.li_g[a1 + st], __ldg(p.val + a1 + st));
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&ms->xd_full);
    }
    // 2-3. row blocks: roles inside the CTA, hand-offs on mbarriers only
    //   warps 2-7   : producers (cp.async gathers of U columns and V rows)
    //   warp 0 lane 0: MMA issuer (mode 1 of rb, then mode 2 of rb - 1)
    //   warps 8-15  : epilogue (D1 -> bf16 A2, D2 diagonal -> Z)
    {
        const int k16_last = (ni - (nch - 1) * 64 + 15) >> 4;
        const int nk2 = (nf + 15) >> 4;
        const int nmg2 = (p.n2 + 63) >> 6;
        if (warp >= 2 && warp < 8) {
          // producers (192 threads): 16-byte cp.async gathers of the U chunks
          // (and, with each row block's first chunk, its V rows) into the
          // MN-major SW128 stages, SP_AHEAD commit groups in flight; each
          // thread arrives on a stage's barrier once its own copies landed
          constexpr int NPT = 192;
          const int pt = tid - 64;
          uint32_t gs = g;
          int pending = 0;  // committed groups whose barriers are not arrived yet
          uint32_t q_slot[SP_AHEAD + 1];
          int q_vs[SP_AHEAD + 1];
          auto retire = [&]() {  // oldest pending group has landed: publish it
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&ms->full[q_slot[0]]);
            if (q_vs[0] >= 0) ptx::mbar_arrive(&ms->vg_full[q_vs[0]]);
#pragma unroll
            for (int e = 0; e < SP_AHEAD; ++e) {
              q_slot[e] = q_slot[e + 1];
              q_vs[e] = q_vs[e + 1];
            }
            --pending;
          };
          for (int rb = 0; rb < p.nrb; ++rb) {
            const uint32_t rs = rbs + rb, vs = rs % SP_NV, vuse = rs / SP_NV;
            for (int c = 0; c < nch; ++c, ++gs) {
              const int slot = static_cast<int>(gs % SP_NS);
              ptx::mbar_wait(&ms->empty[slot], ((gs / SP_NS) & 1) ^ 1);
              uint8_t* udst = ring + slot * UC_BYTES;
              const int kcnt = min(64, ni - c * 64);
              // one task = 64 contiguous bytes (32 rows) of one gathered column
              for (int x = pt; x < kcnt * 4; x += NPT) {
                const int k = x >> 2, q4 = x & 3;
                const __nv_bfloat16* src = p.ut + static_cast<int64_t>(si[c * 64 + k]) * p.ld_ut + rb * 128 + q4 * 32;
                uint8_t* drow = udst + ((k >> 3) * 2 + (q4 >> 1)) * 1024 + (k & 7) * 128;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  ptx::cp_async16(drow + ((((q4 & 1) * 4 + e) ^ (k & 7)) << 4), src + e * 8);
              }
              int vflag_slot = -1;
              if (c == 0) {
                // the MMA may need our unpublished chunks before it frees this V buffer
                if (!ptx::mbar_test(&ms->vg_empty[vs], (vuse & 1) ^ 1)) {
                  ptx::cp_async_wait<0>();
                  while (pending > 0) retire();
                  ptx::mbar_wait(&ms->vg_empty[vs], (vuse & 1) ^ 1);
                }
                uint8_t* vdst = vg + vs * VG_BYTES;
                for (int x = pt; x < nf * 4; x += NPT) {
                  const int fl = x >> 2, q4 = x & 3;
                  const __nv_bfloat16* vrow = p.vtj + static_cast<int64_t>(tfj[fl]) * p.ld_vtj;
                  uint8_t* drow = vdst + ((fl >> 3) * 2 + (q4 >> 1)) * 1024 + (fl & 7) * 128;
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const int qq = q4 * 4 + e;
                    const int64_t col = static_cast<int64_t>(rb) * p.n2 + qq * 8;
                    uint8_t* d = drow + (((qq & 7) ^ (fl & 7)) << 4);
                    if (qq * 8 < p.n2 && col < p.ld_vtj) ptx::cp_async16(d, vrow + col);
                    else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
                  }
                }
                vflag_slot = static_cast<int>(vs);
              }
              ptx::cp_async_commit();
              q_slot[pending] = static_cast<uint32_t>(slot);
              q_vs[pending] = vflag_slot;
              ++pending;
              if (pending == SP_AHEAD) {
                ptx::cp_async_wait<SP_AHEAD - 1>();
                retire();
              }
            }
          }
          ptx::cp_async_wait<0>();
          while (pending > 0) retire();
        } else if (warp == 0 && lane == 0) {
          uint32_t gs = g;
          ptx::mbar_wait(&ms->xd_full, static_cast<uint32_t>(it) & 1);
          auto mode2 = [&](int rb) {
            const uint32_t rs = rbs + rb, vs = rs % SP_NV;
            ptx::mbar_wait(&ms->a2_full, rs & 1);
            ptx::mbar_wait(&ms->vg_full[vs], (rs / SP_NV) & 1);
            ptx::mbar_wait(&ms->d2_empty, (rs & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(a2), b0 = ptx::smem_u32(vg + vs * VG_BYTES);
            for (int kk = 0; kk < nk2; ++kk)
              ptx::mma_bf16(d2, ptx::sw128_desc(a0 + kk * 32), ptx::sw128_mn_desc(b0 + kk * 4096, 1024, 2048),
                            idesc2, kk != 0);
            ptx::mma_commit(&ms->d2_full);
            ptx::mma_commit(&ms->vg_empty[vs]);
          };
          for (int rb = 0; rb < p.nrb; ++rb) {
            const uint32_t rs = rbs + rb, b = rs & 1, use = rs >> 1;
            ptx::mbar_wait(&ms->d1_empty[b], (use & 1) ^ 1);
            ptx::tc_fence_after();
            for (int c = 0; c < nch; ++c, ++gs) {
              const int slot = static_cast<int>(gs % SP_NS);
              ptx::mbar_wait(&ms->full[slot], (gs / SP_NS) & 1);
              ptx::tc_fence_after();
              const uint32_t a0 = ring_u + slot * UC_BYTES, b0 = xd_u + c * XD_CHUNK;
              const int nk = c == nch - 1 ? k16_last : 4;
              for (int kk = 0; kk < nk; ++kk)
                ptx::mma_bf16(d1 + b * 64, ptx::sw128_mn_desc(a0 + kk * 4096, 1024, 2048),
                              ptx::sw128_desc(b0 + kk * 32), idesc1, (c | kk) != 0);
              ptx::mma_commit(&ms->empty[slot]);
            }
            ptx::mma_commit(&ms->d1_full[b]);
            if (rb > 0) mode2(rb - 1);
          }
          mode2(p.nrb - 1);
        } else if (warp >= 8) {
          const int hh = (warp - 8) >> 2;
          for (int rb = 0; rb < p.nrb; ++rb) {
            const uint32_t rs = rbs + rb, b = rs & 1;
            ptx::mbar_wait_sleep(&ms->d1_full[b], (rs >> 1) & 1);
            ptx::tc_fence_after();
            {
              float v[32];
              ptx::tmem_ld32(d1 + b * 64 + lane_addr + hh * 32, v);
              ptx::tmem_wait_ld();
              uint8_t* row = a2 + r * 128;
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                const int q8 = hh * 4 + q4;
                *reinterpret_cast<uint4*>(row + ((q8 ^ (r & 7)) << 4)) = ptx::pack8(v + q4 * 8, F16);
              }
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&ms->a2_full);
            ptx::mbar_arrive(&ms->d1_empty[b]);
            ptx::mbar_wait_sleep(&ms->d2_full, rs & 1);
            ptx::tc_fence_after();
            // diagonal replica block of D2 -> Z (zeroed by the host; fire-and-forget reductions)
            const int64_t prep = static_cast<int64_t>(rb) * rpb + p_local;
            for (int cb = 0; cb < half; cb += 16) {
              float v[16];
              ptx::tmem_ld16(d2 + lane_addr + p_local * p.mpad + hh * half + cb, v);
              ptx::tmem_wait_ld();
              if (prep < p.vp) {
                float* zp = p.z + ((prep * p.n_slices + s) * p.mpad + hh * half + cb) * p.lpad + l;
#pragma unroll
                for (int e = 0; e < 16; ++e) atomicAdd(zp + static_cast<int64_t>(e) * p.lpad, v[e]);
              }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&ms->d2_empty);
          }
        }
        g += static_cast<uint32_t>(p.nrb * nch);
        rbs += static_cast<uint32_t>(p.nrb);
        __syncthreads();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

__global__ void fiber_split_kernel(const uint64_t* __restrict__ fkeys, int64_t nf, int64_t J,
                                   int32_t* __restrict__ fj, int32_t* __restrict__ fk) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nf;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = fkeys[e];
    fj[e] = static_cast<int32_t>(key % static_cast<uint64_t>(J));
    fk[e] = static_cast<int32_t>(key / static_cast<uint64_t>(J));
  }
}

__global__ void payload_unpack_kernel(const uint64_t* __restrict__ pay, int64_t n, int32_t* __restrict__ oi,
                                      float* __restrict__ ov) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t pl = pay[e];
    oi[e] = static_cast<int32_t>(pl >> 32);
    ov[e] = __uint_as_float(static_cast<uint32_t>(pl));
  }
}

// fiber regrouping (COO input): key (k, smallest i), value = fiber index
__global__ void fiber_group_keys_kernel(const int32_t* __restrict__ fk, const int32_t* __restrict__ fmin, int64_t nf,
                                        uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < nf;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[f] = (static_cast<uint64_t>(static_cast<uint32_t>(fk[f])) << 32) | static_cast<uint32_t>(fmin[f]);
    idx[f] = static_cast<int32_t>(f);
  }
}

__global__ void fiber_permute_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ fptr,
                                     const int32_t* __restrict__ fj, int64_t nf, int32_t* __restrict__ cnt,
                                     int32_t* __restrict__ gj) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nf;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t f = perm[q];
    cnt[q] = static_cast<int32_t>(fptr[f + 1] - fptr[f]);
    gj[q] = fj[f];
  }
}

// one warp per (new) fiber: copy its nonzeros to their new place
__global__ void fiber_gather_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ fptr,
                                    const int64_t* __restrict__ gptr, int64_t nf, const int32_t* __restrict__ ni,
                                    const float* __restrict__ nv, int32_t* __restrict__ oi, float* __restrict__ ov) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = w0; q < nf; q += nw) {
    const int32_t f = perm[q];
    const int64_t a = fptr[f], n = fptr[f + 1] - a, d = gptr[q];
    for (int64_t e = lane; e < n; e += 32) {
      oi[d + e] = ni[a + e];
      ov[d + e] = nv[a + e];
    }
  }
}

// ---- COO with compact (rank k, rank j) keys ----------------------------------
// range check, used-k / used-j bitmaps (bits set once: read before the OR, the
// few hot words of a block-structured tensor are not hammered), (k, j) order
__global__ void coo_scan_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                const int32_t* __restrict__ kk, int64_t nnz, int64_t I, int64_t J, int64_t K,
                                uint32_t* __restrict__ usedk, uint32_t* __restrict__ usedj, int* __restrict__ bad) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = ii[e], j = jj[e], k = kk[e];
    if (i < 0 || i >= I || j < 0 || j >= J || k < 0 || k >= K) {
      bad[0] = 1;
      continue;
    }
    const uint32_t bk = 1u << (k & 31), bj = 1u << (j & 31);
    if (!(__ldcg(usedk + (k >> 5)) & bk)) atomicOr(usedk + (k >> 5), bk);
    if (!(__ldcg(usedj + (j >> 5)) & bj)) atomicOr(usedj + (j >> 5), bj);
    if (e + 1 < nnz) {
      const int32_t k2 = kk[e + 1], j2 = jj[e + 1];
      if (k2 < k || (k2 == k && j2 < j)) bad[1] = 1;
    }
  }
}

// Random-order COO: the same checks and bitmaps split by mode so that each
// used-value bitmap (<= 200 KB) sits in one CTA's shared memory — no random
// L2 read per nonzero and mode. coo_check_kernel: range and (k, j) order;
// coo_bits_kernel: one mode's used bits, ORed into the global bitmap once per
// non-zero word per CTA.
__global__ void coo_check_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                 const int32_t* __restrict__ kk, int64_t nnz, int64_t I, int64_t J, int64_t K,
                                 int* __restrict__ bad) {
  bool b0 = false, b1 = false;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = ii[e], j = jj[e], k = kk[e];
    b0 |= i < 0 || i >= I || j < 0 || j >= J || k < 0 || k >= K;
    if (e + 1 < nnz) {
      const int32_t k2 = kk[e + 1], j2 = jj[e + 1];
      b1 |= k2 < k || (k2 == k && j2 < j);
    }
  }
  if (__any_sync(0xffffffffu, b0) && (threadIdx.x & 31) == 0) bad[0] = 1;
  if (__any_sync(0xffffffffu, b1) && (threadIdx.x & 31) == 0) bad[1] = 1;
}

__global__ void __launch_bounds__(1024) coo_bits_kernel(const int32_t* __restrict__ v, int64_t nnz, int64_t n,
                                                        uint32_t* __restrict__ used) {
  extern __shared__ uint32_t sb[];
  const int64_t nw = (n + 31) / 32;
  for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) sb[w] = 0u;
  __syncthreads();
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t x = v[e];
    if (x < 0 || x >= n) continue;  // reported by coo_check_kernel
    const uint32_t bit = 1u << (x & 31);
    if (!(sb[x >> 5] & bit)) atomicOr(&sb[x >> 5], bit);
  }
  __syncthreads();
  for (int64_t w = threadIdx.x; w < nw; w += blockDim.x)
    if (sb[w]) atomicOr(used + w, sb[w]);
}

// rank of every value v < n in the used set (-1 when unused): one 4-byte
// lookup per nonzero instead of a bitmap word + a base
__global__ void rank_table_kernel(const uint32_t* __restrict__ bits, const int64_t* __restrict__ base, int64_t n,
                                  int32_t* __restrict__ rank) {
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t w = bits[x >> 5], bit = 1u << (x & 31);
    rank[x] = (w & bit) ? static_cast<int32_t>(base[x >> 5] + __popc(w & (bit - 1u))) : -1;
  }
}

__global__ void coo_tkey_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                const int32_t* __restrict__ kk, const float* __restrict__ vv, int64_t nnz,
                                const int32_t* __restrict__ rk, const int32_t* __restrict__ rj, uint32_t nju,
                                uint32_t* __restrict__ key, uint64_t* __restrict__ pay) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[e] = static_cast<uint32_t>(rk[kk[e]]) * nju + static_cast<uint32_t>(rj[jj[e]]);
    pay[e] = (static_cast<uint64_t>(static_cast<uint32_t>(ii[e])) << 32) | __float_as_uint(vv[e]);
  }
}

__global__ void popc_kernel(const uint32_t* __restrict__ bits, int64_t nw, int32_t* __restrict__ cnt) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < nw;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cnt[w] = __popc(bits[w]);
}

// rank -> value (the used k or j values in increasing order)
__global__ void rank_inverse_kernel(const uint32_t* __restrict__ bits, const int64_t* __restrict__ base, int64_t nw,
                                    int32_t* __restrict__ inv) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < nw;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t b = bits[w];
    int64_t r = base[w];
    while (b) {
      inv[r++] = static_cast<int32_t>(w * 32 + __ffs(b) - 1);
      b &= b - 1;
    }
  }
}

__device__ __forceinline__ uint32_t bit_rank(const uint32_t* bits, const int64_t* base, int32_t v) {
  return static_cast<uint32_t>(base[v >> 5]) + __popc(bits[v >> 5] & ((1u << (v & 31)) - 1u));
}

// compact key rank(k) * nju + rank(j), payload (i << 32) | value bits
__global__ void coo_ckey_kernel(const int32_t* __restrict__ ii, const int32_t* __restrict__ jj,
                                const int32_t* __restrict__ kk, const float* __restrict__ vv, int64_t nnz,
                                const uint32_t* __restrict__ usedk, const int64_t* __restrict__ basek,
                                const uint32_t* __restrict__ usedj, const int64_t* __restrict__ basej, uint32_t nju,
                                uint32_t* __restrict__ key, uint64_t* __restrict__ pay) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[e] = bit_rank(usedk, basek, kk[e]) * nju + bit_rank(usedj, basej, jj[e]);
    pay[e] = (static_cast<uint64_t>(static_cast<uint32_t>(ii[e])) << 32) | __float_as_uint(vv[e]);
  }
}

__global__ void fiber_decode32_kernel(const uint32_t* __restrict__ fkeys, int64_t nf, uint32_t nju,
                                      const int32_t* __restrict__ invk, const int32_t* __restrict__ invj,
                                      int32_t* __restrict__ fj, int32_t* __restrict__ fk) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nf;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t key = fkeys[e];
    fj[e] = invj[key % nju];
    fk[e] = invk[key / nju];
  }
}

int gridn(int64_t work) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 16))); }

// exclusive scan of cnt[0..n) into ptr[0..n] (ptr[n] = total)
template <class T>
void scan_ptr(const T* cnt, int64_t n, int64_t* ptr, cudaStream_t s) {
  XCUDA(cudaMemsetAsync(ptr, 0, sizeof(int64_t), s));
  if (n == 0) return;
  size_t tb = 0;
  XCUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, ptr + 1, n, s));
  DevBuf<uint8_t> tmp(tb, s);
  XCUDA(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, cnt, ptr + 1, n, s));
  count_launch();
}

}  // namespace

// COO -> (validated, sorted) compact keys -> tile path. Returns false (having
// done nothing but the validation) when rank(k) x rank(j) does not fit 32 bits.
bool Plan::sparse_tc_coo32(const int32_t* i, const int32_t* j, const int32_t* k, const float* val, int64_t nnz,
                           float* ydev, bool accumulate, cudaStream_t s) {
  const int64_t I = desc.dims[0], J = desc.dims[1], K = desc.dims[2];
  PhaseTrace tr("sparse_tc_coo32", s);
  const int64_t nwk = ceil_div(K, 32), nwj = ceil_div(J, 32);
  DevBuf<uint32_t> usedk(static_cast<size_t>(nwk), s), usedj(static_cast<size_t>(nwj), s);
  usedk.zero();
  usedj.zero();
  DevBuf<int> flags(2, s);
  flags.zero();
  // per-mode shared-memory bitmaps when both fit a CTA (C4: 10^6 values, 122 KB)
  const size_t bmk = static_cast<size_t>(nwk) * 4, bmj = static_cast<size_t>(nwj) * 4;
  const bool smem_bits = bmk <= 200 * 1024 && bmj <= 200 * 1024;
  if (smem_bits) {
    coo_check_kernel<<<gridn(nnz), 256, 0, s>>>(i, j, k, nnz, I, J, K, flags.ptr);
    XLAUNCH_CHECK();
    XCUDA(cudaFuncSetAttribute(coo_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    coo_bits_kernel<<<sm_count(), 1024, bmk, s>>>(k, nnz, K, usedk.ptr);
    XLAUNCH_CHECK();
    coo_bits_kernel<<<sm_count(), 1024, bmj, s>>>(j, nnz, J, usedj.ptr);
    XLAUNCH_CHECK();
  } else {
    coo_scan_kernel<<<gridn(nnz), 256, 0, s>>>(i, j, k, nnz, I, J, K, usedk.ptr, usedj.ptr, flags.ptr);
    XLAUNCH_CHECK();
  }
  DevBuf<int32_t> ck(static_cast<size_t>(nwk), s), cj(static_cast<size_t>(nwj), s);
  DevBuf<int64_t> basek(static_cast<size_t>(nwk + 1), s), basej(static_cast<size_t>(nwj + 1), s);
  popc_kernel<<<gridn(nwk), 256, 0, s>>>(usedk.ptr, nwk, ck.ptr);
  XLAUNCH_CHECK();
  popc_kernel<<<gridn(nwj), 256, 0, s>>>(usedj.ptr, nwj, cj.ptr);
  XLAUNCH_CHECK();
  scan_ptr(ck.ptr, nwk, basek.ptr, s);
  scan_ptr(cj.ptr, nwj, basej.ptr, s);
  int hf[2] = {0, 0};
  int64_t nku = 0, nju = 0;
  XCUDA(cudaMemcpyAsync(hf, flags.ptr, sizeof(hf), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaMemcpyAsync(&nku, basek.ptr + nwk, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaMemcpyAsync(&nju, basej.ptr + nwj, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  tr.mark("scan");
  if (hf[0]) data_error("plan_compress_coo: coordinate outside the tensor");
  if (nku * nju >= (int64_t(1) << 32)) return false;
  DevBuf<int32_t> invk(static_cast<size_t>(nku), s), invj(static_cast<size_t>(nju), s);
  rank_inverse_kernel<<<gridn(nwk), 256, 0, s>>>(usedk.ptr, basek.ptr, nwk, invk.ptr);
  XLAUNCH_CHECK();
  rank_inverse_kernel<<<gridn(nwj), 256, 0, s>>>(usedj.ptr, basej.ptr, nwj, invj.ptr);
  XLAUNCH_CHECK();
  DevBuf<uint32_t> keys(static_cast<size_t>(nnz), s);
  DevBuf<uint64_t> pay(static_cast<size_t>(nnz), s);
  if (K + J <= (int64_t(1) << 27)) {
    // rank tables (4 bytes per index value, L2-resident at C4's 2 x 10^6)
    DevBuf<int32_t> rk(static_cast<size_t>(K), s), rj(static_cast<size_t>(J), s);
    rank_table_kernel<<<gridn(K), 256, 0, s>>>(usedk.ptr, basek.ptr, K, rk.ptr);
    XLAUNCH_CHECK();
    rank_table_kernel<<<gridn(J), 256, 0, s>>>(usedj.ptr, basej.ptr, J, rj.ptr);
    XLAUNCH_CHECK();
    coo_tkey_kernel<<<gridn(nnz), 256, 0, s>>>(i, j, k, val, nnz, rk.ptr, rj.ptr, static_cast<uint32_t>(nju),
                                               keys.ptr, pay.ptr);
    XLAUNCH_CHECK();
  } else {
    coo_ckey_kernel<<<gridn(nnz), 256, 0, s>>>(i, j, k, val, nnz, usedk.ptr, basek.ptr, usedj.ptr, basej.ptr,
                                               static_cast<uint32_t>(nju), keys.ptr, pay.ptr);
    XLAUNCH_CHECK();
  }
  tr.mark("keys");
  if (hf[1]) {
    DevBuf<uint32_t> keys2(static_cast<size_t>(nnz), s);
    DevBuf<uint64_t> pay2(static_cast<size_t>(nnz), s);
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t(1) << end_bit) < static_cast<uint64_t>(nku * nju)) ++end_bit;
    cub::DoubleBuffer<uint32_t> dk(keys.ptr, keys2.ptr);
    cub::DoubleBuffer<uint64_t> dp(pay.ptr, pay2.ptr);
    size_t tb = 0;
    XCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dp, nnz, 0, end_bit, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, dk, dp, nnz, 0, end_bit, s));
    count_launch();
    if (dk.Current() != keys.ptr) std::swap(keys, keys2);
    if (dp.Current() != pay.ptr) std::swap(pay, pay2);
    tr.mark("sort");
  }
  sparse_tc_sorted32(keys, pay, invk.ptr, invj.ptr, nju, nnz, ydev, accumulate, s);
  return true;
}

bool Plan::sparse_tc_ok() const {
  // XTSG_SPARSE_TC=0 selects the SIMT fiber kernel (read per call: tests A/B both)
  const char* e = std::getenv("XTSG_SPARSE_TC");
  return (!e || std::atoi(e) != 0) && tensor_core() && !comp() && mpad <= lpad && lpad <= 128;
}

// CSF (slices -> fibers -> nonzeros, already validated, on the device) -> Z
// through the tensor-core tile kernel, then mode 3 over the slices.
void Plan::sparse_tc(int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr, int64_t n_fibers,
                     const int64_t* fiber_ptr, const int32_t* fiber_j, int64_t nnz, const int32_t* nz_i,
                     const float* val, float* ydev, bool accumulate, cudaStream_t s) {
  const int64_t plrows = vP * lpad;
  PhaseTrace tr("sparse_tc", s);
  DevBuf<float> z(static_cast<size_t>(vP * n_slices * mpad * lpad), s);
  z.zero();  // the tensor kernel adds every tile's contribution (empty slices stay zero)
  // 1. plan the tiles (every tile holds >= 1 nonzero and is either whole
  //    fibers or a piece of <= 512 nonzeros of one fiber)
  const int64_t max_tiles = n_fibers + nnz / SP_NI + 1;
  DevBuf<int32_t> si_g(static_cast<size_t>(nnz), s);
  DevBuf<uint16_t> li_g(static_cast<size_t>(nnz) + 8, s);
  DevBuf<SpTile> tiles(static_cast<size_t>(max_tiles), s);
  DevBuf<unsigned long long> ctr(3, s);
  ctr.zero();
  SpPlanParams pp{};
  pp.slice_ptr = slice_ptr;
  pp.fiber_ptr = fiber_ptr;
  pp.nz_i = nz_i;
  pp.n_slices = n_slices;
  pp.si_g = si_g.ptr;
  pp.li_g = li_g.ptr;
  pp.tiles = tiles.ptr;
  pp.max_tiles = max_tiles;
  pp.counters = ctr.ptr;
  {
    int per_sm = 1;
    XCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sparse_plan_kernel, PL_NT, 0));
    const int grid = static_cast<int>(std::min<int64_t>(n_slices, static_cast<int64_t>(sm_count()) * std::max(1, per_sm)));
    tr.mark("alloc");
    sparse_plan_kernel<<<grid, PL_NT, 0, s>>>(pp);
    XLAUNCH_CHECK();
    tr.mark("plan");
  }
  // 2. tensor-core tiles
  SpTcParams prm{};
  prm.fiber_ptr = fiber_ptr;
  prm.fiber_j = fiber_j;
  prm.val = val;
  prm.si_g = si_g.ptr;
  prm.li_g = li_g.ptr;
  prm.tiles = tiles.ptr;
  prm.n_tiles = ctr.ptr + 1;
  prm.max_tiles = max_tiles;
  prm.counter = ctr.ptr + 2;
  prm.n_slices = n_slices;
  prm.ut = ut.ptr;
  prm.ld_ut = (plrows + 255) / 256 * 256;
  prm.vtj = vtj.ptr;
  prm.ld_vtj = vP * mpad;
  prm.lpad = static_cast<int>(lpad);
  prm.mpad = static_cast<int>(mpad);
  prm.nrb = static_cast<int>(ceil_div(plrows, 128));
  prm.n2 = static_cast<int>((128 / lpad) * mpad);
  prm.vp = vP;
  prm.z = z.ptr;
  auto launch = [&](auto kern) {
    XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SP_SMEM));
    kern<<<sm_count(), SP_NT, SP_SMEM, s>>>(prm);
  };
  if (fp16()) launch(sparse_tc_kernel<true>);
  else launch(sparse_tc_kernel<false>);
  XLAUNCH_CHECK();
  tr.mark("tiles");
  sparse_mode3(z.ptr, slice_k, n_slices, ydev, accumulate, s);
  tr.mark("mode3");
}

// sorted COO (keys = k*J + j ascending, payload = (i << 32) | value bits) ->
// CSF arrays -> sparse_tc
void Plan::sparse_tc_sorted(DevBuf<uint64_t>& skeys_buf, DevBuf<uint64_t>* spay_buf, const int32_t* si_in,
                            const float* sv_in, int64_t nnz, float* ydev, bool accumulate, cudaStream_t s) {
  const uint64_t* skeys = skeys_buf.ptr;
  PhaseTrace tr("sparse_tc_sorted", s);
  const int64_t J = desc.dims[1];
  // fibers: runs of equal (k, j)
  DevBuf<uint64_t> fkeys(static_cast<size_t>(nnz), s);
  DevBuf<int32_t> fcnt(static_cast<size_t>(nnz), s);
  DevBuf<int64_t> nruns(2, s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, skeys, fkeys.ptr, fcnt.ptr, nruns.ptr, nnz, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, skeys, fkeys.ptr, fcnt.ptr, nruns.ptr, nnz, s));
    count_launch();
  }
  skeys_buf.release();
  DevBuf<int32_t> bi;
  DevBuf<float> bv;
  const int32_t* ni = si_in;
  const float* nv = sv_in;
  if (spay_buf) {
    bi = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bv = DevBuf<float>(static_cast<size_t>(nnz), s);
    payload_unpack_kernel<<<gridn(nnz), 256, 0, s>>>(spay_buf->ptr, nnz, bi.ptr, bv.ptr);
    XLAUNCH_CHECK();
    spay_buf->release();
    ni = bi.ptr;
    nv = bv.ptr;
  }
  int64_t nf = 0;
  XCUDA(cudaMemcpyAsync(&nf, nruns.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  tr.mark("fiber_rle+unpack");
  if (nf >= (int64_t(1) << 31)) usage("plan_compress_coo: at most 2^31-1 distinct (j, k) fibers per call");
  DevBuf<int64_t> fptr(static_cast<size_t>(nf + 1), s);
  scan_ptr(fcnt.ptr, nf, fptr.ptr, s);
  fcnt.release();
  DevBuf<int32_t> fj(static_cast<size_t>(nf), s), fk(static_cast<size_t>(nf), s);
  fiber_split_kernel<<<gridn(nf), 256, 0, s>>>(fkeys.ptr, nf, J, fj.ptr, fk.ptr);
  XLAUNCH_CHECK();
  fkeys.release();
  sparse_tc_tail(nf, fptr, fj, fk, ni, nv, bi, bv, nnz, ydev, accumulate, s);

}


// sorted compact keys + (i, value) payload -> CSF fibers -> the shared tail
void Plan::sparse_tc_sorted32(DevBuf<uint32_t>& skeys, DevBuf<uint64_t>& spay, const int32_t* invk,
                              const int32_t* invj, int64_t nju, int64_t nnz, float* ydev, bool accumulate,
                              cudaStream_t s) {
  PhaseTrace tr("sparse_tc_sorted32", s);
  DevBuf<uint32_t> fkeys(static_cast<size_t>(nnz), s);
  DevBuf<int32_t> fcnt(static_cast<size_t>(nnz), s);
  DevBuf<int64_t> nruns(1, s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, skeys.ptr, fkeys.ptr, fcnt.ptr, nruns.ptr, nnz, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, skeys.ptr, fkeys.ptr, fcnt.ptr, nruns.ptr, nnz, s));
    count_launch();
  }
  skeys.release();
  DevBuf<int32_t> bi(static_cast<size_t>(nnz), s);
  DevBuf<float> bv(static_cast<size_t>(nnz), s);
  payload_unpack_kernel<<<gridn(nnz), 256, 0, s>>>(spay.ptr, nnz, bi.ptr, bv.ptr);
  XLAUNCH_CHECK();
  spay.release();
  int64_t nf = 0;
  XCUDA(cudaMemcpyAsync(&nf, nruns.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  tr.mark("fiber_rle+unpack");
  if (nf >= (int64_t(1) << 31)) usage("plan_compress_coo: at most 2^31-1 distinct (j, k) fibers per call");
  DevBuf<int64_t> fptr(static_cast<size_t>(nf + 1), s);
  scan_ptr(fcnt.ptr, nf, fptr.ptr, s);
  fcnt.release();
  DevBuf<int32_t> fj(static_cast<size_t>(nf), s), fk(static_cast<size_t>(nf), s);
  fiber_decode32_kernel<<<gridn(nf), 256, 0, s>>>(fkeys.ptr, nf, static_cast<uint32_t>(nju), invk, invj, fj.ptr,
                                                  fk.ptr);
  XLAUNCH_CHECK();
  fkeys.release();
  sparse_tc_tail(nf, fptr, fj, fk, bi.ptr, bv.ptr, bi, bv, nnz, ydev, accumulate, s);
}

// fibers (nf, fptr, fj, fk in (k, j) order) + nonzero i / values -> slices,
// regrouping by smallest i, the tile path. bi / bv own the nonzero arrays when
// the caller unpacked them (released once regrouped).
void Plan::sparse_tc_tail(int64_t nf, DevBuf<int64_t>& fptr, DevBuf<int32_t>& fj, DevBuf<int32_t>& fk,
                          const int32_t* ni, const float* nv, DevBuf<int32_t>& bi, DevBuf<float>& bv, int64_t nnz,
                          float* ydev, bool accumulate, cudaStream_t s) {
  PhaseTrace tr("sparse_tc_tail", s);
  DevBuf<int64_t> nruns(2, s);
  // slices: runs of equal k over the fibers
  DevBuf<int32_t> uk(static_cast<size_t>(nf), s), scnt(static_cast<size_t>(nf), s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, fk.ptr, uk.ptr, scnt.ptr, nruns.ptr, nf, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, fk.ptr, uk.ptr, scnt.ptr, nruns.ptr, nf, s));
    count_launch();
  }
  int64_t kd = 0;
  XCUDA(cudaMemcpyAsync(&kd, nruns.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  tr.mark("slices");
  DevBuf<int64_t> sptr(static_cast<size_t>(kd + 1), s);
  scan_ptr(scnt.ptr, kd, sptr.ptr, s);
  scnt.release();
  // Regroup the fibers of every slice by their smallest i (stable in j): the
  // (k, j) order interleaves fibers of different rank-1 blocks that share a
  // slice, which the planner would cut into one-fiber tiles; fibers with a
  // common i support become neighbours. Slices keep their order and extents.
  const char* rg_env = std::getenv("XTSG_COO_REGROUP");
  if (rg_env && std::atoi(rg_env) == 0) {  // A/B knob: keep the (k, j) fiber order
    fk.release();
    sparse_tc(kd, uk.ptr, sptr.ptr, nf, fptr.ptr, fj.ptr, nnz, ni, nv, ydev, accumulate, s);
    return;
  }
  DevBuf<int32_t> fmin(static_cast<size_t>(nf), s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceSegmentedReduce::Min(nullptr, tb, ni, fmin.ptr, nf, fptr.ptr, fptr.ptr + 1, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceSegmentedReduce::Min(tmp.ptr, tb, ni, fmin.ptr, nf, fptr.ptr, fptr.ptr + 1, s));
    count_launch();
  }
  DevBuf<uint64_t> gk(static_cast<size_t>(nf), s), gk2(static_cast<size_t>(nf), s);
  DevBuf<int32_t> gi(static_cast<size_t>(nf), s), gi2(static_cast<size_t>(nf), s);
  fiber_group_keys_kernel<<<gridn(nf), 256, 0, s>>>(fk.ptr, fmin.ptr, nf, gk.ptr, gi.ptr);
  XLAUNCH_CHECK();
  fk.release();
  fmin.release();
  {
    int end_bit = 33;
    while (end_bit < 64 && (uint64_t(1) << (end_bit - 32)) < static_cast<uint64_t>(desc.dims[2])) ++end_bit;
    size_t tb = 0;
    XCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, gk.ptr, gk2.ptr, gi.ptr, gi2.ptr, nf, 0, end_bit, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, gk.ptr, gk2.ptr, gi.ptr, gi2.ptr, nf, 0, end_bit, s));
    count_launch();
  }
  gk.release();
  gk2.release();
  gi.release();
  DevBuf<int32_t> gcnt(static_cast<size_t>(nf), s), gj(static_cast<size_t>(nf), s);
  fiber_permute_kernel<<<gridn(nf), 256, 0, s>>>(gi2.ptr, fptr.ptr, fj.ptr, nf, gcnt.ptr, gj.ptr);
  XLAUNCH_CHECK();
  DevBuf<int64_t> gptr(static_cast<size_t>(nf + 1), s);
  scan_ptr(gcnt.ptr, nf, gptr.ptr, s);
  gcnt.release();
  DevBuf<int32_t> gni(static_cast<size_t>(nnz), s);
  DevBuf<float> gnv(static_cast<size_t>(nnz), s);
  fiber_gather_kernel<<<gridn(nf * 32), 256, 0, s>>>(gi2.ptr, fptr.ptr, gptr.ptr, nf, ni, nv, gni.ptr, gnv.ptr);
  XLAUNCH_CHECK();
  gi2.release();
  fptr.release();
  fj.release();
  bi.release();
  bv.release();
  tr.mark("regroup");
  sparse_tc(kd, uk.ptr, sptr.ptr, nf, gptr.ptr, gj.ptr, nnz, gni.ptr, gnv.ptr, ydev, accumulate, s);
  // COO calls return with their multi-GB temporaries back in the pool: a
  // caller that enqueues the next call at once otherwise makes the pool map
  // new memory while these are still pending (C4 COO steps of 71 ms became
  // 185-450 ms back to back)
  XCUDA(cudaStreamSynchronize(s));
}

}  // namespace xtsg
