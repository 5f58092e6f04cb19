// K7 (tensor-core form) — sparse compression as dense tiles of a mode-3 slice.
//
// Eq. 3 restricted to the nonzeros (no reference counterpart):
//   Z_k = sum_{(i,j) in slice k} x_ijk * U[:, i] (x) V_p[:, j]   (per replica)
// then mode 3 over the slices exactly like the dense path.
//
// The SIMT fiber kernel (coo.cu) gathers a 1 KB stacked U column per nonzero
// and spends P*L FMAs on it; nothing is reused across the fibers of a slice.
// Here one CTA owns a slice k (dynamic slice counter, one CTA per SM) and
// walks it in tiles of up to 64 fibers whose nonzeros touch at most 512
// distinct i:
//   1. densify: the tile's i are hashed in shared memory (2048 slots, open
//      addressing) to local ids 0..ni-1 (Si = the distinct i), and the
//      nonzeros are scattered as bf16/fp16 into a dense tile
//      Xd[fiber][local i] (UMMA B operand, K-major SWIZZLE_128B; duplicate
//      coordinates sum through shared-memory atomics);
//   2. mode 1 per 128-row block rb of the stacked U (tcgen05, M = 128,
//      N = 64 fibers, K = ni): D1 = U[rb rows, Si] * Xd^T, the U columns
//      gathered from the i-major copy Ut[i][(p, l)] with 16-byte cp.async
//      straight into the MN-major SWIZZLE_128B layout (a 4-slot ring, issued
//      three chunks ahead of the MMA);
//   3. mode 2 (tcgen05, M = 128, N = (128/Lpad)*Mpad, K = fibers): D1 drained
//      to bf16 in shared memory (K-major) times V[(p, m), j_f] gathered from
//      the j-major copy Vtj (MN-major); the diagonal replica blocks of D2 are
//      added into Z[p][slice][m][l] (the slice's Z stays in L2 across tiles).
// A tile whose i support exceeds 512 is retried with half the fibers; a
// single fiber is cut into 512-nonzero pieces. Per nonzero the kernel reads
// 8 B (i, value) from HBM once and the U gather is amortised over the tile's
// fibers (C4: 464 fibers share each U column, ~16 B of L2->SM per nonzero
// instead of 1 KB). Work per tile: 2*PL*64*ni (mode 1) + 2*PL*64*N2 (mode 2)
// tensor flops.
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

constexpr int SP_NT = 512;  // 16 warps: the densify passes are latency-bound
constexpr int SP_SPT = 2048 / SP_NT;  // hash slots per thread in the id compaction
constexpr int SP_NF = 64;    // fibers per tile (mode-1 UMMA N, mode-2 K)
constexpr int SP_NI = 512;   // distinct i per tile (mode-1 K)
constexpr int SP_HS = 2048;  // hash slots (load <= 0.25 + in-flight claims)
constexpr int SP_NS = 4;     // U gather ring slots
constexpr int SP_AHEAD = 3;  // chunks issued ahead of the MMA
constexpr int XD_CHUNK = SP_NF * 128;              // 64 fibers x 64 i, 8 KB
constexpr int XD_BYTES = (SP_NI / 64) * XD_CHUNK;  // 64 KB
constexpr int UC_BYTES = 128 * 64 * 2;             // 128 rows x 64 i, 16 KB
constexpr int A2_BYTES = 128 * 128;                // 128 rows x 64 fibers
constexpr int VG_BYTES = 128 * 64 * 2;             // 128 (p, m) x 64 fibers

struct SpMisc {
  uint64_t mma_done[SP_NS];
  uint64_t d1_full, d2_full;
  uint32_t tmem_base;
  int count, ovf;
  int64_t slice;
  int wsum[SP_NT / 32];
};

constexpr int OFF_RING = XD_BYTES;
constexpr int OFF_A2 = OFF_RING + SP_NS * UC_BYTES;
constexpr int OFF_VG = OFF_A2 + A2_BYTES;
constexpr int OFF_KEYS = OFF_VG + VG_BYTES;
constexpr int OFF_LIS = OFF_KEYS + SP_HS * 4;
constexpr int OFF_SI = OFF_LIS + SP_HS * 2;
constexpr int OFF_TFP = OFF_SI + SP_NI * 4;
constexpr int OFF_TFJ = OFF_TFP + (SP_NF + 2) * 8;
constexpr int OFF_MISC = OFF_TFJ + SP_NF * 4;
constexpr int SP_SMEM = OFF_MISC + static_cast<int>(sizeof(SpMisc)) + 1024;
static_assert(SP_SMEM <= 232448, "shared memory budget");

struct SpTcParams {
  const int64_t* slice_ptr;  // n_slices + 1 fiber offsets
  const int64_t* fiber_ptr;  // nonzero offsets per fiber
  const int32_t* fiber_j;
  const int32_t* nz_i;
  const float* val;
  int64_t n_slices;
  const __nv_bfloat16* ut;  // [I][ld_ut], row (p, l) contiguous
  int64_t ld_ut;
  const __nv_bfloat16* vtj;  // [J][ld_vtj], (p, m) contiguous
  int64_t ld_vtj;
  int lpad, mpad, nrb, n2;
  int64_t vp;
  float* z;  // [vp][n_slices][mpad][lpad]
  unsigned long long* counter;
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
// x += v on a 16-bit float in shared memory (bf16 or fp16): CAS on its 32-bit word
template <bool F16>
__device__ __forceinline__ void atoms_add16(uint8_t* dst, float v) {
  const uint32_t a = ptx::smem_u32(dst);
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

__device__ __forceinline__ uint32_t sp_hash(int32_t key) {
  return (static_cast<uint32_t>(key) * 2654435761u) >> (32 - 11);
}

// f(x, i) over the tile's nonzeros, x = e - e0 the local offset (< 2^30):
// head scalars, 16-byte vector body (U loads in flight per thread), tail
// scalars, so each thread sees increasing x. f returns false to stop early.
template <int U, class F>
__device__ __forceinline__ void for_each_i(const int32_t* __restrict__ nz_i, int64_t e0, int64_t e1,
                                           volatile int* stop, F&& f) {
  const int tid = threadIdx.x;
  const int64_t a0 = min(e1, (e0 + 3) & ~int64_t(3));
  const int64_t a1 = max(a0, e1 & ~int64_t(3));
  for (int64_t e = e0 + tid; e < a0; e += SP_NT) f(static_cast<int>(e - e0), __ldg(nz_i + e));
  const int4* v = reinterpret_cast<const int4*>(nz_i + a0);
  const int nv = static_cast<int>((a1 - a0) >> 2), xa = static_cast<int>(a0 - e0);
  for (int b = 0; b < nv; b += SP_NT * U) {
    if (*stop) return;
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = b + u * SP_NT + tid;
      if (idx < nv) x[u] = __ldg(v + idx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = b + u * SP_NT + tid;
      if (idx < nv) {
        const int xl = xa + idx * 4;
        f(xl, x[u].x);
        f(xl + 1, x[u].y);
        f(xl + 2, x[u].z);
        f(xl + 3, x[u].w);
      }
    }
  }
  for (int64_t e = a1 + tid; e < e1; e += SP_NT) f(static_cast<int>(e - e0), __ldg(nz_i + e));
}

// f(x, i, value) over the tile's nonzeros, same order as for_each_i
template <int U, class F>
__device__ __forceinline__ void for_each_ix(const int32_t* __restrict__ nz_i, const float* __restrict__ val,
                                            int64_t e0, int64_t e1, volatile int* stop, F&& f) {
  const int tid = threadIdx.x;
  const int64_t a0 = min(e1, (e0 + 3) & ~int64_t(3));
  const int64_t a1 = max(a0, e1 & ~int64_t(3));
  for (int64_t e = e0 + tid; e < a0; e += SP_NT) f(static_cast<int>(e - e0), __ldg(nz_i + e), __ldg(val + e));
  const int4* vi = reinterpret_cast<const int4*>(nz_i + a0);
  const float4* vv = reinterpret_cast<const float4*>(val + a0);
  const int nv = static_cast<int>((a1 - a0) >> 2), xa = static_cast<int>(a0 - e0);
  for (int b = 0; b < nv; b += SP_NT * U) {
    if (*stop) return;
    int4 x[U];
    float4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = b + u * SP_NT + tid;
      if (idx < nv) {
        x[u] = __ldg(vi + idx);
        w[u] = __ldg(vv + idx);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = b + u * SP_NT + tid;
      if (idx < nv) {
        const int xl = xa + idx * 4;
        f(xl, x[u].x, w[u].x);
        f(xl + 1, x[u].y, w[u].y);
        f(xl + 2, x[u].z, w[u].z);
        f(xl + 3, x[u].w, w[u].w);
      }
    }
  }
  for (int64_t e = a1 + tid; e < e1; e += SP_NT)
    f(static_cast<int>(e - e0), __ldg(nz_i + e), __ldg(val + e));
}

template <bool F16>
__global__ void __launch_bounds__(SP_NT, 1) sparse_tc_kernel(const SpTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xd = sm;
  uint8_t* ring = sm + OFF_RING;
  uint8_t* a2 = sm + OFF_A2;
  uint8_t* vg = sm + OFF_VG;
  int32_t* keys = reinterpret_cast<int32_t*>(sm + OFF_KEYS);
  uint16_t* lis = reinterpret_cast<uint16_t*>(sm + OFF_LIS);
  int32_t* si = reinterpret_cast<int32_t*>(sm + OFF_SI);
  int32_t* tfp = reinterpret_cast<int32_t*>(sm + OFF_TFP);  // fiber starts, local offsets
  int32_t* tfj = reinterpret_cast<int32_t*>(sm + OFF_TFJ);
  SpMisc* ms = reinterpret_cast<SpMisc*>(sm + OFF_MISC);
  volatile int* vflag = &ms->ovf;  // overflow (insert) or miss (lookup) of the current pass
  volatile int* vcount = &ms->count;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < SP_NS; ++s) ptx::mbar_init(&ms->mma_done[s], 1);
    ptx::mbar_init(&ms->d1_full, 1);
    ptx::mbar_init(&ms->d2_full, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(&ms->tmem_base, 256);
  // stale operand bytes beyond a partial chunk must be finite (they multiply zeros)
  for (int e = tid; e < (SP_NS * UC_BYTES + A2_BYTES + VG_BYTES) / 16; e += SP_NT)
    reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = ms->tmem_base;
  const uint32_t d1 = tmem, d2 = tmem + 128;
  const uint32_t idesc1 = (ptx::idesc_bf16(128, SP_NF) | ptx::IDESC_A_MN) & ptx::idesc_fmt_mask(F16);
  const uint32_t idesc2 = (ptx::idesc_bf16(128, p.n2) | ptx::IDESC_B_MN) & ptx::idesc_fmt_mask(F16);
  const int q = warp & 3, hh = warp >> 2;
  const int r = q * 32 + lane;  // row of the 128-row block == TMEM lane
  const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
  const int p_local = r / p.lpad, l = r % p.lpad;
  const int rpb = 128 / p.lpad;
  const int half = p.mpad >> 1;
  const uint32_t ring_u = ptx::smem_u32(ring), xd_u = ptx::smem_u32(xd);
  uint32_t g = 0, n1 = 0, n2c = 0;  // U chunk sequence number, D1 / D2 commit counts

  // the i -> local id table persists across the tiles of a slice (their i
  // supports usually coincide); lis = 0xFFFF marks a key without an id yet
  auto clear_table = [&]() {
    for (int t = tid; t < SP_HS; t += SP_NT) {
      keys[t] = -1;
      lis[t] = 0xFFFF;
    }
    if (tid == 0) ms->count = 0;
  };
  clear_table();
  __syncthreads();

  for (;;) {
    if (tid == 0) ms->slice = static_cast<int64_t>(atomicAdd(p.counter, 1ull));
    __syncthreads();
    const int64_t s = ms->slice;
    __syncthreads();
    if (s >= p.n_slices) break;
    const int64_t fs0 = p.slice_ptr[s], fs1 = p.slice_ptr[s + 1];
    const int64_t es0 = fs1 > fs0 ? p.fiber_ptr[fs0] : 0, es1 = fs1 > fs0 ? p.fiber_ptr[fs1] : 0;
    if (es1 <= es0) continue;  // no nonzeros: Z of the slice stays zero
    if (*vcount) {
      clear_table();
      __syncthreads();
    }
    int64_t f = fs0, e_in = es0;
    int nt = SP_NF;
    while (f < fs1) {
      int nf = static_cast<int>(imin64(nt, fs1 - f));
      const int64_t fend0 = p.fiber_ptr[f + 1];
      if (nt > 1 && p.fiber_ptr[f + nf] - e_in > (int64_t(1) << 30)) nt = nf = 1;  // local offsets stay 32-bit
      const int64_t e_end = nt == 1 ? imin64(fend0, e_in + SP_NI) : p.fiber_ptr[f + nf];
      for (int t = tid; t <= nf; t += SP_NT)
        tfp[t] = t == 0 ? 0 : static_cast<int32_t>((t == nf ? e_end : p.fiber_ptr[f + t]) - e_in);
      for (int t = tid; t < nf; t += SP_NT) tfj[t] = p.fiber_j[f + t];
      for (int e = tid; e < XD_BYTES / 16; e += SP_NT) reinterpret_cast<uint4*>(xd)[e] = make_uint4(0, 0, 0, 0);
      if (tid == 0) {
        ms->ovf = 0;
        // the next tile's nonzeros (about as many as this one) into L2
        const int64_t n = e_end - e_in;
        const int64_t pa = (e_end + 3) & ~int64_t(3), pb = imin64(es1, e_end + n) & ~int64_t(3);
        if (pb > pa) {
          const uint32_t bytes = static_cast<uint32_t>(imin64((pb - pa) * 4, 1 << 20));
          ptx::bulk_prefetch_l2(p.nz_i + pa, bytes);
          ptx::bulk_prefetch_l2(p.val + pa, bytes);
        }
      }
      __syncthreads();
      // scatter pass: look each i up, add the value into Xd[fiber][id]; a key
      // without an id raises the flag (and the pass stops early)
      auto scatter = [&]() {
        int fl = 0;  // fiber cursor: x only grows per thread
        for_each_ix<2>(p.nz_i, p.val, e_in, e_end, vflag, [&](int x, int32_t key, float v) {
          uint32_t h = sp_hash(key);
          int li;
          for (;;) {
            const int k2 = keys[h];
            if (k2 == key) {
              li = lis[h];
              break;
            }
            if (k2 == -1) {
              li = 0xFFFF;
              break;
            }
            h = (h + 1) & (SP_HS - 1);
          }
          if (li == 0xFFFF) {
            *vflag = 1;
            return;
          }
          while (tfp[fl + 1] <= x) ++fl;
          uint8_t* dst = xd + (li >> 6) * XD_CHUNK + (fl >> 3) * 1024 + (fl & 7) * 128 +
                         ((((li & 63) >> 3) ^ (fl & 7)) << 4) + (li & 7) * 2;
          atoms_add16<F16>(dst, v);
        });
      };
      // insert pass: claim a slot for every new i (ids assigned afterwards)
      auto insert = [&]() {
        for_each_i<4>(p.nz_i, e_in, e_end, vflag, [&](int, int32_t key) {
          uint32_t h = sp_hash(key);
          for (;;) {
            int old = keys[h];
            if (old == key) return;
            if (old == -1) {
              if (*vcount >= SP_NI) {  // bounds the claims: <= SP_NI + SP_NT < SP_HS slots
                *vflag = 1;
                return;
              }
              old = atoms_cas(&keys[h], -1, key);
              if (old == -1) {
                if (atoms_add(&ms->count, 1) >= SP_NI) *vflag = 1;
                return;
              }
              if (old == key) return;
            }
            h = (h + 1) & (SP_HS - 1);
          }
        });
      };
      bool fresh = *vcount == 0;
      bool ok = false;
      if (!fresh) {
        scatter();
        __syncthreads();
        ok = *vflag == 0;
        __syncthreads();
        if (!ok) {  // new keys: extend the table, else start it over for this tile
          for (int e = tid; e < XD_BYTES / 16; e += SP_NT) reinterpret_cast<uint4*>(xd)[e] = make_uint4(0, 0, 0, 0);
          if (tid == 0) ms->ovf = 0;
          __syncthreads();
          insert();
          __syncthreads();
          const bool ovf = *vflag != 0;
          __syncthreads();
          if (ovf) {
            clear_table();
            if (tid == 0) ms->ovf = 0;
            __syncthreads();
            fresh = true;
          }
        }
      }
      if (fresh) {
        insert();
        __syncthreads();
        const bool ovf = *vflag != 0;
        __syncthreads();
        if (ovf) {  // more than SP_NI distinct i: fewer fibers
          clear_table();
          __syncthreads();
          nt = max(1, nt >> 1);
          continue;
        }
      }
      if (!ok) {
        // ids for the keys without one, in slot order: thread t owns SP_SPT slots
        const int base0 = *vcount;
        int c = 0;
#pragma unroll
        for (int k = 0; k < SP_SPT; ++k) c += keys[tid * SP_SPT + k] != -1 && lis[tid * SP_SPT + k] == 0xFFFF;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) ms->wsum[warp] = incl;
        __syncthreads();
        int base = incl - c;
        for (int w = 0; w < warp; ++w) base += ms->wsum[w];
        int nassigned = 0;
        for (int w = 0; w < SP_NT / 32; ++w) nassigned += ms->wsum[w];
        base = base0 - nassigned + base;  // count already includes the new keys
#pragma unroll
        for (int k = 0; k < SP_SPT; ++k) {
          const int key = keys[tid * SP_SPT + k];
          if (key != -1 && lis[tid * SP_SPT + k] == 0xFFFF) {
            lis[tid * SP_SPT + k] = static_cast<uint16_t>(base);
            si[base] = key;
            ++base;
          }
        }
        __syncthreads();
        scatter();
      }
      const int ni = *vcount;
      ptx::fence_proxy_async_smem();
      __syncthreads();
      // next cursor (every thread computes the same)
      int64_t f_next = f + nf, e_next;
      if (nt == 1 && e_end < fend0) {
        f_next = f;
        e_next = e_end;
      } else {
        if (nt == 1) f_next = f + 1;
        e_next = f_next < fs1 ? p.fiber_ptr[f_next] : 0;
      }
      {
        const int nch = (ni + 63) >> 6;
        const int k16_last = (ni - (nch - 1) * 64 + 15) >> 4;
        // 2-3. row blocks: gathered-U mode 1, then mode 2 into Z
        const int total = p.nrb * nch;
        auto issue = [&](int t) {
          const int rb = t / nch, c = t - rb * nch;
          const uint32_t gg = g + static_cast<uint32_t>(t);
          const int slot = static_cast<int>(gg % SP_NS);
          if (gg >= SP_NS) ptx::mbar_wait(&ms->mma_done[slot], ((gg / SP_NS) + 1) & 1);
          uint8_t* dst = ring + slot * UC_BYTES;
          const int kcnt = min(64, ni - c * 64);
          for (int x = tid; x < kcnt * 16; x += SP_NT) {
            const int k = x >> 4, qq = x & 15;
            const __nv_bfloat16* src = p.ut + static_cast<int64_t>(si[c * 64 + k]) * p.ld_ut + rb * 128 + qq * 8;
            ptx::cp_async16(dst + ((k >> 3) * 2 + (qq >> 3)) * 1024 + (k & 7) * 128 + (((qq & 7) ^ (k & 7)) << 4),
                            src);
          }
          ptx::cp_async_commit();
        };
        const int pre = min(SP_AHEAD, total);
        for (int t = 0; t < pre; ++t) issue(t);
        int t = 0;
        for (int rb = 0; rb < p.nrb; ++rb) {
          // V rows of this block's replicas for the tile's fibers (MN-major B of mode 2)
          constexpr int VU = 1024 / SP_NT;
          uint4 vreg[VU];
#pragma unroll
          for (int u = 0; u < VU; ++u) {
            const int x = tid + u * SP_NT, fl = x >> 4, qq = x & 15;
            const int64_t col = static_cast<int64_t>(rb) * p.n2 + qq * 8;
            vreg[u] = make_uint4(0, 0, 0, 0);
            if (fl < nf && qq * 8 < p.n2 && col < p.ld_vtj)
              vreg[u] = __ldg(reinterpret_cast<const uint4*>(p.vtj + static_cast<int64_t>(tfj[fl]) * p.ld_vtj + col));
          }
          for (int c = 0; c < nch; ++c, ++t) {
            const int allow = min(SP_AHEAD - 1, total - t - 1);
            if (allow >= 2) ptx::cp_async_wait<2>();
            else if (allow == 1) ptx::cp_async_wait<1>();
            else ptx::cp_async_wait<0>();
            ptx::fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
              ptx::tc_fence_after();
              const int slot = static_cast<int>((g + static_cast<uint32_t>(t)) % SP_NS);
              const uint32_t a0 = ring_u + slot * UC_BYTES, b0 = xd_u + c * XD_CHUNK;
              const int nk = c == nch - 1 ? k16_last : 4;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                if (kk < nk)
                  ptx::mma_bf16(d1, ptx::sw128_mn_desc(a0 + kk * 4096, 1024, 2048), ptx::sw128_desc(b0 + kk * 32),
                                idesc1, (c | kk) != 0);
              ptx::mma_commit(&ms->mma_done[slot]);
              if (c == nch - 1) ptx::mma_commit(&ms->d1_full);
            }
            if (t + SP_AHEAD < total) issue(t + SP_AHEAD);
          }
          // D1 -> bf16 A operand of mode 2 (row r, fibers contiguous)
          ptx::mbar_wait(&ms->d1_full, n1 & 1);
          ++n1;
          ptx::tc_fence_after();
          if (warp < 8) {
            float v[32];
            ptx::tmem_ld32(d1 + lane_addr + hh * 32, v);
            ptx::tmem_wait_ld();
            uint8_t* row = a2 + r * 128;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int q8 = hh * 4 + q4;
              *reinterpret_cast<uint4*>(row + ((q8 ^ (r & 7)) << 4)) = ptx::pack8(v + q4 * 8, F16);
            }
          }
#pragma unroll
          for (int u = 0; u < VU; ++u) {
            const int x = tid + u * SP_NT, fl = x >> 4, qq = x & 15;
            *reinterpret_cast<uint4*>(vg + ((fl >> 3) * 2 + (qq >> 3)) * 1024 + (fl & 7) * 128 +
                                      (((qq & 7) ^ (fl & 7)) << 4)) = vreg[u];
          }
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          __syncthreads();
          if (tid == 0) {
            ptx::tc_fence_after();
            const int nk2 = (nf + 15) >> 4;
            const uint32_t a0 = ptx::smem_u32(a2), b0 = ptx::smem_u32(vg);
            for (int kk = 0; kk < nk2; ++kk)
              ptx::mma_bf16(d2, ptx::sw128_desc(a0 + kk * 32), ptx::sw128_mn_desc(b0 + kk * 4096, 1024, 2048),
                            idesc2, kk != 0);
            ptx::mma_commit(&ms->d2_full);
          }
          ptx::mbar_wait(&ms->d2_full, n2c & 1);
          ++n2c;
          ptx::tc_fence_after();
          // diagonal replica block of D2 -> Z (zeroed by the host; fire-and-forget reductions)
          const int64_t prep = static_cast<int64_t>(rb) * rpb + p_local;
          for (int cb = 0; cb < (warp < 8 ? half : 0); cb += 16) {
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
          __syncthreads();
        }
        g += static_cast<uint32_t>(total);
      }
      f = f_next;
      e_in = e_next;
      nt = (f < fs1 && e_in != p.fiber_ptr[f]) ? 1 : min(SP_NF, nt * 2);
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

bool Plan::sparse_tc_ok() const {
  // XTSG_SPARSE_TC=0 selects the SIMT fiber kernel (read per call: tests A/B both)
  const char* e = std::getenv("XTSG_SPARSE_TC");
  return (!e || std::atoi(e) != 0) && tensor_core() && !comp() && mpad <= lpad && lpad <= 128;
}

// CSF (slices -> fibers -> nonzeros, already validated, on the device) -> Z
// through the tensor-core tile kernel, then mode 3 over the slices.
void Plan::sparse_tc(int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr, const int64_t* fiber_ptr,
                     const int32_t* fiber_j, const int32_t* nz_i, const float* val, float* ydev, bool accumulate,
                     cudaStream_t s) {
  const int64_t plrows = vP * lpad;
  DevBuf<float> z(static_cast<size_t>(vP * n_slices * mpad * lpad), s);
  z.zero();  // the kernel adds every tile's contribution (and skips empty slices)
  DevBuf<unsigned long long> ctr(1, s);
  ctr.zero();
  SpTcParams prm{};
  prm.slice_ptr = slice_ptr;
  prm.fiber_ptr = fiber_ptr;
  prm.fiber_j = fiber_j;
  prm.nz_i = nz_i;
  prm.val = val;
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
  prm.counter = ctr.ptr;
  auto launch = [&](auto kern) {
    XCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SP_SMEM));
    const int grid = static_cast<int>(std::min<int64_t>(n_slices, sm_count()));
    kern<<<grid, SP_NT, SP_SMEM, s>>>(prm);
  };
  if (fp16()) launch(sparse_tc_kernel<true>);
  else launch(sparse_tc_kernel<false>);
  XLAUNCH_CHECK();
  sparse_mode3(z.ptr, slice_k, n_slices, ydev, accumulate, s);
}

// sorted COO (keys = k*J + j ascending, payload = (i << 32) | value bits) ->
// CSF arrays -> sparse_tc
void Plan::sparse_tc_sorted(const uint64_t* skeys, const uint64_t* spay, const int32_t* si_in, const float* sv_in,
                            int64_t nnz, float* ydev, bool accumulate, cudaStream_t s) {
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
  int64_t nf = 0;
  XCUDA(cudaMemcpyAsync(&nf, nruns.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  DevBuf<int64_t> fptr(static_cast<size_t>(nf + 1), s);
  scan_ptr(fcnt.ptr, nf, fptr.ptr, s);
  fcnt.release();
  DevBuf<int32_t> fj(static_cast<size_t>(nf), s), fk(static_cast<size_t>(nf), s);
  fiber_split_kernel<<<gridn(nf), 256, 0, s>>>(fkeys.ptr, nf, J, fj.ptr, fk.ptr);
  XLAUNCH_CHECK();
  fkeys.release();
  // slices: runs of equal k over the fibers
  DevBuf<int32_t> uk(static_cast<size_t>(nf), s), scnt(static_cast<size_t>(nf), s);
  {
    size_t tb = 0;
    XCUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, fk.ptr, uk.ptr, scnt.ptr, nruns.ptr + 1, nf, s));
    DevBuf<uint8_t> tmp(tb, s);
    XCUDA(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, fk.ptr, uk.ptr, scnt.ptr, nruns.ptr + 1, nf, s));
    count_launch();
  }
  int64_t kd = 0;
  XCUDA(cudaMemcpyAsync(&kd, nruns.ptr + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  XCUDA(cudaStreamSynchronize(s));
  DevBuf<int64_t> sptr(static_cast<size_t>(kd + 1), s);
  scan_ptr(scnt.ptr, kd, sptr.ptr, s);
  fk.release();
  scnt.release();
  DevBuf<int32_t> bi;
  DevBuf<float> bv;
  const int32_t* ni = si_in;
  const float* nv = sv_in;
  if (spay) {
    bi = DevBuf<int32_t>(static_cast<size_t>(nnz), s);
    bv = DevBuf<float>(static_cast<size_t>(nnz), s);
    payload_unpack_kernel<<<gridn(nnz), 256, 0, s>>>(spay, nnz, bi.ptr, bv.ptr);
    XLAUNCH_CHECK();
    ni = bi.ptr;
    nv = bv.ptr;
  }
  sparse_tc(kd, uk.ptr, sptr.ptr, fptr.ptr, fj.ptr, ni, nv, ydev, accumulate, s);
}

}  // namespace xtsg
