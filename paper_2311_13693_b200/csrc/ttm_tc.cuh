#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xtsg {

struct TtmParams {
  int32_t n_rb;      // row blocks of 128 stacked U rows
  int32_t kc;        // slices k in this launch (units = n_rb * kc)
  int32_t k_first;   // first slice (X map coordinate)
  int32_t j_tiles;   // ceil(nj / 256)
  int32_t k_steps;   // ceil(ni / 64)
  int32_t lpad, rpb; // padded L, replicas per row block (lpad * rpb == 128)
  int32_t n2;        // rpb * mpad (mode-2 MMA N)
  int32_t count;     // P
  int32_t k16_last;        // K=16 MMA slices holding data in the last i step (1..4)
  int32_t n_last;          // UMMA N of the last j tile (multiple of 16, <= 256)
  int32_t chunks_last;     // 64-wide mode-2 chunks in the last j tile
  int32_t k16_chunk_last;  // K=16 slices in the last chunk of the last tile
  int32_t rb_group;        // row blocks (pairs, for the pair kernel) per unit group
  int32_t lanes;           // pair kernel: static slice lanes (0 = round robin)
  unsigned* sync;          // pair kernel: per-lane slot counters (null = no lane barrier)
  int32_t sync_j;          // pair kernel: lane barrier every sync_j j tiles
  uint64_t u_policy, x_policy;  // L2 cache-policy hints of the U / X tile loads
  int32_t f16;             // operands are fp16 (XTSG_PREC_FP16) instead of bf16
  // compensated fp16 hi/lo mode (XTSG_PREC_FP16X3, pair kernel only)
  int32_t comp;            // 1: three products per mode, planes below
  int32_t u_plane_rows;    // rows between the U planes (Uh, Ul)
  int32_t v_plane_rows;    // rows between the V planes (Vh, Vl)
  int32_t i_chunks, kpc;   // i steps split into i_chunks chunks of kpc (0: one chunk)
  const unsigned* amax;    // max |x| of this launch's X (float bits; mode 3's scale)
  int32_t comp_c0;         // 2^-comp_c0 scales the mode-1 result before its split
  float* z;          // out: Z[p][kk][m][l], kk in [0, kc)
};

struct TtmLaunch {
  const void* u;      // bf16/fp16 stacked U: rows_u x ld_u (row-major), columns [0, ni) used
  int64_t rows_u, ld_u;
  const void* x;      // bf16 X block: (i, j, k) at i + ld_x0*j + ld_x1*k
  const void* x_lo;   // compensated: the lo' plane of X, same layout (else null)
  int64_t ni, nj, nk, ld_x0, ld_x1;
  const void* v;      // bf16 Vt: rows_v x ld_v (row (p,m), j contiguous)
  int64_t rows_v, ld_v;
  int mpad;
  int grid_limit;     // 0 = number of SMs
  unsigned* sync;     // >= 256 zeroable counters for the pair kernel's lane barrier (optional)
  TtmParams prm;
};

void launch_ttm_fused(const TtmLaunch& l, cudaStream_t st);
int ttm_block_n();
int ttm_cluster_size();
bool ttm_pair_supported(const TtmLaunch& l);
void launch_ttm_pair(const TtmLaunch& l, cudaStream_t st);
bool ttm_pair_enabled();


}  // namespace xtsg
