#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace xtsg {

// compensated mode: X is scaled by 2^comp_x_shift(amax) before its hi/lo split
// so that max |x| lands in [2^13, 2^14)
__device__ __forceinline__ int comp_x_shift(const unsigned* amax) {
  return 13 - ilogbf(fmaxf(__uint_as_float(*amax), 1e-30f));
}

struct Plan {
  xtsg_plan_desc desc;
  // Calls on one plan serialise: the host side under `mu`, the device side
  // through `ev_done` (each call's stream waits for the previous call's work,
  // on whatever stream it ran), because Z, the lane counters and the pinned
  // ring are per plan. Concurrent compressions use one plan each.
  std::mutex mu;
  cudaEvent_t ev_done = nullptr;
  int device = 0;
  cudaStream_t st = nullptr;       // creation stream
  cudaStream_t copy_st = nullptr;  // H2D slab stream
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  // fp64 reference-layout ensemble (kept for the fp64 path; W also feeds Wf)
  DevBuf<double> u64, v64, w64;
  // tensor-core operands
  int64_t lpad = 0, mpad = 0, rpb = 0, n2 = 0, rows_u = 0, ld_u = 0, ld_v = 0;
  // virtual replicas: reduced dims above 128 are split into lsplit x msplit
  // pieces of at most Lv x Mv rows (each a tensor-core replica of its own
  // with the same W); vP = P * lsplit * msplit. M splits repeat the mode-1
  // product of their rows (algorithmic flops stay P*L*...), L splits are free.
  int64_t vP = 0, lsplit = 1, msplit = 1, Lv = 0, Mv = 0;
  DevBuf<__nv_bfloat16> ustack, vt;
  DevBuf<float> wf;
  DevBuf<float> zbuf;
  DevBuf<unsigned> sync_ctr;  // lane-barrier counters of the pair TTM kernel
  DevBuf<__nv_bfloat16> ut;   // i-major U copy for the sparse path (lazy)
  DevBuf<__nv_bfloat16> vtj;  // j-major V copy for the sparse path (lazy)
  int grid_limit = 0;  // testing knob: cap on persistent CTAs (0 = #SMs)
  // host-narrowing pipeline (f32/f64 host input on a bf16 plan): pinned bf16
  // slab buffers and their device twins, cached across calls
  void* hpin[2] = {nullptr, nullptr};
  size_t hpin_bytes = 0;
  DevBuf<__nv_bfloat16> dstage[2];
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr};
  void compress_host_narrow(const void* x, int32_t dtype, const int64_t ld[2], const int64_t off[3],
                            const int64_t ext[3], float* ydst, bool acc_first, cudaStream_t s);
  // Live profiling (xtsg_plan_profile): CUDA events around every fused-TTM
  // and mode-3 launch on the launching stream, plus algorithmic flop counts.
  bool profiling = false;
  struct EvPair {
    cudaEvent_t a, b;
  };
  std::vector<EvPair> ev_pool, ev_fused, ev_mode3;
  double flops_fused = 0.0, flops_mode3 = 0.0;
  EvPair take_pair();

  // two-stage plans: stage-1 plan over the shared inner matrices + outer (fp64)
  std::unique_ptr<Plan> stage1;
  DevBuf<double> outer[3];
  int64_t inner_dims[3] = {0, 0, 0};

  // compensated fp16 hi/lo mode (XTSG_PREC_FP16X3): U, V and X as two fp16
  // planes each (hi, lo = v - hi); `amax` holds the current launch's max |x|
  // (float bits, or an upper bound for factored sources) that sets X's
  // power-of-two pre-scale (comp_x_shift) and mode 3's undo; comp_bu/bv are
  // the pre-scales 2^-b of U/V (max in [2^13, 2^14)); mode 3 accumulates in
  // fp64 into comp_y (padded layout)
  DevBuf<unsigned> amax;
  const unsigned* cur_amax = nullptr;  // the amax slot of the slab being consumed (null: amax.ptr)
  int comp_bu = 0, comp_bv = 0;
  double* comp_y = nullptr;
  bool comp() const { return desc.precision == XTSG_PREC_FP16X3; }
  // fp32 mode-1 accumulation per chunk of comp_kpc 64-wide i steps
  int comp_kpc() const;
  int comp_c0(int64_t ni) const;
  void comp_finish(const double* y64, float* y, bool accumulate, cudaStream_t s);

  bool tensor_core() const {
    return desc.precision == XTSG_PREC_BF16 || desc.precision == XTSG_PREC_FP16 || comp();
  }
  bool fp16() const { return desc.precision == XTSG_PREC_FP16; }
  bool f16_operands() const { return fp16() || comp(); }
  void check_finite16(const float* y, int64_t n, cudaStream_t s);
  bool virt_padded() const {
    return lsplit > 1 || msplit > 1 || lpad != desc.reduced[0] || mpad != desc.reduced[1];
  }
  // ypad (vP x (Mpad*Lpad) x N, the tensor-core layout) -> y (P replicas L x M x N)
  void compact(const float* ypad, float* y, bool accumulate, cudaStream_t s);
  explicit Plan(const xtsg_plan_desc& d);
  Plan(const xtsg_plan_desc& d, const double* u, const double* v, const double* w);
  void build_tc_operands();
  void stage2(const float* zin, float* y, bool accumulate, cudaStream_t s);
  ~Plan();
  void check_block(const int64_t off[3], const int64_t ext[3]) const;
  void compress(const void* x, int32_t dtype, const int64_t ld[2], const int64_t off[3], const int64_t ext[3],
                void* y, bool accumulate, cudaStream_t s);
  void run_bf16_block(const __nv_bfloat16* x, int64_t ld0, int64_t ld1, const int64_t off[3],
                      const int64_t ext[3], float* ydst, bool first_accumulate, cudaStream_t s,
                      const __nv_bfloat16* x_lo = nullptr);
  void ensure_z(int64_t floats, cudaStream_t s);
  void compress_factors(const double* a, const double* b, const double* c, int64_t rank, int64_t k0, int64_t k1,
                        float* y, bool accumulate, cudaStream_t s);
  void compress_coo(const int32_t* i, const int32_t* j, const int32_t* k, const float* val, int64_t nnz, float* y,
                    bool accumulate, cudaStream_t s);
  void compress_csf(int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr, int64_t n_fibers,
                    const int32_t* fiber_j, const int64_t* fiber_ptr, int64_t nnz, const int32_t* nz_i,
                    const float* val, float* y, bool accumulate, cudaStream_t s);
  void ensure_sparse_operands(cudaStream_t s);
  void coo_slices(const int32_t* si, const int32_t* sj, const float* sv, const int64_t* off, const int32_t* cnt,
                  const int32_t* uk, int64_t kd, float* ydev, bool accumulate, cudaStream_t s);
  // mode 3 of the sparse path: y (+)= Z[p][kd][m][l] x W_p[:, uk]^T
  void sparse_mode3(const float* z, const int32_t* uk, int64_t kd, float* ydev, bool accumulate, cudaStream_t s);
  // tensor-core sparse path (sparse_tc.cu): dense tiles of a slice
  bool sparse_tc_ok() const;
  void sparse_tc(int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr, int64_t n_fibers,
                 const int64_t* fiber_ptr, const int32_t* fiber_j, int64_t nnz, const int32_t* nz_i,
                 const float* val, float* ydev, bool accumulate, cudaStream_t s);
  // skeys / spay are consumed (released as soon as they are read)
  void sparse_tc_sorted(DevBuf<uint64_t>& skeys, DevBuf<uint64_t>* spay, const int32_t* si, const float* sv,
                        int64_t nnz, float* ydev, bool accumulate, cudaStream_t s);
  bool sparse_tc_coo32(const int32_t* i, const int32_t* j, const int32_t* k, const float* val, int64_t nnz,
                       float* ydev, bool accumulate, cudaStream_t s);
  // 32-bit (rank k, rank j) keys + (i, value) payload, already sorted
  void sparse_tc_sorted32(DevBuf<uint32_t>& skeys, DevBuf<uint64_t>& spay, const int32_t* invk, const int32_t* invj,
                          int64_t nju, int64_t nnz, float* ydev, bool accumulate, cudaStream_t s);
  void sparse_tc_tail(int64_t nf, DevBuf<int64_t>& fptr, DevBuf<int32_t>& fj, DevBuf<int32_t>& fk,
                      const int32_t* ni, const float* nv, DevBuf<int32_t>& bi, DevBuf<float>& bv, int64_t nnz,
                      float* ydev, bool accumulate, cudaStream_t s);
};

// RAII use of a plan by one C-ABI call on stream s (see Plan::mu).
struct PlanUse {
  Plan* p;
  cudaStream_t s;
  std::lock_guard<std::mutex> lk;
  PlanUse(Plan* p_, cudaStream_t s_) : p(p_), s(s_), lk(p_->mu) { XCUDA(cudaStreamWaitEvent(s, p->ev_done, 0)); }
  ~PlanUse() { cudaEventRecord(p->ev_done, s); }
  PlanUse(const PlanUse&) = delete;
  PlanUse& operator=(const PlanUse&) = delete;
};

}  // namespace xtsg
