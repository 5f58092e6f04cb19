/*
 * xtsg — C ABI of the B200-native Exascale-Tensor compression path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/xts/{compression,cp_als,alignment}.hpp).
 * Every entry point below names the reference function it replaces
 * (file:line); the C++ facade paper_2311_13693_b200/facade/xts_facade.cpp
 * implements the reference's own declarations (the unmodified
 * headers under /root/reference/proj/include/xts) on top of them, with the exact C++
 * signatures and exception types.
 *
 * Conventions (shared by every function):
 *  - Plain pointers and sizes only. Matrices are column-major
 *    ((i,j) at i + rows*j, tensor.hpp:10-20); tensors are column-major
 *    ((i,j,k) at i + n1*(j + n2*k), tensor.hpp:30-44); "P matrices back to
 *    back" means replica p starts at p*rows*cols.
 *  - A pointer may be host memory (pageable or pinned) or device memory of
 *    the calling thread's current CUDA device; the library detects which and
 *    stages host buffers itself. Results land where the output pointer points.
 *  - Return value is a status code. Exceptions never cross the ABI: the
 *    reference's exception taxonomy (errors.hpp:10-59) maps to the codes
 *    below, the payload (effective_rank, column, survivors/required) is read
 *    back with xtsg_last_payload(), the message with xtsg_last_error().
 *    Both are thread-local.
 *  - Thread-safe and re-entrant: each host thread gets its own CUDA stream
 *    (the reference calls comp/cp_als concurrently from parallel_for,
 *    pipeline.cpp:386-434). Calls that share one xtsg_plan serialise on it
 *    (host mutex, and each call's stream waits for the previous call's device
 *    work), because a plan owns its scratch; use one plan per concurrent
 *    stream for overlap. There is no CPU fallback: without a usable sm_100
 *    device every compute entry point returns XTSG_E_CUDA.
 */
#ifndef XTSG_H_
#define XTSG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:10-59) ---------------------------------- */
#define XTSG_OK 0
#define XTSG_E_USAGE 1        /* xts::UsageError */
#define XTSG_E_DATA 2         /* xts::DataError */
#define XTSG_E_ILLPOSED 3     /* xts::IllPosedError; payload(0) = effective_rank */
#define XTSG_E_DEGENERATE 4   /* xts::DegenerateColumnError; payload(0) = column */
#define XTSG_E_INSUFFICIENT 5 /* xts::InsufficientReplicasError; payload(0)=survivors, (1)=required */
#define XTSG_E_HALFRANGE 6    /* xts::HalfRangeError */
#define XTSG_E_STAGE 7        /* xts::StageError; payload(0) = stage index */
#define XTSG_E_CUDA 8         /* device missing / CUDA runtime failure */
#define XTSG_E_INTERNAL 99

const char* xtsg_last_error(void);
int64_t xtsg_last_payload(int32_t which);
/* Library/ABI version (major*100 + minor). */
int32_t xtsg_version(void);
/* 1 when an sm_100 device is usable by this thread, else 0. */
int32_t xtsg_device_ready(void);
/* Create the CUDA context and this thread's stream ahead of the first call. */
int32_t xtsg_warmup(void);

/* ---- ensembles (compression.hpp:13-65, compression.cpp:15-200) --------- */
#define XTSG_KIND_GAUSSIAN 0
#define XTSG_KIND_SPARSE 1
#define XTSG_KIND_TWO_STAGE 2

typedef struct xtsg_ensemble_spec {
  int32_t kind;       /* EnsembleSpec::Kind */
  int32_t inner_kind; /* TwoStageSpec::inner_kind: 0 gaussian, 1 sparse */
  double s;           /* SparseProjectionSpec::s for kind == sparse */
  double alpha, beta, gamma; /* TwoStageSpec ratios */
  double inner_s;     /* TwoStageSpec::inner_spec.s */
} xtsg_ensemble_spec;

/* compute_replica_count (compression.cpp:82-95) */
int32_t xtsg_replica_count(const int64_t dims[3], const int64_t reduced[3], int64_t slack,
                           int64_t* out);

/* gen_gaussian (compression.cpp:97-103): one polar stream over all entries. */
int32_t xtsg_gen_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* gen_sparse_projection (compression.cpp:105-113) */
int32_t xtsg_gen_sparse_projection(int64_t rows, int64_t cols, double s, uint64_t seed,
                                   double* out);

/* make_ensemble (compression.cpp:115-200). u: count matrices reduced[0] x dims[0]
 * back to back (likewise v, w). For two-stage, inner_* (alpha*L x I ...) and
 * outer_* (count matrices L x alpha*L ...) are written when non-null.
 * Bit-exact with the reference on this image (glibc 2.39 log). */
int32_t xtsg_make_ensemble(const int64_t dims[3], const int64_t reduced[3], int64_t count,
                           int64_t shared_rows, const xtsg_ensemble_spec* spec, uint64_t seed,
                           double* u, double* v, double* w, double* inner_u, double* inner_v,
                           double* inner_w, double* outer_u, double* outer_v,
                           double* outer_w);

/* ---- compression, fp64 compatibility path ------------------------------ */
/* comp (compression.cpp:211-213): y (l x m x n) = t x1 u x2 v x3 w, modes in
 * the reference order 1 -> 2 -> 3, fp64 on the device. */
int32_t xtsg_comp(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                  int64_t l, const double* v, int64_t m, const double* w, int64_t n, double* y);

/* comp_from_factors (compression.cpp:215-220) */
int32_t xtsg_comp_from_factors(const double* a, const double* b, const double* c, int64_t i,
                               int64_t j, int64_t k, int64_t rank, const double* u, int64_t l,
                               const double* v, int64_t m, const double* w, int64_t n,
                               double* y);

/* reconstruct (tensor.cpp:133-150) */
int32_t xtsg_reconstruct(const double* a, const double* b, const double* c, int64_t i,
                         int64_t j, int64_t k, int64_t rank, double* out);

/* comp_blocked (compression.cpp:332-404) as a push stream. begin() checks the
 * grid (BlockGrid ctor :222-230) and ensemble shapes; push() validates the
 * record (:319-328) and rejects duplicates (:344-351, XTSG_E_DATA); finish()
 * rejects gaps and writes the count replicas back to back. deterministic=1
 * reassembles and runs one-shot comp (bitwise grid independent, :355-379);
 * deterministic=0 compresses each block on arrival into fp64 accumulators in
 * a fixed order (:381-403). */
typedef struct xtsg_blocked xtsg_blocked;
int32_t xtsg_blocked_begin(const int64_t dims[3], const int64_t block[3], int64_t count,
                           const int64_t reduced[3], const double* u, const double* v,
                           const double* w, int32_t deterministic, xtsg_blocked** out);
int32_t xtsg_blocked_push(xtsg_blocked* h, const int64_t cell[3], const int64_t shape[3],
                          const double* data);
/* A region of whole cells at once: offset/shape in elements, aligned to the
 * grid's cells (the region's end may be the tensor's ragged edge); data
 * column-major over the region. Marks every covered cell as seen (duplicates
 * -> XTSG_E_DATA). deterministic=0 compresses the region like one block (its
 * cells' contributions summed in fp64, equal to the per-cell sum up to
 * rounding). The facade pushes an untouched
 * in-memory block source (make_memory_block_source, compression.cpp:256-278)
 * as one region: the tensor goes to the device once, without the per-block
 * host copies. */
int32_t xtsg_blocked_push_region(xtsg_blocked* h, const int64_t offset[3], const int64_t shape[3],
                                 const double* data);
int32_t xtsg_blocked_finish(xtsg_blocked* h, double* y);
void xtsg_blocked_destroy(xtsg_blocked* h);

/* ---- precision model (half.hpp, mixed.hpp) ----------------------------- */
/* Device replays of the reference's binary16 arithmetic, bit-identical to it:
 * values are binary16 numbers carried as doubles, every product is a
 * half_gemm (fixed k-inner order, one rounding per product and per add). */
#define XTSG_SPLIT_ROUND 0   /* round_to_half only (residual unused) */
#define XTSG_SPLIT_FULL 1    /* fp16_split: half + residual == x exactly */
#define XTSG_SPLIT_STORED 2  /* fp16_split_stored: residual itself binary16 (scaled 2^11) */

/* split_matrix / split_tensor / round_matrix_to_half / round_tensor_to_half
 * (mixed.cpp:11-61) over n values; XTSG_E_HALFRANGE like double_to_half_bits
 * (half.cpp:10-47) for NaN, Inf or magnitudes rounding above 65504. */
int32_t xtsg_split_half(const double* x, int64_t n, int32_t mode, double* half, double* residual);

/* half_gemm (mixed.cpp:63-76): out (rows x cols) = a (rows x inner) * b (b_rows x cols). */
int32_t xtsg_half_gemm(const double* a, int64_t rows, int64_t inner, const double* b, int64_t b_rows,
                       int64_t cols, double* out);

/* comp_with(t, u, v, w, &half_gemm) (compression.cpp:202-209, mixed.cpp:84-86) */
int32_t xtsg_comp_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                       const double* v, int64_t m, const double* w, int64_t n, double* y);

/* comp_mixed (mixed.cpp:88-98, the paper's Eq. 5): the half x half x half x
 * half term plus the four single-residual terms, summed in the reference's
 * order. Inputs are the half/residual parts of split_tensor / split_matrix. */
int32_t xtsg_comp_mixed(const double* t_half, const double* t_res, int64_t n1, int64_t n2, int64_t n3,
                        const double* u_half, const double* u_res, int64_t l, const double* v_half,
                        const double* v_res, int64_t m, const double* w_half, const double* w_res,
                        int64_t n, double* y);

/* comp_naive_half (mixed.cpp:100-104) */
int32_t xtsg_comp_naive_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                             int64_t l, const double* v, int64_t m, const double* w, int64_t n,
                             double* y);

/* ---- compression, tensor-core fast path (the B200 hot path) ------------ */
/* A plan owns the device-resident ensemble of one compression job: the P
 * replicas' U stacked into one (P*L) x I bf16 operand, V transposed per
 * replica, W in fp32, all generated on the device from the seed with the
 * bit-exact RNG above (make_ensemble semantics). It then compresses dense
 * slabs/blocks of X with the fused tcgen05 TTM kernel. */
#define XTSG_PREC_FP64 0   /* DFMA chain; reference-order arithmetic */
#define XTSG_PREC_BF16 1   /* tcgen05 kind::f16, bf16 operands, fp32 accumulation */
#define XTSG_PREC_FP16 2   /* tcgen05 kind::f16, fp16 operands (3 more mantissa bits, range 65504:
                              U scaled by 2^-s / W by 2^s internally; overflow -> XTSG_E_HALFRANGE) */
#define XTSG_PREC_FP16X3 3 /* compensated tensor-core mode (the reference's Eq. 5 split, mixed.cpp:18-24,
                              done on tcgen05): every operand is an fp16 pair (hi, lo = x - hi) after a
                              power-of-two pre-scale that puts its max |x| in [2^13, 2^14) (any input
                              magnitude), each mode product is hi*hi + hi*lo + lo*hi (3 MMAs; lo*lo
                              dropped, 2^-22 relative), the mode-1 sum over i in chunks, the mode-3 sum
                              over k in fp64; replicas ~2.5e-6 relative vs fp64 at C2/C3; output fp32
                              like the other tensor-core modes */

#define XTSG_DTYPE_BF16 0
#define XTSG_DTYPE_F32 1
#define XTSG_DTYPE_F64 2
#define XTSG_DTYPE_F16 3

typedef struct xtsg_plan_desc {
  int64_t dims[3];     /* I, J, K */
  int64_t reduced[3];  /* L, M, N */
  int64_t count;       /* P */
  int64_t shared_rows; /* S */
  xtsg_ensemble_spec spec;
  uint64_t seed;       /* make_ensemble seed */
  int32_t precision;   /* XTSG_PREC_* */
  int32_t reserved;
} xtsg_plan_desc;

typedef struct xtsg_plan xtsg_plan;
int32_t xtsg_plan_create(const xtsg_plan_desc* desc, xtsg_plan** out);
void xtsg_plan_destroy(xtsg_plan* plan);

/* Compress the block of X that starts at offset[3] with extent[3] (a cell of
 * a BlockGrid, a mode-3 slab, or the whole tensor) into the P replicas y
 * (P x L x M x N, column-major per replica; fp32 for the tensor-core
 * precisions XTSG_PREC_BF16/FP16/FP16X3, fp64 for XTSG_PREC_FP64), accumulating when accumulate != 0. x points at the block's first element; ld[0] is the
 * distance between consecutive j (>= extent[0]), ld[1] between consecutive k
 * (>= ld[0]*extent[1]), in elements. x may be host or device memory, any
 * XTSG_DTYPE_*; host or non-bf16 input is streamed slab by slab through a
 * double-buffered H2D/convert pipeline overlapped with the tensor cores.
 * stream: cudaStream_t to run on (NULL = the thread's stream). Returns
 * after enqueueing when x and y are device memory, else synchronously. */
int32_t xtsg_plan_compress(xtsg_plan* plan, const void* x, int32_t x_dtype, const int64_t ld[2],
                           const int64_t offset[3], const int64_t extent[3], void* y,
                           int32_t accumulate, void* stream);

/* Same contraction for a tensor given by its CP factors (a: I x R, b: J x R,
 * c: K x R, fp64): blocks of X are generated on the device slab by slab and
 * never exist whole (the 10^12-element configs). k range [k0, k1). */
int32_t xtsg_plan_compress_factors(xtsg_plan* plan, const double* a, const double* b,
                                   const double* c, int64_t rank, int64_t k0, int64_t k1,
                                   void* y, int32_t accumulate, void* stream);

/* ---- multi-GPU compression (SURVEY §8 e; no reference counterpart: the
 * reference compresses on one host, pipeline.cpp:386-405) ------------------
 * One plan per GPU of the node (the same ensemble regenerated on each from
 * the seed), one persistent host thread per GPU, contiguous mode-3 slabs
 * k in [K*g/G, K*(g+1)/G) per GPU, and one NCCL reduce (sum, fp32) of the
 * P*L*M*N partial replicas onto gpus[0] (ncclCommInitAll clique; NCCL is
 * dlopen'ed, "libnccl.so.2"). y: host memory or device memory on gpus[0].
 * gpus may be NULL (devices 0..ngpus-1). Calls on one xtsg_multi serialise. */
typedef struct xtsg_multi xtsg_multi;
int32_t xtsg_multi_create(const xtsg_plan_desc* desc, int32_t ngpus, const int32_t* gpus, xtsg_multi** out);
void xtsg_multi_destroy(xtsg_multi* multi);
/* X = reconstruct(a, b, c) (host fp64 factors I x R, J x R, K x R), every GPU
 * generating its own slab on the device */
int32_t xtsg_multi_compress_factors(xtsg_multi* multi, const double* a, const double* b, const double* c,
                                    int64_t rank, void* y, int32_t accumulate);
/* dense X (whole tensor, column-major with leading dimensions ld like
 * xtsg_plan_compress; host memory is streamed to each GPU slab by slab) */
int32_t xtsg_multi_compress(xtsg_multi* multi, const void* x, int32_t x_dtype, const int64_t ld[2], void* y,
                            int32_t accumulate);
/* Sparse input across the GPUs (SURVEY §8 e: C4 at 1/2/4/8 GPUs; Eq. 3 is
 * linear in the nonzeros, so any partition sums to the whole). Arguments as
 * xtsg_plan_compress_coo / _csf; all inputs host memory (XTSG_E_USAGE for
 * device pointers). COO: GPU g takes nonzeros [nnz*g/G, nnz*(g+1)/G) — a
 * k-range for a k-sorted stream. CSF: GPU g takes a contiguous slice range
 * holding ~1/G of the nonzeros (a k-range for k-sorted slices), pointers
 * rebased on its worker thread. Each share runs as device calls of at most
 * XTSG_SPARSE_CHUNK nonzeros (env, default 2^31; a CSF call holds at least
 * one whole slice), accumulated on its GPU, then the one NCCL reduce. */
int32_t xtsg_multi_compress_coo(xtsg_multi* multi, const int32_t* i, const int32_t* j, const int32_t* k,
                                const float* val, int64_t nnz, void* y, int32_t accumulate);
int32_t xtsg_multi_compress_csf(xtsg_multi* multi, int64_t n_slices, const int32_t* slice_k,
                                const int64_t* slice_ptr, int64_t n_fibers, const int32_t* fiber_j,
                                const int64_t* fiber_ptr, int64_t nnz, const int32_t* nz_i, const float* val,
                                void* y, int32_t accumulate);
/* device time of the last call: max over the GPUs of compress + reduce (ms) */
int32_t xtsg_multi_last_ms(xtsg_multi* multi, double* ms);
/* the NCCL version the multi-GPU path resolved (e.g. 22809), or XTSG_E_CUDA */
int32_t xtsg_nccl_version(int32_t* version);

/* Sparse COO input (new, no reference counterpart; Eq. 3 restricted to the
 * nonzeros, duplicates sum): coordinates int32 SoA (i[nnz], j[nnz], k[nnz]),
 * values fp32. */
int32_t xtsg_plan_compress_coo(xtsg_plan* plan, const int32_t* i, const int32_t* j,
                               const int32_t* k, const float* val, int64_t nnz, void* y,
                               int32_t accumulate, void* stream);

/* Sparse input already in CSF form (new; mode order k -> j -> i): slice q
 * has mode-3 index slice_k[q] and fibers [slice_ptr[q], slice_ptr[q+1]);
 * fiber f has mode-2 index fiber_j[f] and nonzeros [fiber_ptr[f],
 * fiber_ptr[f+1]) with mode-1 indices nz_i and values val. No sort or
 * run-length pass: the fibers feed the fiber kernel directly. Duplicated
 * slices/fibers/coordinates sum. XTSG_E_DATA for out-of-range indices or
 * inconsistent pointers. */
int32_t xtsg_plan_compress_csf(xtsg_plan* plan, int64_t n_slices, const int32_t* slice_k,
                               const int64_t* slice_ptr, int64_t n_fibers, const int32_t* fiber_j,
                               const int64_t* fiber_ptr, int64_t nnz, const int32_t* nz_i,
                               const float* val, void* y, int32_t accumulate, void* stream);

/* Out-of-core .xts source (io.hpp:9-12, io.cpp:55-125).
 * xts_header reads and validates a file's header: kind 0 dense tensor, 1
 * factor triple; dims; rank (factors). plan_compress_file compresses the
 * file's tensor (dims must equal the plan's) straight from disk: dense
 * payloads stream as mode-3 slabs of ~slab_bytes (0 = 512 MiB) through a
 * reader thread and a ring of pinned buffers into the plan's H2D/convert/
 * tensor-core pipeline; factor files generate their slabs on the device.
 * Malformed / truncated files: XTSG_E_DATA with the reference's messages. */
int32_t xtsg_xts_header(const char* path, int32_t* kind, int64_t dims[3], int64_t* rank);
int32_t xtsg_plan_compress_file(xtsg_plan* plan, const char* path, int64_t slab_bytes, void* y,
                                int32_t accumulate, void* stream);

/* Number of this library's kernels launched by the calling thread so far
 * (evidence for the bench's gpu_launches). */
int64_t xtsg_launch_count(void);

/* Live profiling of a plan: when on, every fused-TTM launch and every mode-3
 * GEMM is bracketed by CUDA events on its launching stream. profile() waits
 * for them and returns out[6] = {fused_ms, fused_launches, mode3_ms,
 * mode3_launches, fused_algorithmic_flops, mode3_algorithmic_flops}
 * accumulated since the last reset. */
int32_t xtsg_plan_set_profiling(xtsg_plan* plan, int32_t on);
int32_t xtsg_plan_profile(xtsg_plan* plan, int32_t reset, double out[6]);

/* ---- CP-ALS (cp_als.hpp:10-40, cp_als.cpp:22-111) ---------------------- */
typedef struct xtsg_als_config {
  int64_t rank;
  int64_t max_iters;
  double tol;
  uint64_t seed;
  int32_t init; /* 0 normal, 1 nvecs */
  int32_t reserved;
} xtsg_als_config;

/* relative_error (cp_als.cpp:37-44) */
int32_t xtsg_relative_error(const double* t, int64_t n1, int64_t n2, int64_t n3,
                            const double* a, const double* b, const double* c, int64_t rank,
                            double* out);

/* cp_als on count tensors at once (each n1 x n2 x n3, back to back), one
 * config per tensor. a/b/c: count factor matrices back to back. history:
 * count x max_iters (unused tail untouched), iters/converged per tensor.
 * count == 1 is the drop-in for xts::cp_als. */
int32_t xtsg_cp_als_batched(int64_t count, const double* t, int64_t n1, int64_t n2, int64_t n3,
                            const xtsg_als_config* cfg, double* a, double* b, double* c,
                            int64_t* iters, int32_t* converged, double* history);

/* ---- alignment & recovery (alignment.hpp:11-77, alignment.cpp) --------- */
/* normalize_shared (alignment.cpp:66-85) */
int32_t xtsg_normalize_shared(const double* m, int64_t rows, int64_t cols, int64_t shared_rows,
                              double* normalized, double* pivots);
/* max_trace_assignment (alignment.cpp:87-144) */
int32_t xtsg_max_trace_assignment(const double* objective, int64_t n, int64_t* perm);
/* align_replicas (alignment.cpp:154-218): factors = count triples back to back,
 * each (a: dims[0] x r, b: dims[1] x r, c: dims[2] x r). */
int32_t xtsg_align_replicas(int64_t count, const int64_t dims[3], int64_t r,
                            const double* factors, int64_t shared_rows, int64_t min_survivors,
                            double* aligned, int32_t* dropped, int64_t* survivors,
                            int64_t* n_survivors);
/* solve_stacked_ls (alignment.cpp:220-252 + linalg.cpp:76-92): column-pivoted
 * Householder QR on the device, fp64; rank test like Eigen's
 * ColPivHouseholderQR (|R_ii| > eps * cols * max|R_ii|). */
int32_t xtsg_solve_stacked_ls(int64_t count, const int64_t* rows, int64_t r, int64_t cols,
                              const double* f, const double* u, double* x);
/* recover_perm_scale (alignment.cpp:254-278) */
int32_t xtsg_recover_perm_scale(const double* global_head, const double* sampled,
                                int64_t rows, int64_t cols, int64_t* perm, double* scale);

/* omp_recover (alignment.cpp:306-419): column-wise greedy sparse recovery.
 * Below 4096 atoms one CTA per measured column; from 4096 atoms the atom
 * search of each iteration spreads over the GPU (warp per atom, a batch of
 * the columns' residuals in shared memory), then a per-column Cholesky
 * update. out: atoms x ncols. */
int32_t xtsg_omp_recover(const double* measured, int64_t rows, int64_t ncols, const double* dictionary,
                         int64_t atoms, int64_t sparsity, double residual_tol, double* out);

/* ---- dense linear algebra (linalg.hpp:8-24) ---------------------------- */
/* C (m x n, ldc) = op(A) op(B), fp64 on the device (gemm, linalg.cpp:24-43) */
int32_t xtsg_gemm(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k, const double* a,
                  int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);
/* pseudo_inverse (linalg.cpp:52-61): out is cols x rows */
int32_t xtsg_pseudo_inverse(const double* m, int64_t rows, int64_t cols, double rcond, double* out);
/* leading_left_singular_vectors (linalg.cpp:63-74): out is rows x count */
int32_t xtsg_leading_left_singular_vectors(const double* m, int64_t rows, int64_t cols, int64_t count,
                                           double* out);
/* solve_least_squares (linalg.cpp:76-92): x is cols x nrhs */
int32_t xtsg_solve_least_squares(const double* a, int64_t rows, int64_t cols, const double* rhs,
                                 int64_t nrhs, double* x);

/* ---- synthetic problems and the end-to-end pipeline (pipeline.hpp) ------ */
#define XTSG_LAW_DENSE 0
#define XTSG_LAW_SPARSE 1

/* generate (pipeline.cpp:176-207) without materialization: the factor triple
 * (a: dims[0] x rank, ...) of SyntheticSpec{dims, rank, law, nnz_per_col,
 * seed}, bit-exact with the reference. Host or device outputs. */
int32_t xtsg_generate_factors(const int64_t dims[3], int64_t rank, int32_t law, int64_t nnz_per_col,
                              uint64_t seed, double* a, double* b, double* c);

#define XTSG_MODE_DENSE 0
#define XTSG_MODE_SPARSE 1
#define XTSG_MODE_TWO_STAGE 2

/* PipelineConfig (pipeline.hpp:16-45) minus dims/block/deterministic/workers
 * (the device path has no block grid or worker pool), plus the compression
 * precision: XTSG_PREC_FP64 is the reference's full precision, XTSG_PREC_BF16
 * the tcgen05 path (then replica_fit_tol must admit the bf16 compression
 * error, ~1e-2). */
typedef struct xtsg_pipeline_config {
  int64_t reduced[3];
  int64_t rank;
  int64_t replicas;      /* < 1 -> compute_replica_count(dims, reduced, slack) */
  int64_t slack;         /* 10 */
  int64_t shared;        /* < 1 -> min(2 * rank, min reduced) */
  int32_t mode;          /* XTSG_MODE_* */
  int32_t precision;     /* XTSG_PREC_FP64 / XTSG_PREC_BF16 */
  double alpha, beta, gamma;  /* 1.6 */
  double projection_s;   /* 0 -> max(1, min dims/reduced) */
  int64_t omp_sparsity;  /* required for sparse and two-stage */
  double omp_residual_tol;  /* 1e-9 */
  int64_t sample_b;      /* < 1 -> max(2 * rank, 8) */
  uint64_t seed;
  int64_t als_max_iters; /* 500 */
  double als_tol;        /* 1e-10 */
  double replica_fit_tol;  /* 1e-6 */
  int64_t als_restarts;  /* 3 */
} xtsg_pipeline_config;

/* RunMetrics (metrics.hpp) subset; stages: compression, decomposition,
 * alignment, recovery. status 0 skipped, 1 ok, 2 error. */
typedef struct xtsg_pipeline_metrics {
  double stage_seconds[4];
  int32_t stage_status[4];
  int64_t replicas_total;
  int64_t replicas_dropped;
  double sample_mse;   /* held-out sample MSE (pipeline.cpp:561-570) */
  double block_fit;    /* relative error of the sampled-block ALS */
  int64_t als_sweeps;  /* ALS sweeps over all replicas and restarts */
} xtsg_pipeline_metrics;

/* decompose (pipeline.cpp:245-573): source = a column-major tensor (host or
 * device fp64) or, when tensor is NULL, a factor triple of factor_rank
 * columns (compressed from device-generated slabs on the bf16 path, by
 * comp_from_factors on the fp64 path). Recovered factors: dims[m] x rank.
 * Stage failures return XTSG_E_STAGE (payload 0 = stage index, payload 1 =
 * the inner status). */
int32_t xtsg_decompose(const xtsg_pipeline_config* cfg, const int64_t dims[3], const double* tensor,
                       const double* fa, const double* fb, const double* fc, int64_t factor_rank,
                       double* a_out, double* b_out, double* c_out, xtsg_pipeline_metrics* metrics);

/* Stages 1-3 of decompose on replicas compressed by the caller (e.g. a
 * mode-3-sharded multi-GPU compression reduced to this rank): count replicas
 * L x M x N back to back, f32 or f64, host or device. The source is needed
 * only for the sampled and held-out blocks. */
int32_t xtsg_decompose_replicas(const xtsg_pipeline_config* cfg, const int64_t dims[3],
                                const void* replicas, int32_t replicas_dtype, const double* tensor,
                                const double* fa, const double* fb, const double* fc,
                                int64_t factor_rank, double* a_out, double* b_out, double* c_out,
                                xtsg_pipeline_metrics* metrics);

/* decompose split at the stage-1 boundary, for multi-GPU pipelines that
 * spread the per-replica CP-ALS over ranks (SURVEY §8 e).
 * stage1: stage 1 (pipeline.cpp:410-446) for n replicas (L x M x N back to
 * back, f32/f64, host or device) whose global indices are ids[n] (restart
 * seeds derive(derive(cfg.seed, 500 + id), attempt)); per replica: the best
 * attempt's factors (per_f = (L + M + N) * rank doubles: A, then B, then C,
 * column-major), its relative fit error, its convergence flag and the sweeps
 * of every attempt the reference's sequential restart loop runs.
 * finish: stages 1 (survivor rule) - 3 on those results for all `replicas`
 * replicas in index order; identical output to xtsg_decompose_replicas. */
int32_t xtsg_decompose_stage1(const xtsg_pipeline_config* cfg, const int64_t dims[3], int64_t n,
                              const int64_t* ids, const void* replicas, int32_t replicas_dtype,
                              double* factors, double* fit_err, int32_t* converged, int64_t* sweeps);
int32_t xtsg_decompose_finish(const xtsg_pipeline_config* cfg, const int64_t dims[3], const double* factors,
                              const double* fit_err, const int32_t* converged, const int64_t* sweeps,
                              const double* tensor, const double* fa, const double* fb, const double* fc,
                              int64_t factor_rank, double* a_out, double* b_out, double* c_out,
                              xtsg_pipeline_metrics* metrics);

/* evaluate (pipeline.cpp:577-609): joint permutation/scale against the truth,
 * per-mode relative errors, leading-corner sample MSE. aligned_* optional. */
int32_t xtsg_evaluate(const int64_t dims[3], int64_t rank, const double* ta, const double* tb,
                      const double* tc, const double* ra, const double* rb, const double* rc,
                      int64_t sample, double mode_rel_err[3], double* sample_mse,
                      double* aligned_a, double* aligned_b, double* aligned_c);

#ifdef __cplusplus
}
#endif
#endif /* XTSG_H_ */
