// TEST INFRASTRUCTURE ONLY (oracle build). Not part of the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/ref_build/Makefile) so that the Python
// tests, golden-vector generator and bench.py's CPU-baseline leg can call the
// reference implementation through ctypes. Every function forwards to the
// reference entry point named in its comment; exceptions are mapped to the
// same status codes the product C ABI uses (include/xtsg.h).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "xts/alignment.hpp"
#include "xts/compression.hpp"
#include "xts/cp_als.hpp"
#include "xts/errors.hpp"
#include "xts/linalg.hpp"
#include "xts/io.hpp"
#include "xts/mixed.hpp"
#include "xts/half.hpp"
#include "xts/pipeline.hpp"
#include "xts/rng.hpp"

extern "C" void scipy_openblas_set_num_threads64_(int);

using namespace xts;

namespace {

thread_local int64_t g_payload = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError&) {
    return 1;
  } catch (const DataError&) {
    return 2;
  } catch (const IllPosedError& e) {
    g_payload = e.effective_rank;
    return 3;
  } catch (const DegenerateColumnError& e) {
    g_payload = e.column;
    return 4;
  } catch (const InsufficientReplicasError& e) {
    g_payload = e.survivors;
    return 5;
  } catch (const HalfRangeError&) {
    return 6;
  } catch (const StageError&) {
    return 7;
  } catch (...) {
    return 99;
  }
}

Matrix mat(const double* p, int64_t r, int64_t c) {
  Matrix m(r, c);
  if (r * c != 0) std::memcpy(m.values.data(), p, sizeof(double) * r * c);
  return m;
}
Tensor3 ten(const double* p, int64_t a, int64_t b, int64_t c) {
  Tensor3 t(a, b, c);
  if (a * b * c != 0) std::memcpy(t.values.data(), p, sizeof(double) * a * b * c);
  return t;
}
void put(double* dst, const std::vector<double>& v) {
  if (!v.empty()) std::memcpy(dst, v.data(), sizeof(double) * v.size());
}

}  // namespace

extern "C" {

int64_t xref_last_payload() { return g_payload; }
void xref_set_blas_threads(int n) { scipy_openblas_set_num_threads64_(n); }

// rng.hpp:15-20 / :23 / :26-41 / :46-50
void xref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void xref_rng_normal(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}
uint64_t xref_derive(uint64_t seed, uint64_t tag) { return Rng::derive(seed, tag); }
double xref_log(double x) { return std::log(x); }
void xref_log_many(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = std::log(x[i]);
}

// compression.cpp:82-95
int xref_replica_count(const int64_t* dims, const int64_t* red, int64_t slack, int64_t* out) {
  return guard([&] {
    *out = compute_replica_count({dims[0], dims[1], dims[2]}, {red[0], red[1], red[2]}, slack);
  });
}

// compression.cpp:97-113
int xref_gen_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] { put(out, gen_gaussian(rows, cols, seed).values); });
}
int xref_gen_sparse_projection(int64_t rows, int64_t cols, double s, uint64_t seed,
                               double* out) {
  return guard([&] {
    SparseProjectionSpec sp;
    sp.s = s;
    put(out, gen_sparse_projection(rows, cols, sp, seed).values);
  });
}

// compression.cpp:115-200. kind: 0 gaussian, 1 sparse, 2 two_stage.
// Outputs are the P materialized matrices back to back (u: P x L x I, ...).
// For two-stage, inner_{u,v,w} receive the inner matrices and outer_{u,v,w}
// the P outer matrices (may be null otherwise).
int xref_make_ensemble(const int64_t* dims, const int64_t* red, int64_t count,
                       int64_t shared, int kind, double s, double alpha, double beta,
                       double gamma, int inner_kind, double inner_s, uint64_t seed,
                       double* u, double* v, double* w, double* inner_u, double* inner_v,
                       double* inner_w, double* outer_u, double* outer_v, double* outer_w) {
  return guard([&] {
    EnsembleSpec spec;
    spec.kind = kind == 0 ? EnsembleSpec::Kind::gaussian
                          : kind == 1 ? EnsembleSpec::Kind::sparse
                                      : EnsembleSpec::Kind::two_stage;
    spec.sparse.s = s;
    spec.two_stage.alpha = alpha;
    spec.two_stage.beta = beta;
    spec.two_stage.gamma = gamma;
    spec.two_stage.inner_kind = inner_kind == 0 ? ProjectionKind::gaussian : ProjectionKind::sparse;
    spec.two_stage.inner_spec.s = inner_s;
    const auto ens = make_ensemble({dims[0], dims[1], dims[2]}, {red[0], red[1], red[2]},
                                   count, shared, spec, seed);
    for (int64_t p = 0; p < count; ++p) {
      put(u + p * red[0] * dims[0], ens.u[p].values);
      put(v + p * red[1] * dims[1], ens.v[p].values);
      put(w + p * red[2] * dims[2], ens.w[p].values);
    }
    if (ens.two_stage && inner_u) {
      const auto& ts = *ens.two_stage;
      put(inner_u, ts.u_inner.values);
      put(inner_v, ts.v_inner.values);
      put(inner_w, ts.w_inner.values);
      for (int64_t p = 0; p < count; ++p) {
        put(outer_u + p * ts.u_outer[p].size(), ts.u_outer[p].values);
        put(outer_v + p * ts.v_outer[p].size(), ts.v_outer[p].values);
        put(outer_w + p * ts.w_outer[p].size(), ts.w_outer[p].values);
      }
    }
  });
}

// compression.cpp:211-213
int xref_comp(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
              int64_t l, const double* v, int64_t m, const double* w, int64_t n, double* y) {
  return guard([&] {
    put(y, comp(ten(t, n1, n2, n3), mat(u, l, n1), mat(v, m, n2), mat(w, n, n3)).values);
  });
}

// mixed.cpp:90-98 (Eq. 5) on the full-residual split
int xref_comp_mixed(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u,
                    int64_t l, const double* v, int64_t m, const double* w, int64_t n,
                    int stored_residual, double* y) {
  return guard([&] {
    const bool st = stored_residual != 0;
    put(y, comp_mixed(split_tensor(ten(t, n1, n2, n3), st), split_matrix(mat(u, l, n1), st),
                      split_matrix(mat(v, m, n2), st), split_matrix(mat(w, n, n3), st))
               .values);
  });
}

// compression.cpp:215-220
int xref_comp_from_factors(const double* a, const double* b, const double* c, int64_t i,
                           int64_t j, int64_t k, int64_t r, const double* u, int64_t l,
                           const double* v, int64_t m, const double* w, int64_t n,
                           double* y) {
  return guard([&] {
    const FactorTriple f(mat(a, i, r), mat(b, j, r), mat(c, k, r));
    put(y, comp_from_factors(f, mat(u, l, i), mat(v, m, j), mat(w, n, k)).values);
  });
}

// tensor.cpp:133-150
int xref_reconstruct(const double* a, const double* b, const double* c, int64_t i, int64_t j,
                     int64_t k, int64_t r, double* out) {
  return guard([&] {
    put(out, reconstruct(FactorTriple(mat(a, i, r), mat(b, j, r), mat(c, k, r))).values);
  });
}

// compression.cpp:332-404 fed by make_memory_block_source (:254-278)
int xref_comp_blocked(const double* t, const int64_t* dims, const int64_t* block,
                      int64_t count, const int64_t* red, const double* u, const double* v,
                      const double* w, int deterministic, int workers, double* y) {
  return guard([&] {
    const Tensor3 tt = ten(t, dims[0], dims[1], dims[2]);
    CompressionEnsemble ens;
    ens.count = count;
    for (int64_t p = 0; p < count; ++p) {
      ens.u.push_back(mat(u + p * red[0] * dims[0], red[0], dims[0]));
      ens.v.push_back(mat(v + p * red[1] * dims[1], red[1], dims[1]));
      ens.w.push_back(mat(w + p * red[2] * dims[2], red[2], dims[2]));
    }
    const BlockGrid grid({dims[0], dims[1], dims[2]}, {block[0], block[1], block[2]});
    const auto reps = comp_blocked(grid, make_memory_block_source(tt, grid), ens,
                                   deterministic != 0, workers);
    const int64_t sz = red[0] * red[1] * red[2];
    for (int64_t p = 0; p < count; ++p) put(y + p * sz, reps[p].values);
  });
}

// cp_als.cpp:46-111. init: 0 normal, 1 nvecs. hist must hold max_iters doubles.
int xref_cp_als(const double* t, int64_t n1, int64_t n2, int64_t n3, int64_t rank,
                int64_t max_iters, double tol, uint64_t seed, int init, double* a, double* b,
                double* c, int64_t* iters, int* converged, double* hist) {
  return guard([&] {
    AlsConfig cfg;
    cfg.rank = rank;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.seed = seed;
    cfg.init = init ? AlsConfig::Init::nvecs : AlsConfig::Init::normal;
    const AlsResult r = cp_als(ten(t, n1, n2, n3), cfg);
    put(a, r.factors.a.values);
    put(b, r.factors.b.values);
    put(c, r.factors.c.values);
    *iters = r.iters;
    *converged = r.converged ? 1 : 0;
    put(hist, r.error_history);
  });
}

// cp_als.cpp:22-44
int xref_relative_error(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* a,
                        const double* b, const double* c, int64_t r, double* out) {
  return guard([&] {
    *out = relative_error(ten(t, n1, n2, n3),
                          FactorTriple(mat(a, n1, r), mat(b, n2, r), mat(c, n3, r)));
  });
}

// alignment.cpp:220-252. Blocks stacked back to back: f_p is rows[p] x r,
// u_p is rows[p] x cols.
int xref_solve_stacked_ls(int64_t count, const int64_t* rows, int64_t r, int64_t cols,
                          const double* f, const double* u, double* x) {
  return guard([&] {
    std::vector<Matrix> fs, us;
    int64_t fo = 0, uo = 0;
    for (int64_t p = 0; p < count; ++p) {
      fs.push_back(mat(f + fo, rows[p], r));
      us.push_back(mat(u + uo, rows[p], cols));
      fo += rows[p] * r;
      uo += rows[p] * cols;
    }
    put(x, solve_stacked_ls(fs, us).values);
  });
}

// alignment.cpp:87-144
int xref_max_trace_assignment(const double* obj, int64_t n, int64_t* perm) {
  return guard([&] {
    const auto p = max_trace_assignment(mat(obj, n, n));
    for (int64_t i = 0; i < n; ++i) perm[i] = p[i];
  });
}

// alignment.cpp:66-85
int xref_normalize_shared(const double* m, int64_t rows, int64_t cols, int64_t shared,
                          double* normalized, double* pivots) {
  return guard([&] {
    const auto r = normalize_shared(mat(m, rows, cols), shared);
    put(normalized, r.normalized.values);
    put(pivots, r.pivots);
  });
}

// alignment.cpp:154-218. factors: P triples back to back (a: rows[0] x r, ...).
// aligned receives the surviving triples back to back; dropped[p] flags.
int xref_align_replicas(int64_t count, const int64_t* dims, int64_t r, const double* factors,
                        int64_t shared, int64_t min_survivors, double* aligned,
                        int* dropped, int64_t* survivors, int64_t* n_survivors) {
  return guard([&] {
    std::vector<FactorTriple> fs;
    const int64_t per = (dims[0] + dims[1] + dims[2]) * r;
    for (int64_t p = 0; p < count; ++p) {
      const double* base = factors + p * per;
      fs.push_back(FactorTriple(mat(base, dims[0], r), mat(base + dims[0] * r, dims[1], r),
                                mat(base + (dims[0] + dims[1]) * r, dims[2], r)));
    }
    const auto res = align_replicas(fs, shared, min_survivors);
    for (int64_t p = 0; p < count; ++p) dropped[p] = res.dropped[p] ? 1 : 0;
    *n_survivors = static_cast<int64_t>(res.survivors.size());
    for (std::size_t i = 0; i < res.survivors.size(); ++i) {
      survivors[i] = res.survivors[i];
      double* base = aligned + static_cast<int64_t>(i) * per;
      put(base, res.aligned[i].a.values);
      put(base + dims[0] * r, res.aligned[i].b.values);
      put(base + (dims[0] + dims[1]) * r, res.aligned[i].c.values);
    }
  });
}

// alignment.cpp:254-278
int xref_recover_perm_scale(const double* head, const double* sampled, int64_t rows,
                            int64_t cols, int64_t* perm, double* scale) {
  return guard([&] {
    const auto ps = recover_perm_scale(mat(head, rows, cols), mat(sampled, rows, cols));
    for (int64_t i = 0; i < cols; ++i) {
      perm[i] = ps.perm[i];
      scale[i] = ps.scale[i];
    }
  });
}

// pipeline.cpp:182-220 (factors only). law: 0 dense, 1 sparse.
int xref_generate(const int64_t* dims, int64_t rank, int law, int64_t nnz_per_col,
                  uint64_t seed, double* a, double* b, double* c) {
  return guard([&] {
    SyntheticSpec spec;
    spec.dims = {dims[0], dims[1], dims[2]};
    spec.rank = rank;
    spec.law = law ? SyntheticSpec::Law::sparse : SyntheticSpec::Law::dense;
    spec.nnz_per_col = nnz_per_col;
    spec.seed = seed;
    const Synthetic s = generate(spec, false);
    put(a, s.factors.a.values);
    put(b, s.factors.b.values);
    put(c, s.factors.c.values);
  });
}

// pipeline.cpp:242-575 + evaluate :577-609. Source is the factor triple
// (factored) or, when tensor != null, the materialized tensor.
// cfg_i: [reduced0, reduced1, reduced2, rank, replicas, slack, shared,
//         block0, block1, block2, mode, omp_sparsity, sample_b, precision,
//         deterministic, als_max_iters, als_restarts, workers]
// cfg_d: [alpha, beta, gamma, projection_s, omp_residual_tol, als_tol,
//         replica_fit_tol]
// stats: [t_comp, t_decomp, t_align, t_recov, replicas_total, replicas_dropped,
//         sample_mse, err_a, err_b, err_c, eval_mse]
int xref_decompose(const double* a, const double* b, const double* c, const int64_t* dims,
                   int64_t true_rank, const double* tensor, const int64_t* cfg_i,
                   const double* cfg_d, uint64_t seed, double* out_a, double* out_b,
                   double* out_c, double* stats) {
  return guard([&] {
    const FactorTriple truth(mat(a, dims[0], true_rank), mat(b, dims[1], true_rank),
                             mat(c, dims[2], true_rank));
    Tensor3 t;
    if (tensor) t = ten(tensor, dims[0], dims[1], dims[2]);
    PipelineConfig cfg;
    cfg.dims = {dims[0], dims[1], dims[2]};
    cfg.reduced = {cfg_i[0], cfg_i[1], cfg_i[2]};
    cfg.rank = cfg_i[3];
    cfg.replicas = cfg_i[4];
    cfg.slack = cfg_i[5];
    cfg.shared = cfg_i[6];
    cfg.block = {cfg_i[7], cfg_i[8], cfg_i[9]};
    cfg.mode = cfg_i[10] == 0   ? PipelineConfig::Mode::dense
               : cfg_i[10] == 1 ? PipelineConfig::Mode::sparse
                                : PipelineConfig::Mode::two_stage;
    cfg.omp_sparsity = cfg_i[11];
    cfg.sample_b = cfg_i[12];
    cfg.precision = cfg_i[13] ? PipelineConfig::Precision::mixed : PipelineConfig::Precision::full;
    cfg.deterministic = cfg_i[14] != 0;
    cfg.als_max_iters = cfg_i[15];
    cfg.als_restarts = cfg_i[16];
    cfg.workers = static_cast<int>(cfg_i[17]);
    cfg.alpha = cfg_d[0];
    cfg.beta = cfg_d[1];
    cfg.gamma = cfg_d[2];
    cfg.projection_s = cfg_d[3];
    cfg.omp_residual_tol = cfg_d[4];
    cfg.als_tol = cfg_d[5];
    cfg.replica_fit_tol = cfg_d[6];
    cfg.seed = seed;
    RunMetrics metrics;
    const TensorSource src = tensor ? TensorSource::from_tensor(t) : TensorSource::from_factors(truth);
    FactorTriple rec;
    try {
      rec = decompose(src, cfg, metrics);
    } catch (...) {
      for (int s = 0; s < 4; ++s) stats[s] = metrics.stages[s].elapsed_s;
      throw;
    }
    put(out_a, rec.a.values);
    put(out_b, rec.b.values);
    put(out_c, rec.c.values);
    for (int s = 0; s < 4; ++s) stats[s] = metrics.stages[s].elapsed_s;
    stats[4] = static_cast<double>(metrics.replicas_total);
    stats[5] = static_cast<double>(metrics.replicas_dropped);
    stats[6] = metrics.sample_mse;
    const EvalReport ev = evaluate(truth, rec);
    stats[7] = ev.mode_rel_err[0];
    stats[8] = ev.mode_rel_err[1];
    stats[9] = ev.mode_rel_err[2];
    stats[10] = ev.sample_mse;
  });
}

// pipeline.cpp:577-609
int xref_evaluate(const int64_t* dims, int64_t r, const double* ta, const double* tb,
                  const double* tc, const double* ra, const double* rb, const double* rc,
                  double* out4) {
  return guard([&] {
    const FactorTriple truth(mat(ta, dims[0], r), mat(tb, dims[1], r), mat(tc, dims[2], r));
    const FactorTriple rec(mat(ra, dims[0], r), mat(rb, dims[1], r), mat(rc, dims[2], r));
    const EvalReport ev = evaluate(truth, rec);
    out4[0] = ev.mode_rel_err[0];
    out4[1] = ev.mode_rel_err[1];
    out4[2] = ev.mode_rel_err[2];
    out4[3] = ev.sample_mse;
  });
}

// half.cpp:10-47
int xref_double_to_half_bits(double x, uint16_t* out) {
  return guard([&] { *out = double_to_half_bits(x); });
}

// mixed.cpp:47-61 (mode 0) and split_tensor (mode 1 full, 2 stored residual)
int xref_split(const double* x, int64_t n, int mode, double* half, double* res) {
  return guard([&] {
    const Tensor3 t = ten(x, n, 1, 1);
    if (mode == 0) {
      put(half, round_tensor_to_half(t).values);
    } else {
      const SplitTensor3 s = split_tensor(t, mode == 2);
      put(half, s.half.values);
      put(res, s.residual.values);
    }
  });
}

// mixed.cpp:63-76
int xref_half_gemm(const double* a, int64_t rows, int64_t inner, const double* b, int64_t cols, double* out) {
  return guard([&] { put(out, half_gemm(mat(a, rows, inner), mat(b, inner, cols)).values); });
}

// comp_with(..., &half_gemm) (compression.cpp:202-209)
int xref_comp_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                   const double* v, int64_t m, const double* w, int64_t n, double* y) {
  return guard([&] {
    put(y, comp_with(ten(t, n1, n2, n3), mat(u, l, n1), mat(v, m, n2), mat(w, n, n3), &half_gemm).values);
  });
}

// mixed.cpp:100-104
int xref_comp_naive_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                         const double* v, int64_t m, const double* w, int64_t n, double* y) {
  return guard([&] {
    put(y, comp_naive_half(ten(t, n1, n2, n3), mat(u, l, n1), mat(v, m, n2), mat(w, n, n3)).values);
  });
}

// io.cpp:55-89 (fixtures for the out-of-core source tests)
int xref_write_tensor_file(const char* path, const double* t, int64_t n1, int64_t n2, int64_t n3) {
  return guard([&] { write_tensor_file(path, ten(t, n1, n2, n3)); });
}

int xref_write_factor_file(const char* path, const double* a, const double* b, const double* c, int64_t i,
                           int64_t j, int64_t k, int64_t r) {
  return guard([&] { write_factor_file(path, FactorTriple(mat(a, i, r), mat(b, j, r), mat(c, k, r))); });
}

}  // extern "C"
