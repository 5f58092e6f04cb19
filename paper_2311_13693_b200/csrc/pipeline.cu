// End-to-end decomposition on the device: the reference's decompose()
// (/root/reference/proj/src/pipeline.cpp:245-573) re-planned around the
// device-resident pieces of this library, plus generate() (:157-220) and
// evaluate() (:577-609).
//
// Stage structure, seeds, defaults, survivor rules and error mapping follow
// the reference line by line (cited below); what changes is where the data
// lives: the ensemble is generated on the device and never leaves it, the
// compression is one Plan (tcgen05 TTM for XTSG_PREC_BF16, fp64 DFMA chains
// for XTSG_PREC_FP64), all replicas' CP-ALS runs as one batched launch per
// restart round, and the stacked least squares runs on the device-resident
// ensemble. Only R-column factor matrices and the b^3 sampled blocks touch
// the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "xrng.cuh"

namespace xtsg {

namespace {

using Clock = std::chrono::steady_clock;

// Re-raise the status of an inner C-ABI call as an exception.
void ck(int32_t rc) {
  if (rc != XTSG_OK) {
    const ErrState e = err_state();
    throw Status(rc, e.msg, e.p0, e.p1);
  }
}

// ---- host helpers (pipeline.cpp:28-128) -----------------------------------

std::vector<int64_t> leading_rows(int64_t count) {
  std::vector<int64_t> out(static_cast<size_t>(std::max<int64_t>(count, 0)));
  std::iota(out.begin(), out.end(), int64_t{0});
  return out;
}

// random_rows (pipeline.cpp:98-111): partial Fisher-Yates, then sorted.
std::vector<int64_t> random_rows(int64_t dim, int64_t count, uint64_t seed) {
  count = std::min(count, dim);
  std::vector<int64_t> idx(static_cast<size_t>(dim));
  std::iota(idx.begin(), idx.end(), int64_t{0});
  HostRng rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    const int64_t j = i + static_cast<int64_t>(rng.next() % static_cast<uint64_t>(dim - i));
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(j)]);
  }
  idx.resize(static_cast<size_t>(count));
  std::sort(idx.begin(), idx.end());
  return idx;
}

// select_rows_by_mass (pipeline.cpp:63-96): round-robin over columns, each
// column's rows by descending |value| (lower row index on ties).
std::vector<int64_t> select_rows_by_mass(const std::vector<double>& est, int64_t rows, int64_t cols,
                                         int64_t count) {
  count = std::min(count, rows);
  std::vector<std::vector<int64_t>> order(static_cast<size_t>(cols));
  for (int64_t j = 0; j < cols; ++j) {
    auto& o = order[static_cast<size_t>(j)];
    o.resize(static_cast<size_t>(rows));
    std::iota(o.begin(), o.end(), int64_t{0});
    const double* c = est.data() + rows * j;
    std::sort(o.begin(), o.end(), [&](int64_t x, int64_t y) {
      const double ax = std::fabs(c[x]), ay = std::fabs(c[y]);
      return ax != ay ? ax > ay : x < y;
    });
  }
  std::vector<char> chosen(static_cast<size_t>(rows), 0);
  std::vector<size_t> cursor(static_cast<size_t>(cols), 0);
  std::vector<int64_t> out;
  while (static_cast<int64_t>(out.size()) < count) {
    bool progressed = false;
    for (int64_t j = 0; j < cols && static_cast<int64_t>(out.size()) < count; ++j) {
      auto& cur = cursor[static_cast<size_t>(j)];
      const auto& o = order[static_cast<size_t>(j)];
      while (cur < o.size() && chosen[static_cast<size_t>(o[cur])]) ++cur;
      if (cur < o.size()) {
        chosen[static_cast<size_t>(o[cur])] = 1;
        out.push_back(o[cur]);
        progressed = true;
      }
    }
    if (!progressed) break;
  }
  std::sort(out.begin(), out.end());
  return out;
}

std::vector<double> gather_rows(const std::vector<double>& m, int64_t rows, int64_t cols,
                                const std::vector<int64_t>& sel) {
  std::vector<double> out(sel.size() * static_cast<size_t>(cols));
  for (int64_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < sel.size(); ++i) out[i + sel.size() * j] = m[sel[i] + rows * j];
  return out;
}

// reconstruct (tensor.cpp:133-150) of row-gathered factors (reconstruct_rows,
// pipeline.cpp:46-52): sequential over r, slab[i] += a[i,r] * (b[j,r] c[k,r]).
std::vector<double> reconstruct_rows(const std::vector<double>* f, const int64_t* rows, int64_t R,
                                     const std::vector<int64_t>* sel) {
  const int64_t n1 = static_cast<int64_t>(sel[0].size()), n2 = static_cast<int64_t>(sel[1].size()),
                n3 = static_cast<int64_t>(sel[2].size());
  std::vector<double> t(static_cast<size_t>(n1 * n2 * n3), 0.0);
  for (int64_t r = 0; r < R; ++r) {
    const double* ca = f[0].data() + rows[0] * r;
    const double* cb = f[1].data() + rows[1] * r;
    const double* cc = f[2].data() + rows[2] * r;
    for (int64_t k = 0; k < n3; ++k)
      for (int64_t j = 0; j < n2; ++j) {
        const double s = cb[sel[1][j]] * cc[sel[2][k]];
        double* slab = t.data() + n1 * (j + n2 * k);
        for (int64_t i = 0; i < n1; ++i) slab[i] += ca[sel[0][i]] * s;
      }
  }
  return t;
}

// device side of gather_block: out[i + n1*(j + n2*k)] = t[si[i] + d0*(sj[j] + d1*sk[k])]
__global__ void gather_block_kernel(const double* __restrict__ t, int64_t d0, int64_t d1,
                                    const int64_t* __restrict__ sel, int64_t n1, int64_t n2, int64_t n3,
                                    double* __restrict__ out) {
  const int64_t total = n1 * n2 * n3;
  const int64_t *si = sel, *sj = sel + n1, *sk = sel + n1 + n2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % n1, jk = e / n1, j = jk % n2, k = jk / n2;
    out[e] = t[si[i] + d0 * (sj[j] + d1 * sk[k])];
  }
}

// gather_block (pipeline.cpp:36-44) from a host or device column-major tensor
// (device tensors: one gather kernel and one D2H copy of the block).
std::vector<double> gather_block(const double* t, const int64_t* dims, const std::vector<int64_t>* sel,
                                 cudaStream_t st) {
  const size_t n1 = sel[0].size(), n2 = sel[1].size(), n3 = sel[2].size();
  std::vector<double> out(n1 * n2 * n3);
  if (out.empty()) return out;
  if (is_device_ptr(t)) {
    std::vector<int64_t> idx;
    idx.reserve(n1 + n2 + n3);
    for (int m = 0; m < 3; ++m) idx.insert(idx.end(), sel[m].begin(), sel[m].end());
    DevBuf<int64_t> dsel(idx.size(), st);
    DevBuf<double> dout(out.size(), st);
    XCUDA(cudaMemcpyAsync(dsel.ptr, idx.data(), idx.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const int64_t total = static_cast<int64_t>(out.size());
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    gather_block_kernel<<<grid, 256, 0, st>>>(t, dims[0], dims[1], dsel.ptr, static_cast<int64_t>(n1),
                                              static_cast<int64_t>(n2), static_cast<int64_t>(n3), dout.ptr);
    XLAUNCH_CHECK();
    XCUDA(cudaMemcpyAsync(out.data(), dout.ptr, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    XCUDA(cudaStreamSynchronize(st));
    return out;
  }
  for (size_t k = 0; k < n3; ++k)
    for (size_t j = 0; j < n2; ++j)
      for (size_t i = 0; i < n1; ++i)
        out[i + n1 * (j + n2 * k)] = t[sel[0][i] + dims[0] * (sel[1][j] + dims[1] * sel[2][k])];
  return out;
}

double mse(const std::vector<double>& x, const std::vector<double>& y) {
  if (x.empty()) return 0.0;
  double acc = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    const double d = x[i] - y[i];
    acc += d * d;
  }
  return acc / static_cast<double>(x.size());
}

// host copy of a host or device buffer (host-only callers need no device)
void copy_in(std::vector<double>& dst, const double* src) {
  if (is_device_ptr(src))
    XCUDA(cudaMemcpy(dst.data(), src, sizeof(double) * dst.size(), cudaMemcpyDeviceToHost));
  else
    std::copy(src, src + dst.size(), dst.begin());
}

struct PermScale {
  std::vector<int64_t> perm;
  std::vector<double> scale;
};

// match_factor_triples (pipeline.cpp:130-155): one joint assignment fed by all
// three modes' normalized Gram blocks, per-mode pivot-ratio scales.
void match_factor_triples(const std::vector<double>* global, const std::vector<double>* sampled, const int64_t* rows,
                          int64_t R, PermScale* ps) {
  std::vector<double> gn[3], gp[3], sn[3], sp[3];
  for (int m = 0; m < 3; ++m) {
    gn[m].resize(global[m].size()); gp[m].resize(static_cast<size_t>(R));
    sn[m].resize(sampled[m].size()); sp[m].resize(static_cast<size_t>(R));
    ck(xtsg_normalize_shared(global[m].data(), rows[m], R, rows[m], gn[m].data(), gp[m].data()));
    ck(xtsg_normalize_shared(sampled[m].data(), rows[m], R, rows[m], sn[m].data(), sp[m].data()));
  }
  std::vector<double> obj(static_cast<size_t>(R * R), 0.0);  // sum_m s_m^T g_m
  for (int m = 0; m < 3; ++m)
    for (int64_t j = 0; j < R; ++j)
      for (int64_t i = 0; i < R; ++i) {
        double acc = 0.0;
        for (int64_t q = 0; q < rows[m]; ++q) acc += sn[m][q + rows[m] * i] * gn[m][q + rows[m] * j];
        obj[i + R * j] += acc;
      }
  std::vector<int64_t> perm(static_cast<size_t>(R));
  ck(xtsg_max_trace_assignment(obj.data(), R, perm.data()));
  for (int m = 0; m < 3; ++m) {
    ps[m].perm = perm;
    ps[m].scale.resize(static_cast<size_t>(R));
    for (int64_t r = 0; r < R; ++r) ps[m].scale[r] = sp[m][r] / gp[m][perm[r]];
  }
}

// apply_forward (alignment.cpp:280-291): column r = m[:, perm[r]] * scale[r].
std::vector<double> apply_forward(const std::vector<double>& m, int64_t rows, const PermScale& ps) {
  const int64_t R = static_cast<int64_t>(ps.perm.size());
  std::vector<double> out(static_cast<size_t>(rows * R));
  for (int64_t r = 0; r < R; ++r)
    for (int64_t i = 0; i < rows; ++i) out[i + rows * r] = m[i + rows * ps.perm[r]] * ps.scale[r];
  return out;
}

__global__ void widen_kernel(const float* __restrict__ s, int64_t n, double* __restrict__ d) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[e] = static_cast<double>(s[e]);
}

// ---- configuration resolution (pipeline.cpp:253-326) ----------------------

struct Resolved {
  int64_t dims[3], reduced[3], rank, replicas, shared, sample_b, min_survivors;
  bool sparse, two_stage;
  xtsg_ensemble_spec spec;
  uint64_t ensemble_seed;
};

Resolved resolve(const xtsg_pipeline_config& cfg, const int64_t dims[3]) {
  Resolved r{};
  for (int m = 0; m < 3; ++m) {
    r.dims[m] = dims[m];
    r.reduced[m] = cfg.reduced[m];
    if (dims[m] < 1) usage("decompose: dims must be >= 1");
    if (cfg.reduced[m] < 1 || cfg.reduced[m] > dims[m]) usage("decompose: reduced dims must lie in [1, dims]");
  }
  r.rank = cfg.rank;
  if (r.rank < 1) usage("decompose: rank must be >= 1");
  if (cfg.mode < XTSG_MODE_DENSE || cfg.mode > XTSG_MODE_TWO_STAGE) usage("decompose: unknown mode");
  r.sparse = cfg.mode == XTSG_MODE_SPARSE;
  r.two_stage = cfg.mode == XTSG_MODE_TWO_STAGE;
  if ((r.sparse || r.two_stage) && cfg.omp_sparsity < 1)
    usage("decompose: sparse and two-stage modes need omp_sparsity >= 1");
  const int64_t min_reduced = std::min({r.reduced[0], r.reduced[1], r.reduced[2]});
  r.replicas = cfg.replicas;
  if (r.replicas < 1) {
    if (min_reduced < 3)
      usage("decompose: auto replica count needs reduced dims >= 3; pass an explicit replica count");
    ck(xtsg_replica_count(r.dims, r.reduced, cfg.slack, &r.replicas));
  }
  r.shared = cfg.shared;
  if (r.shared > 0 && r.shared > min_reduced) usage("decompose: shared anchor exceeds the reduced dims");
  if (r.shared < 1) r.shared = std::min<int64_t>(2 * r.rank, min_reduced);
  int64_t sb = cfg.sample_b;
  if (sb < 1) {
    sb = std::max<int64_t>(2 * r.rank, 8);
    if (r.sparse || r.two_stage) sb = std::max(sb, cfg.omp_sparsity * r.rank);
  }
  r.sample_b = std::min({sb, r.dims[0], r.dims[1], r.dims[2]});
  r.min_survivors = 1;
  if (min_reduced >= 3) {
    int64_t bound = 0;
    ck(xtsg_replica_count(r.dims, r.reduced, 0, &bound));
    if (r.two_stage)
      r.min_survivors = std::min<int64_t>(
          r.replicas, static_cast<int64_t>(std::ceil(std::max({cfg.alpha, cfg.beta, cfg.gamma}))));
    else if (r.sparse)
      r.min_survivors = r.replicas >= bound ? bound : 1;
    else
      r.min_survivors = bound;
  }
  // ensemble spec (pipeline.cpp:355-378)
  const double ratio_min = std::min({static_cast<double>(r.dims[0]) / static_cast<double>(r.reduced[0]),
                                     static_cast<double>(r.dims[1]) / static_cast<double>(r.reduced[1]),
                                     static_cast<double>(r.dims[2]) / static_cast<double>(r.reduced[2])});
  r.spec = xtsg_ensemble_spec{};
  r.spec.kind = XTSG_KIND_GAUSSIAN;
  r.spec.inner_kind = XTSG_KIND_SPARSE;
  r.spec.s = 1.0;
  r.spec.alpha = cfg.alpha; r.spec.beta = cfg.beta; r.spec.gamma = cfg.gamma;
  r.spec.inner_s = 1.0;
  if (r.sparse) {
    r.spec.kind = XTSG_KIND_SPARSE;
    r.spec.s = cfg.projection_s > 0.0 ? cfg.projection_s : std::max(1.0, ratio_min);
  } else if (r.two_stage) {
    r.spec.kind = XTSG_KIND_TWO_STAGE;
    const double inner_ratio =
        std::min({static_cast<double>(r.dims[0]) / (cfg.alpha * static_cast<double>(r.reduced[0])),
                  static_cast<double>(r.dims[1]) / (cfg.beta * static_cast<double>(r.reduced[1])),
                  static_cast<double>(r.dims[2]) / (cfg.gamma * static_cast<double>(r.reduced[2]))});
    r.spec.inner_s = cfg.projection_s > 0.0 ? cfg.projection_s : std::max(1.0, inner_ratio);
  }
  r.ensemble_seed = derive(cfg.seed, 11);
  return r;
}

// The ensemble, device-resident, in the reference layout.
struct EnsembleDev {
  DevBuf<double> u[3], inner[3], outer[3];
  int64_t inner_rows[3] = {0, 0, 0};
};

void make_ensemble_dev(const Resolved& r, EnsembleDev& e, cudaStream_t st) {
  double* io[3] = {nullptr, nullptr, nullptr};
  double* oo[3] = {nullptr, nullptr, nullptr};
  const double ratio[3] = {r.spec.alpha, r.spec.beta, r.spec.gamma};
  for (int m = 0; m < 3; ++m) {
    e.u[m] = DevBuf<double>(static_cast<size_t>(r.replicas * r.reduced[m] * r.dims[m]), st);
    if (r.two_stage) {
      e.inner_rows[m] = std::llround(ratio[m] * static_cast<double>(r.reduced[m]));
      e.inner[m] = DevBuf<double>(static_cast<size_t>(e.inner_rows[m] * r.dims[m]), st);
      e.outer[m] = DevBuf<double>(static_cast<size_t>(r.replicas * r.reduced[m] * e.inner_rows[m]), st);
      io[m] = e.inner[m].ptr;
      oo[m] = e.outer[m].ptr;
    }
  }
  ck(xtsg_make_ensemble(r.dims, r.reduced, r.replicas, r.shared, &r.spec, r.ensemble_seed, e.u[0].ptr, e.u[1].ptr,
                        e.u[2].ptr, io[0], io[1], io[2], oo[0], oo[1], oo[2]));
}

struct Source {
  const double* tensor = nullptr;  // column-major dims[0] x dims[1] x dims[2] (host or device)
  std::vector<double> f[3];        // factors (host copies), rows dims[m] x frank
  int64_t frank = 0;
};

Source make_source(const int64_t* dims, const double* tensor, const double* fa, const double* fb, const double* fc,
                   int64_t frank, cudaStream_t st) {
  Source s;
  s.tensor = tensor;
  if (!tensor) {
    if (!fa || !fb || !fc || frank < 1) usage("decompose: neither tensor nor factors set");
    const double* src[3] = {fa, fb, fc};
    for (int m = 0; m < 3; ++m) {
      s.f[m].resize(static_cast<size_t>(dims[m] * frank));
      XCUDA(cudaMemcpyAsync(s.f[m].data(), src[m], sizeof(double) * s.f[m].size(), cudaMemcpyDefault, st));
    }
    XCUDA(cudaStreamSynchronize(st));
    s.frank = frank;
  }
  return s;
}

std::vector<double> source_block(const Source& s, const int64_t* dims, const std::vector<int64_t>* sel,
                                 cudaStream_t st) {
  if (s.tensor) return gather_block(s.tensor, dims, sel, st);
  return reconstruct_rows(s.f, dims, s.frank, sel);
}

template <class F>
void run_stage(xtsg_pipeline_metrics* met, int idx, const char* name, cudaStream_t st, F&& fn) {
  const auto t0 = Clock::now();
  auto done = [&](int32_t status) {
    XCUDA(cudaStreamSynchronize(st));
    if (met) {
      met->stage_seconds[idx] = std::chrono::duration<double>(Clock::now() - t0).count();
      met->stage_status[idx] = status;
    }
  };
  try {
    fn();
  } catch (const Status& e) {
    if (met) {
      met->stage_seconds[idx] = std::chrono::duration<double>(Clock::now() - t0).count();
      met->stage_status[idx] = 2;
    }
    // StageError (pipeline.cpp:346-351): stage index in payload 0, the inner
    // status code in payload 1
    throw Status(XTSG_E_STAGE, std::string("stage '") + name + "' failed: " + e.what(), idx, e.code);
  }
  done(1);
}

// Stage-1 result of one replica: the best attempt's factors (A | B | C,
// column-major) and its fit error / convergence, plus the sweeps of every
// attempt the reference's sequential restart loop would have run.
struct Stage1Out {
  std::vector<double> f;
  double err = 1.0;
  int32_t conv = 0, have = 0;
  int64_t sweeps = 0;
};

// Stage 1 of decompose (pipeline.cpp:410-446) for n replicas with global
// indices ids[q] (seeds derive(cfg.seed, 500 + ids[q])), fp64 on the device
// back to back at Yd. Restart rounds run batched; once the pending replicas'
// remaining attempts fit the SMs they all run in ONE launch (speculatively)
// and the sequential rule is replayed on the results: same factors, errors
// and sweep counts as the reference's per-replica loop.
std::vector<Stage1Out> run_stage1(const xtsg_pipeline_config& cfg, const Resolved& rs, int64_t n_rep,
                                  const int64_t* ids, const double* Yd, cudaStream_t st) {
  const int64_t R = rs.rank;
  const int64_t* red = rs.reduced;
  const int64_t lmn = red[0] * red[1] * red[2];
  const int64_t per_f = (red[0] + red[1] + red[2]) * R;
  if (cfg.als_max_iters < 1) usage("cp_als: max_iters must be >= 1");
  std::vector<Stage1Out> out(static_cast<size_t>(n_rep));
  auto done = [&](int64_t q) {
    const Stage1Out& o = out[static_cast<size_t>(q)];
    return o.have && o.conv && o.err <= cfg.replica_fit_tol;
  };
  DevBuf<double> gather;
  const int64_t last_attempt = std::max<int64_t>(cfg.als_restarts, 0);
  for (int64_t attempt = 0; attempt <= last_attempt; ++attempt) {
    std::vector<int64_t> pend;
    for (int64_t q = 0; q < n_rep; ++q)
      if (!done(q)) pend.push_back(q);
    if (pend.empty()) break;
    const int64_t rounds_left = last_attempt - attempt + 1;
    const bool all_at_once = rounds_left > 1 && static_cast<int64_t>(pend.size()) * rounds_left <= sm_count();
    const int64_t span = all_at_once ? rounds_left : 1;
    std::vector<int64_t> item_q, item_a;
    for (int64_t a = attempt; a < attempt + span; ++a)
      for (int64_t q : pend) {
        item_q.push_back(q);
        item_a.push_back(a);
      }
    const int64_t n = static_cast<int64_t>(item_q.size());
    const double* t = Yd;
    bool identity = n == n_rep;
    for (int64_t k = 0; identity && k < n; ++k) identity = item_q[k] == k;
    if (!identity) {
      if (!gather.ptr || static_cast<int64_t>(gather.n) < n * lmn)
        gather = DevBuf<double>(static_cast<size_t>(std::max(n_rep, n) * lmn), st);
      for (int64_t k = 0; k < n; ++k)
        XCUDA(cudaMemcpyAsync(gather.ptr + k * lmn, Yd + item_q[k] * lmn, sizeof(double) * lmn,
                              cudaMemcpyDeviceToDevice, st));
      t = gather.ptr;
    }
    std::vector<xtsg_als_config> cfgs(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      const uint64_t replica_seed = derive(cfg.seed, 500 + static_cast<uint64_t>(ids[item_q[k]]));
      cfgs[k].rank = R;
      cfgs[k].max_iters = cfg.als_max_iters;
      cfgs[k].tol = cfg.als_tol;
      cfgs[k].seed = derive(replica_seed, static_cast<uint64_t>(item_a[k]));
      cfgs[k].init = item_a[k] == 1 ? 1 : 0;
      cfgs[k].reserved = 0;
    }
    std::vector<double> fa(static_cast<size_t>(n * red[0] * R)), fb(static_cast<size_t>(n * red[1] * R)),
        fc(static_cast<size_t>(n * red[2] * R)), hist(static_cast<size_t>(n * cfg.als_max_iters));
    std::vector<int64_t> iters(static_cast<size_t>(n));
    std::vector<int32_t> conv(static_cast<size_t>(n));
    ck(xtsg_cp_als_batched(n, t, red[0], red[1], red[2], cfgs.data(), fa.data(), fb.data(), fc.data(), iters.data(),
                           conv.data(), hist.data()));
    // items are attempt-major: this walk replays each replica's attempts in
    // order and skips the ones the sequential loop would not have run
    for (int64_t k = 0; k < n; ++k) {
      const int64_t q = item_q[k];
      if (done(q)) continue;
      Stage1Out& o = out[static_cast<size_t>(q)];
      o.sweeps += iters[k];
      const double err = iters[k] > 0 ? hist[k * cfg.als_max_iters + iters[k] - 1] : 1.0;
      if (!o.have || err < o.err) {
        o.f.resize(static_cast<size_t>(per_f));
        std::copy_n(fa.data() + k * red[0] * R, red[0] * R, o.f.data());
        std::copy_n(fb.data() + k * red[1] * R, red[1] * R, o.f.data() + red[0] * R);
        std::copy_n(fc.data() + k * red[2] * R, red[2] * R, o.f.data() + (red[0] + red[1]) * R);
        o.err = err;
        o.conv = conv[k] != 0;
        o.have = 1;
      }
    }
    attempt += span - 1;
  }
  return out;
}

// Stages 1-3 of decompose (pipeline.cpp:410-572) on device-resident fp64
// replicas (Yd, all P of them), or — when `pre` is given — stages 2-3 on the
// stage-1 results of all P replicas computed elsewhere (multi-GPU: each rank
// ran stage 1 on its share of the replicas).
void decompose_stages(const xtsg_pipeline_config& cfg, const Resolved& rs, const EnsembleDev& ens, const double* Yd,
                      const Source& src, double* a_out, double* b_out, double* c_out, xtsg_pipeline_metrics* met,
                      cudaStream_t st, const std::vector<Stage1Out>* pre = nullptr) {
  const int64_t P = rs.replicas, R = rs.rank;
  const int64_t* red = rs.reduced;
  const int64_t per_f = (red[0] + red[1] + red[2]) * R;

  // ---- stage 1: decomposition (pipeline.cpp:410-446) ----------------------
  std::vector<double> flat_surv;
  std::vector<int64_t> decomp_survivors;
  int64_t sweeps = 0;
  run_stage(met, 1, "decomposition", st, [&] {
    std::vector<Stage1Out> res;
    if (pre) {
      res = *pre;
    } else {
      std::vector<int64_t> ids(static_cast<size_t>(P));
      for (int64_t p = 0; p < P; ++p) ids[p] = p;
      res = run_stage1(cfg, rs, P, ids.data(), Yd, st);
    }
    for (int64_t p = 0; p < P; ++p) {
      const Stage1Out& o = res[static_cast<size_t>(p)];
      sweeps += o.sweeps;
      if (o.have && o.conv && o.err <= cfg.replica_fit_tol) {
        flat_surv.insert(flat_surv.end(), o.f.begin(), o.f.end());
        decomp_survivors.push_back(p);
      }
    }
    if (decomp_survivors.empty())
      throw Status(XTSG_E_INSUFFICIENT, "decompose: every replica failed to fit", 0, rs.min_survivors);
  });
  if (met) {
    met->replicas_total = P;
    met->replicas_dropped = P - static_cast<int64_t>(decomp_survivors.size());
    met->als_sweeps = sweeps;
  }

  // ---- stage 2: alignment (pipeline.cpp:450-455) --------------------------
  const int64_t nd = static_cast<int64_t>(decomp_survivors.size());
  std::vector<double> aligned(static_cast<size_t>(nd * per_f));
  std::vector<int64_t> survivors;
  run_stage(met, 2, "alignment", st, [&] {
    std::vector<int32_t> dropped(static_cast<size_t>(nd));
    std::vector<int64_t> surv(static_cast<size_t>(nd));
    int64_t ns = 0;
    ck(xtsg_align_replicas(nd, red, R, flat_surv.data(), rs.shared, rs.min_survivors, aligned.data(), dropped.data(),
                           surv.data(), &ns));
    for (int64_t i = 0; i < ns; ++i) survivors.push_back(decomp_survivors[surv[i]]);
  });
  if (met) met->replicas_dropped = P - static_cast<int64_t>(survivors.size());

  // ---- stage 3: recovery (pipeline.cpp:458-572) ---------------------------
  run_stage(met, 3, "recovery", st, [&] {
    const int64_t S = static_cast<int64_t>(survivors.size());
    const int64_t off[3] = {0, red[0] * R, (red[0] + red[1]) * R};
    std::vector<double> est[3];
    for (int m = 0; m < 3; ++m) {
      const int64_t rows_u = rs.two_stage ? ens.inner_rows[m] : rs.dims[m];  // columns of the stacked compressor
      // stack_f: survivors' aligned factors; stack_u: their compressors (device)
      std::vector<double> sf(static_cast<size_t>(S * red[m] * R));
      for (int64_t i = 0; i < S; ++i)
        std::copy_n(aligned.data() + i * per_f + off[m], red[m] * R, sf.data() + i * red[m] * R);
      const double* ubase = rs.two_stage ? ens.outer[m].ptr : ens.u[m].ptr;
      const int64_t ublk = red[m] * rows_u;
      DevBuf<double> su(static_cast<size_t>(S * ublk), st);
      for (int64_t i = 0; i < S; ++i)
        XCUDA(cudaMemcpyAsync(su.ptr + i * ublk, ubase + survivors[i] * ublk, sizeof(double) * ublk,
                              cudaMemcpyDeviceToDevice, st));
      std::vector<int64_t> rows(static_cast<size_t>(S), red[m]);
      const int64_t stacked_rows = S * red[m];
      est[m].assign(static_cast<size_t>(rs.dims[m] * R), 0.0);
      // vstack(stack_f) in the reference layout (stacked_rows x R column-major)
      auto vstack_f = [&] {
        std::vector<double> v(static_cast<size_t>(stacked_rows * R));
        for (int64_t i = 0; i < S; ++i)
          for (int64_t c = 0; c < R; ++c)
            for (int64_t q = 0; q < red[m]; ++q)
              v[i * red[m] + q + stacked_rows * c] = sf[i * red[m] * R + q + red[m] * c];
        return v;
      };
      auto vstack_u = [&] {
        DevBuf<double> v(static_cast<size_t>(stacked_rows * rows_u), st);
        for (int64_t i = 0; i < S; ++i)
          XCUDA(cudaMemcpy2DAsync(v.ptr + i * red[m], sizeof(double) * stacked_rows, su.ptr + i * ublk,
                                  sizeof(double) * red[m], sizeof(double) * red[m], rows_u, cudaMemcpyDeviceToDevice,
                                  st));
        return v;
      };
      auto omp = [&](const double* measured, int64_t mrows, const double* dict, int64_t atoms, double* out) {
        ck(xtsg_omp_recover(measured, mrows, R, dict, atoms, cfg.omp_sparsity, cfg.omp_residual_tol, out));
      };
      if (rs.two_stage) {
        std::vector<double> x(static_cast<size_t>(rows_u * R));
        ck(xtsg_solve_stacked_ls(S, rows.data(), R, rows_u, sf.data(), su.ptr, x.data()));
        omp(x.data(), rows_u, ens.inner[m].ptr, rs.dims[m], est[m].data());
      } else if (rs.sparse && stacked_rows < rs.dims[m]) {
        const auto vf = vstack_f();
        const auto vu = vstack_u();
        omp(vf.data(), stacked_rows, vu.ptr, rs.dims[m], est[m].data());
      } else if (rs.sparse) {
        const int32_t rc = xtsg_solve_stacked_ls(S, rows.data(), R, rs.dims[m], sf.data(), su.ptr, est[m].data());
        if (rc == XTSG_E_ILLPOSED) {
          // sparse recovery does not need a full-rank stack (pipeline.cpp:510-517)
          const auto vf = vstack_f();
          const auto vu = vstack_u();
          omp(vf.data(), stacked_rows, vu.ptr, rs.dims[m], est[m].data());
        } else {
          ck(rc);
        }
      } else {
        ck(xtsg_solve_stacked_ls(S, rows.data(), R, rs.dims[m], sf.data(), su.ptr, est[m].data()));
      }
    }

    // sampled block (pipeline.cpp:521-545)
    std::vector<int64_t> sel[3];
    for (int m = 0; m < 3; ++m)
      sel[m] = (rs.sparse || rs.two_stage) ? select_rows_by_mass(est[m], rs.dims[m], R, rs.sample_b)
                                           : leading_rows(std::min(rs.sample_b, rs.dims[m]));
    const std::vector<double> block = source_block(src, rs.dims, sel, st);
    const int64_t bn[3] = {static_cast<int64_t>(sel[0].size()), static_cast<int64_t>(sel[1].size()),
                           static_cast<int64_t>(sel[2].size())};
    std::vector<double> bbest[3];
    double bbest_err = 1.0;
    bool have_block = false;
    {
      // the sampled block's 3 attempts (pipeline.cpp:524-537) run in one
      // batched launch; the sequential rule (keep the best, stop once it
      // fits to 1e-6) is replayed on the results in attempt order
      const int64_t bsz = bn[0] * bn[1] * bn[2];
      std::vector<double> blocks(static_cast<size_t>(3 * bsz));
      for (int q = 0; q < 3; ++q) std::copy(block.begin(), block.end(), blocks.begin() + q * bsz);
      xtsg_als_config als[3] = {};
      for (int q = 0; q < 3; ++q) {
        als[q].rank = R;
        als[q].max_iters = cfg.als_max_iters;
        als[q].tol = cfg.als_tol;
        als[q].seed = derive(cfg.seed, 31 + static_cast<uint64_t>(q));
        als[q].init = q == 1 ? 1 : 0;
      }
      std::vector<double> f[3];
      for (int m = 0; m < 3; ++m) f[m].resize(static_cast<size_t>(3 * bn[m] * R));
      std::vector<double> hist(static_cast<size_t>(3 * cfg.als_max_iters));
      int64_t it[3] = {0, 0, 0};
      int32_t conv[3] = {0, 0, 0};
      ck(xtsg_cp_als_batched(3, blocks.data(), bn[0], bn[1], bn[2], als, f[0].data(), f[1].data(), f[2].data(), it,
                             conv, hist.data()));
      for (int q = 0; q < 3; ++q) {
        const double err = it[q] > 0 ? hist[q * cfg.als_max_iters + it[q] - 1] : 1.0;
        if (!have_block || err < bbest_err) {
          for (int m = 0; m < 3; ++m)
            bbest[m].assign(f[m].begin() + q * bn[m] * R, f[m].begin() + (q + 1) * bn[m] * R);
          bbest_err = err;
          have_block = true;
        }
        if (bbest_err <= 1e-6) break;
      }
    }
    if (met) met->block_fit = bbest_err;
    std::vector<double> heads[3];
    for (int m = 0; m < 3; ++m) heads[m] = gather_rows(est[m], rs.dims[m], R, sel[m]);
    PermScale ps[3];
    match_factor_triples(heads, bbest, bn, R, ps);

    std::vector<double> fin[3];
    for (int m = 0; m < 3; ++m) {
      if (rs.sparse) {
        // re-solve sparsely in the recovered column order (pipeline.cpp:551-556)
        const int64_t rows_u = rs.dims[m];
        std::vector<double> vf(static_cast<size_t>(S * red[m] * R));
        for (int64_t i = 0; i < S; ++i)
          for (int64_t c = 0; c < R; ++c)
            for (int64_t q = 0; q < red[m]; ++q)
              vf[i * red[m] + q + S * red[m] * c] = aligned[i * per_f + off[m] + q + red[m] * c];
        PermScale& p = ps[m];
        const auto fwd = apply_forward(vf, S * red[m], p);
        DevBuf<double> vu(static_cast<size_t>(S * red[m] * rows_u), st);
        const int64_t ublk = red[m] * rows_u;
        for (int64_t i = 0; i < S; ++i)
          XCUDA(cudaMemcpy2DAsync(vu.ptr + i * red[m], sizeof(double) * S * red[m],
                                  ens.u[m].ptr + survivors[i] * ublk, sizeof(double) * red[m],
                                  sizeof(double) * red[m], rows_u, cudaMemcpyDeviceToDevice, st));
        fin[m].resize(static_cast<size_t>(rs.dims[m] * R));
        ck(xtsg_omp_recover(fwd.data(), S * red[m], R, vu.ptr, rs.dims[m], cfg.omp_sparsity, cfg.omp_residual_tol,
                            fin[m].data()));
      } else {
        fin[m] = apply_forward(est[m], rs.dims[m], ps[m]);
      }
    }
    double* outs[3] = {a_out, b_out, c_out};
    for (int m = 0; m < 3; ++m)
      XCUDA(cudaMemcpyAsync(outs[m], fin[m].data(), sizeof(double) * fin[m].size(), cudaMemcpyDefault, st));
    XCUDA(cudaStreamSynchronize(st));

    // held-out sample MSE on random rows (pipeline.cpp:561-570)
    std::vector<int64_t> hold[3];
    for (int m = 0; m < 3; ++m)
      hold[m] = random_rows(rs.dims[m], rs.sample_b, derive(cfg.seed, 41 + static_cast<uint64_t>(m)));
    const std::vector<double> truth = source_block(src, rs.dims, hold, st);
    const std::vector<double> rec = reconstruct_rows(fin, rs.dims, R, hold);
    if (met) met->sample_mse = mse(truth, rec);
  });
}

}  // namespace

}  // namespace xtsg

using namespace xtsg;

extern "C" {

int32_t xtsg_generate_factors(const int64_t dims[3], int64_t rank, int32_t law, int64_t nnz_per_col, uint64_t seed,
                              double* a, double* b, double* c) {
  // generate (pipeline.cpp:176-207) without materialization: gaussian_factor
  // (:157-162) is one flat polar stream per matrix; sparse_factor (:164-172)
  // draws each column's support by random_rows and its values by a polar stream.
  return guard([&] {
    for (int m = 0; m < 3; ++m)
      if (dims[m] < 1) usage("generate: dims must be >= 1");
    if (rank < 1) usage("generate: rank must be >= 1");
    double* outs[3] = {a, b, c};
    for (int m = 0; m < 3; ++m) {
      std::vector<double> f(static_cast<size_t>(dims[m] * rank), 0.0);
      if (law == XTSG_LAW_DENSE) {
        HostRng rng(derive(seed, 1 + static_cast<uint64_t>(m)));
        for (double& v : f) v = rng.normal();
      } else if (law == XTSG_LAW_SPARSE) {
        const int64_t nnz = nnz_per_col > 0 ? nnz_per_col : std::max<int64_t>(1, dims[m] / 100);
        if (nnz > dims[m]) usage("generate: nnz per column exceeds the dimension");
        const uint64_t ms = derive(seed, 4 + static_cast<uint64_t>(m));
        for (int64_t j = 0; j < rank; ++j) {
          const auto pos = random_rows(dims[m], nnz, derive(ms, 7000 + static_cast<uint64_t>(j)));
          HostRng rng(derive(ms, 9000 + static_cast<uint64_t>(j)));
          for (int64_t i : pos) f[i + dims[m] * j] = rng.normal();
        }
      } else {
        usage("generate: unknown law");
      }
      if (is_device_ptr(outs[m]))
        XCUDA(cudaMemcpy(outs[m], f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice));
      else
        std::copy(f.begin(), f.end(), outs[m]);
    }
  });
}

namespace {

// replicas (host or device, f32 or f64) -> device fp64
const double* replicas_f64(const void* replicas, int32_t dtype, int64_t n, DevBuf<double>& keep, cudaStream_t st) {
  if (dtype == XTSG_DTYPE_F64) {
    InView<double> v(static_cast<const double*>(replicas), static_cast<size_t>(n), st);
    if (v.tmp.ptr) {
      keep = std::move(v.tmp);
      return keep.ptr;
    }
    return v.dev;
  }
  if (dtype == XTSG_DTYPE_F32) {
    InView<float> v(static_cast<const float*>(replicas), static_cast<size_t>(n), st);
    keep = DevBuf<double>(static_cast<size_t>(n), st);
    widen_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16)), 256, 0, st>>>(v.dev, n, keep.ptr);
    XLAUNCH_CHECK();
    return keep.ptr;
  }
  usage("decompose: replicas must be f32 or f64");
}

}  // namespace

int32_t xtsg_decompose_stage1(const xtsg_pipeline_config* cfg, const int64_t dims[3], int64_t n, const int64_t* ids,
                              const void* replicas, int32_t replicas_dtype, double* factors, double* fit_err,
                              int32_t* converged, int64_t* sweeps) {
  return guard([&] {
    const Resolved rs = resolve(*cfg, dims);
    if (n < 0) usage("decompose_stage1: negative replica count");
    for (int64_t q = 0; q < n; ++q)
      if (ids[q] < 0 || ids[q] >= rs.replicas) usage("decompose_stage1: replica index outside [0, replicas)");
    if (n == 0) return;
    require_device();
    cudaStream_t st = thread_stream();
    const int64_t lmn = rs.reduced[0] * rs.reduced[1] * rs.reduced[2];
    const int64_t per_f = (rs.reduced[0] + rs.reduced[1] + rs.reduced[2]) * rs.rank;
    DevBuf<double> keep;
    const double* y = replicas_f64(replicas, replicas_dtype, n * lmn, keep, st);
    const std::vector<Stage1Out> res = run_stage1(*cfg, rs, n, ids, y, st);
    for (int64_t q = 0; q < n; ++q) {
      const Stage1Out& o = res[static_cast<size_t>(q)];
      if (o.have) std::copy(o.f.begin(), o.f.end(), factors + q * per_f);
      else std::fill_n(factors + q * per_f, per_f, 0.0);
      fit_err[q] = o.err;
      converged[q] = o.have && o.conv ? 1 : 0;
      sweeps[q] = o.sweeps;
    }
  });
}

int32_t xtsg_decompose_finish(const xtsg_pipeline_config* cfg, const int64_t dims[3], const double* factors,
                              const double* fit_err, const int32_t* converged, const int64_t* sweeps,
                              const double* tensor, const double* fa, const double* fb, const double* fc,
                              int64_t factor_rank, double* a_out, double* b_out, double* c_out,
                              xtsg_pipeline_metrics* metrics) {
  return guard([&] {
    if (metrics) *metrics = xtsg_pipeline_metrics{};
    const Resolved rs = resolve(*cfg, dims);
    require_device();
    cudaStream_t st = thread_stream();
    const Source src = make_source(dims, tensor, fa, fb, fc, factor_rank, st);
    EnsembleDev ens;
    make_ensemble_dev(rs, ens, st);
    const int64_t per_f = (rs.reduced[0] + rs.reduced[1] + rs.reduced[2]) * rs.rank;
    std::vector<Stage1Out> pre(static_cast<size_t>(rs.replicas));
    for (int64_t p = 0; p < rs.replicas; ++p) {
      Stage1Out& o = pre[static_cast<size_t>(p)];
      o.f.assign(factors + p * per_f, factors + (p + 1) * per_f);
      o.err = fit_err[p];
      o.conv = converged[p];
      o.have = 1;
      o.sweeps = sweeps[p];
    }
    decompose_stages(*cfg, rs, ens, nullptr, src, a_out, b_out, c_out, metrics, st, &pre);
  });
}

int32_t xtsg_decompose_replicas(const xtsg_pipeline_config* cfg, const int64_t dims[3], const void* replicas,
                                int32_t replicas_dtype, const double* tensor, const double* fa, const double* fb,
                                const double* fc, int64_t factor_rank, double* a_out, double* b_out, double* c_out,
                                xtsg_pipeline_metrics* metrics) {
  return guard([&] {
    if (metrics) *metrics = xtsg_pipeline_metrics{};
    const Resolved rs = resolve(*cfg, dims);
    require_device();
    cudaStream_t st = thread_stream();
    const Source src = make_source(dims, tensor, fa, fb, fc, factor_rank, st);
    EnsembleDev ens;
    make_ensemble_dev(rs, ens, st);
    const int64_t n = rs.replicas * rs.reduced[0] * rs.reduced[1] * rs.reduced[2];
    DevBuf<double> yd;
    const double* y = nullptr;
    if (replicas_dtype == XTSG_DTYPE_F64) {
      InView<double> v(static_cast<const double*>(replicas), static_cast<size_t>(n), st);
      if (v.tmp.ptr) {
        yd = std::move(v.tmp);
        y = yd.ptr;
      } else {
        y = v.dev;
      }
    } else if (replicas_dtype == XTSG_DTYPE_F32) {
      InView<float> v(static_cast<const float*>(replicas), static_cast<size_t>(n), st);
      yd = DevBuf<double>(static_cast<size_t>(n), st);
      widen_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16)), 256, 0, st>>>(v.dev, n, yd.ptr);
      XLAUNCH_CHECK();
      y = yd.ptr;
    } else {
      usage("decompose_replicas: replicas must be f32 or f64");
    }
    decompose_stages(*cfg, rs, ens, y, src, a_out, b_out, c_out, metrics, st);
  });
}

int32_t xtsg_decompose(const xtsg_pipeline_config* cfg, const int64_t dims[3], const double* tensor, const double* fa,
                       const double* fb, const double* fc, int64_t factor_rank, double* a_out, double* b_out,
                       double* c_out, xtsg_pipeline_metrics* metrics) {
  return guard([&] {
    if (metrics) *metrics = xtsg_pipeline_metrics{};
    const Resolved rs = resolve(*cfg, dims);
    if (cfg->precision != XTSG_PREC_FP64 && cfg->precision != XTSG_PREC_BF16 && cfg->precision != XTSG_PREC_FP16 &&
        cfg->precision != XTSG_PREC_FP16X3)
      usage("decompose: precision must be XTSG_PREC_FP64, XTSG_PREC_BF16, XTSG_PREC_FP16 or XTSG_PREC_FP16X3");
    require_device();
    cudaStream_t st = thread_stream();
    const Source src = make_source(dims, tensor, fa, fb, fc, factor_rank, st);
    EnsembleDev ens;
    const int64_t lmn = rs.reduced[0] * rs.reduced[1] * rs.reduced[2];
    DevBuf<double> yd(static_cast<size_t>(rs.replicas * lmn), st);
    // ---- stage 0: compression (pipeline.cpp:360-406) ----------------------
    run_stage(metrics, 0, "compression", st, [&] {
      make_ensemble_dev(rs, ens, st);
      if (cfg->precision == XTSG_PREC_FP64 && !tensor) {
        // comp_from_factors per replica (exact for factored sources, :397-405)
        for (int64_t p = 0; p < rs.replicas; ++p)
          ck(xtsg_comp_from_factors(fa, fb, fc, dims[0], dims[1], dims[2], factor_rank,
                                    ens.u[0].ptr + p * rs.reduced[0] * dims[0], rs.reduced[0],
                                    ens.u[1].ptr + p * rs.reduced[1] * dims[1], rs.reduced[1],
                                    ens.u[2].ptr + p * rs.reduced[2] * dims[2], rs.reduced[2], yd.ptr + p * lmn));
        return;
      }
      xtsg_plan_desc d{};
      for (int m = 0; m < 3; ++m) {
        d.dims[m] = dims[m];
        d.reduced[m] = rs.reduced[m];
      }
      d.count = rs.replicas;
      d.shared_rows = rs.shared;
      d.spec = rs.spec;
      d.seed = rs.ensemble_seed;
      d.precision = cfg->precision;
      xtsg_plan* plan = nullptr;
      ck(xtsg_plan_create(&d, &plan));
      struct Closer {
        xtsg_plan* p;
        ~Closer() { xtsg_plan_destroy(p); }
      } closer{plan};
      if (cfg->precision == XTSG_PREC_FP64) {
        const int64_t ld[2] = {dims[0], dims[0] * dims[1]};
        const int64_t zero[3] = {0, 0, 0};
        ck(xtsg_plan_compress(plan, tensor, XTSG_DTYPE_F64, ld, zero, dims, yd.ptr, 0, st));
        return;
      }
      DevBuf<float> yf(static_cast<size_t>(rs.replicas * lmn), st);
      if (tensor) {
        const int64_t ld[2] = {dims[0], dims[0] * dims[1]};
        const int64_t zero[3] = {0, 0, 0};
        ck(xtsg_plan_compress(plan, tensor, XTSG_DTYPE_F64, ld, zero, dims, yf.ptr, 0, st));
      } else {
        ck(xtsg_plan_compress_factors(plan, fa, fb, fc, factor_rank, 0, dims[2], yf.ptr, 0, st));
      }
      const int64_t n = rs.replicas * lmn;
      widen_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16)), 256, 0, st>>>(yf.ptr, n,
                                                                                                  yd.ptr);
      XLAUNCH_CHECK();
    });
    decompose_stages(*cfg, rs, ens, yd.ptr, src, a_out, b_out, c_out, metrics, st);
  });
}

int32_t xtsg_evaluate(const int64_t dims[3], int64_t rank, const double* ta, const double* tb, const double* tc,
                      const double* ra, const double* rb, const double* rc, int64_t sample, double mode_rel_err[3],
                      double* sample_mse, double* aligned_a, double* aligned_b, double* aligned_c) {
  // evaluate (pipeline.cpp:577-609), host arithmetic on host factor copies
  return guard([&] {
    if (rank < 1) usage("evaluate: ranks disagree");
    for (int m = 0; m < 3; ++m)
      if (dims[m] < 1) usage("evaluate: factor dimensions disagree");
    const double* tp[3] = {ta, tb, tc};
    const double* rp[3] = {ra, rb, rc};
    std::vector<double> t[3], r[3];
    for (int m = 0; m < 3; ++m) {
      t[m].resize(static_cast<size_t>(dims[m] * rank));
      r[m].resize(static_cast<size_t>(dims[m] * rank));
      copy_in(t[m], tp[m]);
      copy_in(r[m], rp[m]);
    }
    PermScale ps[3];
    match_factor_triples(r, t, dims, rank, ps);
    std::vector<double> al[3];
    double* outs[3] = {aligned_a, aligned_b, aligned_c};
    for (int m = 0; m < 3; ++m) {
      al[m] = apply_forward(r[m], dims[m], ps[m]);
      double num = 0.0, den = 0.0;
      for (size_t i = 0; i < t[m].size(); ++i) {
        const double d = t[m][i] - al[m][i];
        num += d * d;
        den += t[m][i] * t[m][i];
      }
      mode_rel_err[m] = den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
      if (outs[m] && is_device_ptr(outs[m]))
        XCUDA(cudaMemcpy(outs[m], al[m].data(), sizeof(double) * al[m].size(), cudaMemcpyHostToDevice));
      else if (outs[m])
        std::copy(al[m].begin(), al[m].end(), outs[m]);
    }
    int64_t b = sample > 0 ? sample : std::max<int64_t>(2 * rank, 8);
    b = std::min({b, dims[0], dims[1], dims[2]});
    std::vector<int64_t> head[3] = {leading_rows(b), leading_rows(b), leading_rows(b)};
    if (sample_mse) *sample_mse = mse(reconstruct_rows(t, dims, rank, head), reconstruct_rows(r, dims, rank, head));
  });
}

}  // extern "C"
