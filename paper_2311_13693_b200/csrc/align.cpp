// Replica alignment and permutation/scale recovery — host C++.
//
// These are O(P * R^3) bookkeeping steps on R <= ~64 columns (SURVEY §8 a12,
// a14: microseconds); the reference runs them on the host as well. They live
// in libxtsg so the C ABI is complete and the C++ facade can forward to them.
//   normalize_shared      alignment.cpp:66-85
//   max_trace_assignment  alignment.cpp:87-144 (exact, O(n^3), ties -> lowest index)
//   align_replicas        alignment.cpp:154-218
//   recover_perm_scale    alignment.cpp:254-278
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/xtsg.h"

namespace {

struct AbiError {
  int32_t code;
  std::string msg;
  int64_t p0, p1;
};

thread_local std::string t_msg;
thread_local int64_t t_p0 = 0, t_p1 = 0;

}  // namespace

// The CUDA translation unit owns the thread-local error state; host-only
// functions report through this hook so xtsg_last_error() sees them.
namespace xtsg {
void set_host_error(const std::string& msg, int64_t p0, int64_t p1);
}

namespace {

template <class F>
int32_t host_guard(F&& f) {
  try {
    f();
    return XTSG_OK;
  } catch (const AbiError& e) {
    xtsg::set_host_error(e.msg, e.p0, e.p1);
    return e.code;
  } catch (const std::exception& e) {
    xtsg::set_host_error(e.what(), 0, 0);
    return XTSG_E_INTERNAL;
  }
}

[[noreturn]] void fail(int32_t code, const std::string& m, int64_t p0 = 0, int64_t p1 = 0) {
  throw AbiError{code, m, p0, p1};
}

// Column-major view helpers.
inline double& at(double* m, int64_t rows, int64_t i, int64_t j) { return m[i + rows * j]; }
inline double at(const double* m, int64_t rows, int64_t i, int64_t j) { return m[i + rows * j]; }

// Pivot = entry of largest magnitude among the first `shared` rows (first
// occurrence wins on ties, sign kept); zero pivot -> degenerate column.
void normalize_cols(const double* m, int64_t rows, int64_t cols, int64_t shared, double* out,
                    double* pivots) {
  if (shared < 1 || shared > rows) fail(XTSG_E_USAGE, "normalize_shared: shared row count out of range");
  for (int64_t j = 0; j < cols; ++j) {
    double piv = 0.0;
    for (int64_t i = 0; i < shared; ++i) {
      const double x = at(m, rows, i, j);
      if (std::fabs(x) > std::fabs(piv)) piv = x;
    }
    if (piv == 0.0)
      fail(XTSG_E_DEGENERATE, "normalize_shared: column " + std::to_string(j) + " is zero within the shared rows",
           j);
    pivots[j] = piv;
    for (int64_t i = 0; i < rows; ++i) at(out, rows, i, j) = at(m, rows, i, j) / piv;
  }
}

// Maximum-trace assignment: minimum-cost perfect matching on -objective via
// successive shortest augmenting paths with row/column potentials.
std::vector<int64_t> assignment(const double* obj, int64_t n) {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> pot_r(n + 1, 0.0), pot_c(n + 1, 0.0), dist(n + 1);
  std::vector<int64_t> owner(n + 1, 0), prev(n + 1, 0);  // owner[c] = row matched to column c (1-based)
  std::vector<char> done(n + 1);
  for (int64_t row = 1; row <= n; ++row) {
    owner[0] = row;
    int64_t col = 0;
    std::fill(dist.begin(), dist.end(), inf);
    std::fill(done.begin(), done.end(), 0);
    while (owner[col] != 0) {
      done[col] = 1;
      const int64_t r = owner[col];
      double best = inf;
      int64_t best_col = 0;
      for (int64_t c = 1; c <= n; ++c) {
        if (done[c]) continue;
        const double reduced = -obj[(r - 1) + n * (c - 1)] - pot_r[r] - pot_c[c];
        if (reduced < dist[c]) {
          dist[c] = reduced;
          prev[c] = col;
        }
        if (dist[c] < best) {
          best = dist[c];
          best_col = c;
        }
      }
      for (int64_t c = 0; c <= n; ++c) {
        if (done[c]) {
          pot_r[owner[c]] += best;
          pot_c[c] -= best;
        } else {
          dist[c] -= best;
        }
      }
      col = best_col;
    }
    while (col != 0) {
      const int64_t pc = prev[col];
      owner[col] = owner[pc];
      col = pc;
    }
  }
  std::vector<int64_t> perm(n, 0);
  for (int64_t c = 1; c <= n; ++c) perm[owner[c] - 1] = c - 1;
  return perm;
}

// objective(r, c) = sum_i ref(i, r) * tgt(i, c) over the first `rows` rows.
void accumulate_gram(const double* ref, const double* tgt, int64_t ld, int64_t rows, int64_t r, double* obj) {
  for (int64_t c = 0; c < r; ++c)
    for (int64_t q = 0; q < r; ++q) {
      double s = 0.0;
      for (int64_t i = 0; i < rows; ++i) s += ref[i + ld * q] * tgt[i + ld * c];
      obj[q + r * c] += s;
    }
}

}  // namespace

extern "C" {

int32_t xtsg_normalize_shared(const double* m, int64_t rows, int64_t cols, int64_t shared_rows,
                              double* normalized, double* pivots) {
  return host_guard([&] { normalize_cols(m, rows, cols, shared_rows, normalized, pivots); });
}

int32_t xtsg_max_trace_assignment(const double* objective, int64_t n, int64_t* perm) {
  return host_guard([&] {
    if (n < 0) fail(XTSG_E_USAGE, "max_trace_assignment: objective must be square");
    const auto p = assignment(objective, n);
    std::copy(p.begin(), p.end(), perm);
  });
}

int32_t xtsg_align_replicas(int64_t count, const int64_t dims[3], int64_t r, const double* factors,
                            int64_t shared_rows, int64_t min_survivors, double* aligned, int32_t* dropped,
                            int64_t* survivors, int64_t* n_survivors) {
  return host_guard([&] {
    if (count < 1) fail(XTSG_E_USAGE, "align_replicas: no replicas");
    const int64_t per = (dims[0] + dims[1] + dims[2]) * r;
    std::vector<double> norm(static_cast<size_t>(count * per)), piv(static_cast<size_t>(r));
    std::vector<char> drop(static_cast<size_t>(count), 0);
    for (int64_t p = 0; p < count; ++p) {
      const double* f = factors + p * per;
      double* o = norm.data() + p * per;
      try {
        int64_t off = 0;
        for (int m = 0; m < 3; ++m) {
          normalize_cols(f + off, dims[m], r, shared_rows, o + off, piv.data());
          off += dims[m] * r;
        }
      } catch (const AbiError& e) {
        if (e.code != XTSG_E_DEGENERATE) throw;
        drop[p] = 1;
      }
    }
    int64_t ref = -1, alive = 0;
    for (int64_t p = 0; p < count; ++p)
      if (!drop[p]) {
        if (ref < 0) ref = p;
        ++alive;
      }
    for (int64_t p = 0; p < count; ++p) dropped[p] = drop[p];
    if (ref < 0 || alive < min_survivors)
      fail(XTSG_E_INSUFFICIENT,
           "align_replicas: only " + std::to_string(alive) + " of " + std::to_string(count) +
               " replicas survived, need " + std::to_string(min_survivors),
           alive, min_survivors);
    const double* refn = norm.data() + ref * per;
    int64_t ns = 0;
    std::vector<double> obj(static_cast<size_t>(r * r));
    for (int64_t p = 0; p < count; ++p) {
      if (drop[p]) continue;
      const double* src = norm.data() + p * per;
      double* dst = aligned + ns * per;
      if (p == ref) {
        std::memcpy(dst, src, sizeof(double) * per);
      } else {
        // all three modes' anchor blocks feed one assignment (:191-213)
        std::fill(obj.begin(), obj.end(), 0.0);
        int64_t off = 0;
        for (int m = 0; m < 3; ++m) {
          accumulate_gram(refn + off, src + off, dims[m], shared_rows, r, obj.data());
          off += dims[m] * r;
        }
        const auto perm = assignment(obj.data(), r);
        off = 0;
        for (int m = 0; m < 3; ++m) {
          for (int64_t c = 0; c < r; ++c)
            std::memcpy(dst + off + dims[m] * c, src + off + dims[m] * perm[c], sizeof(double) * dims[m]);
          off += dims[m] * r;
        }
      }
      survivors[ns++] = p;
    }
    *n_survivors = ns;
  });
}

int32_t xtsg_recover_perm_scale(const double* global_head, const double* sampled, int64_t rows, int64_t cols,
                                int64_t* perm, double* scale) {
  return host_guard([&] {
    std::vector<double> g(static_cast<size_t>(rows * cols)), s(static_cast<size_t>(rows * cols));
    std::vector<double> gp(static_cast<size_t>(cols)), sp(static_cast<size_t>(cols));
    normalize_cols(global_head, rows, cols, rows, g.data(), gp.data());
    normalize_cols(sampled, rows, cols, rows, s.data(), sp.data());
    double max_abs = 0.0;
    for (int64_t e = 0; e < rows * cols; ++e)
      max_abs = std::max({max_abs, std::fabs(global_head[e]), std::fabs(sampled[e])});
    const double tiny = 1e-12 * std::max(1.0, max_abs);
    for (int64_t j = 0; j < cols; ++j)
      if (std::fabs(gp[j]) < tiny || std::fabs(sp[j]) < tiny)
        fail(XTSG_E_DEGENERATE, "recover_perm_scale: near-zero pivot in column " + std::to_string(j), j);
    // hungarian_match(s, g): objective = s^T g
    std::vector<double> obj(static_cast<size_t>(cols * cols), 0.0);
    accumulate_gram(s.data(), g.data(), rows, rows, cols, obj.data());
    const auto p = assignment(obj.data(), cols);
    for (int64_t c = 0; c < cols; ++c) {
      perm[c] = p[c];
      scale[c] = sp[c] / gp[p[c]];
    }
  });
}

}  // extern "C"
