// The facade's batching of concurrent cp_als calls (xts_facade.cpp AlsBatcher)
// and its whole-tensor push of in-memory block sources, checked through the
// reference's own API: 16 threads each decompose their own tensor (two
// shapes interleaved, so batches mix and split), every result must equal the
// same call made alone (bitwise: a batched replica runs the same device
// instance), and one tensor with a NaN must fail only its own call.
// comp_blocked over make_memory_block_source must equal comp() per replica.
// Prints "facade_concurrency: ok" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "xts/compression.hpp"
#include "xts/cp_als.hpp"
#include "xts/errors.hpp"
#include "xts/rng.hpp"

namespace {
xts::Tensor3 low_rank(xts::index_t n, xts::index_t r, std::uint64_t seed) {
  xts::Rng rng(seed);
  std::vector<double> a(n * r), b(n * r), c(n * r);
  for (auto* v : {&a, &b, &c})
    for (double& x : *v) x = rng.normal();
  xts::Tensor3 t(n, n, n);
  for (xts::index_t k = 0; k < n; ++k)
    for (xts::index_t j = 0; j < n; ++j)
      for (xts::index_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (xts::index_t q = 0; q < r; ++q) s += a[i + n * q] * b[j + n * q] * c[k + n * q];
        t(i, j, k) = s;
      }
  return t;
}

bool same(const xts::AlsResult& x, const xts::AlsResult& y) {
  if (x.iters != y.iters || x.converged != y.converged || x.error_history != y.error_history) return false;
  return x.factors.a.values == y.factors.a.values && x.factors.b.values == y.factors.b.values &&
         x.factors.c.values == y.factors.c.values;
}
}  // namespace

int main() {
  constexpr int Q = 16;
  std::vector<xts::Tensor3> ts;
  std::vector<xts::AlsConfig> cfg(Q);
  for (int q = 0; q < Q; ++q) {
    const xts::index_t n = q % 2 ? 20 : 24;
    ts.push_back(low_rank(n, 4, 100 + q));
    cfg[q].rank = 4;
    cfg[q].max_iters = 200;
    cfg[q].seed = 7 + q;
    if (q % 5 == 1) cfg[q].init = xts::AlsConfig::Init::nvecs;
  }
  ts[9].values[17] = std::numeric_limits<double>::quiet_NaN();
  std::vector<xts::AlsResult> alone(Q), together(Q);
  std::vector<int> err_alone(Q, 0), err_together(Q, 0);
  for (int q = 0; q < Q; ++q) {
    try {
      alone[q] = xts::cp_als(ts[q], cfg[q]);
    } catch (const xts::DataError&) {
      err_alone[q] = 1;
    }
  }
  std::vector<std::thread> th;
  for (int q = 0; q < Q; ++q)
    th.emplace_back([&, q] {
      try {
        together[q] = xts::cp_als(ts[q], cfg[q]);
      } catch (const xts::DataError&) {
        err_together[q] = 1;
      }
    });
  for (auto& t : th) t.join();
  int bad = 0;
  for (int q = 0; q < Q; ++q) {
    if (err_alone[q] != err_together[q] || err_alone[q] != (q == 9)) {
      std::printf("replica %d: error status alone %d concurrent %d\n", q, err_alone[q], err_together[q]);
      ++bad;
    } else if (!err_alone[q] && !same(alone[q], together[q])) {
      std::printf("replica %d: concurrent result differs from the single call\n", q);
      ++bad;
    }
  }
  // comp_blocked over an in-memory source (pushed whole) vs comp per replica
  const xts::Tensor3 t = low_rank(30, 3, 5);
  xts::EnsembleSpec spec;
  const xts::CompressionEnsemble ens = xts::make_ensemble({30, 30, 30}, {6, 5, 4}, 3, 2, spec, 11);
  for (bool det : {true, false}) {
    const xts::BlockGrid grid({30, 30, 30}, {30, 30, 30});
    const auto reps = xts::comp_blocked(grid, xts::make_memory_block_source(t, grid), ens, det);
    for (int p = 0; p < 3; ++p) {
      const xts::Tensor3 want = xts::comp(t, ens.u[p], ens.v[p], ens.w[p]);
      if (reps[p].values != want.values) {
        std::printf("comp_blocked (deterministic=%d) replica %d differs from comp\n", int(det), p);
        ++bad;
      }
    }
  }
  if (bad) return 1;
  std::printf("facade_concurrency: ok\n");
  return 0;
}
