// Eigen-free implementations of the three out-of-line helpers declared in the
// reference's tests/test_support.hpp:84-111 (the reference's own
// test_support.cpp needs Eigen, which is not installed). Test infrastructure
// only: lets the reference's unit and acceptance tests build unchanged.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <numeric>
#include <vector>

#include "test_support.hpp"

namespace xts::testsupport {

namespace {

// cyclic Jacobi eigendecomposition of a small symmetric matrix (row-major n x n)
void sym_eig(std::vector<double>& a, int n, std::vector<double>& evals, std::vector<double>& evecs) {
  evecs.assign(static_cast<std::size_t>(n * n), 0.0);
  for (int i = 0; i < n; ++i) evecs[static_cast<std::size_t>(i * n + i)] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += a[i * n + j] * a[i * n + j];
        if (i != j) off += a[i * n + j] * a[i * n + j];
      }
    if (off <= 1e-26 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double tau = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double kp = a[k * n + p], kq = a[k * n + q];
          a[k * n + p] = c * kp - s * kq;
          a[k * n + q] = s * kp + c * kq;
        }
        for (int k = 0; k < n; ++k) {
          const double pk = a[p * n + k], qk = a[q * n + k];
          a[p * n + k] = c * pk - s * qk;
          a[q * n + k] = s * pk + c * qk;
        }
        for (int k = 0; k < n; ++k) {
          const double vp = evecs[k * n + p], vq = evecs[k * n + q];
          evecs[k * n + p] = c * vp - s * vq;
          evecs[k * n + q] = s * vp + c * vq;
        }
      }
  }
  evals.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) evals[static_cast<std::size_t>(i)] = a[i * n + i];
}

double residual_of_support(const Matrix& d, const std::vector<double>& y, const std::vector<index_t>& s) {
  const int k = static_cast<int>(s.size());
  std::vector<double> g(static_cast<std::size_t>(k * k)), b(static_cast<std::size_t>(k));
  for (int i = 0; i < k; ++i) {
    for (int j = 0; j < k; ++j) {
      double acc = 0.0;
      for (index_t r = 0; r < d.rows; ++r) acc += d(r, s[i]) * d(r, s[j]);
      g[static_cast<std::size_t>(i * k + j)] = acc;
    }
    double acc = 0.0;
    for (index_t r = 0; r < d.rows; ++r) acc += d(r, s[i]) * y[static_cast<std::size_t>(r)];
    b[static_cast<std::size_t>(i)] = acc;
  }
  // Cholesky solve of the normal equations (tiny k)
  for (int j = 0; j < k; ++j) {
    double diag = g[j * k + j];
    for (int q = 0; q < j; ++q) diag -= g[j * k + q] * g[j * k + q];
    if (diag <= 0.0) return std::numeric_limits<double>::infinity();
    diag = std::sqrt(diag);
    g[j * k + j] = diag;
    for (int i = j + 1; i < k; ++i) {
      double v = g[i * k + j];
      for (int q = 0; q < j; ++q) v -= g[i * k + q] * g[j * k + q];
      g[i * k + j] = v / diag;
    }
  }
  for (int i = 0; i < k; ++i) {
    double v = b[i];
    for (int q = 0; q < i; ++q) v -= g[i * k + q] * b[q];
    b[i] = v / g[i * k + i];
  }
  for (int i = k - 1; i >= 0; --i) {
    double v = b[i];
    for (int q = i + 1; q < k; ++q) v -= g[q * k + i] * b[q];
    b[i] = v / g[i * k + i];
  }
  double res = 0.0;
  for (index_t r = 0; r < d.rows; ++r) {
    double fit = 0.0;
    for (int i = 0; i < k; ++i) fit += d(r, s[i]) * b[i];
    const double e = y[static_cast<std::size_t>(r)] - fit;
    res += e * e;
  }
  return res;
}

}  // namespace

Matrix low_coherence_dictionary(index_t rows, index_t atoms, std::uint64_t seed, int iters) {
  const int n = static_cast<int>(atoms);
  Matrix best;
  double best_mu = 2.0;
  for (int restart = 0; restart < 4; ++restart) {
    Matrix d(rows, atoms);
    Rng rng(seed + 7919ull * static_cast<std::uint64_t>(restart));
    for (index_t j = 0; j < atoms; ++j) {
      double nn = 0.0;
      for (index_t i = 0; i < rows; ++i) {
        d(i, j) = rng.normal();
        nn += d(i, j) * d(i, j);
      }
      for (index_t i = 0; i < rows; ++i) d(i, j) /= std::sqrt(nn);
    }
    for (int it = 0; it < iters; ++it) {
      // Gram, shrink the largest 40% of off-diagonal magnitudes, project onto
      // rank-`rows` PSD matrices, refactor and renormalise.
      std::vector<double> g(static_cast<std::size_t>(n * n)), mags;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
          double acc = 0.0;
          for (index_t i = 0; i < rows; ++i) acc += d(i, a) * d(i, b);
          g[a * n + b] = acc;
          if (a != b) mags.push_back(std::fabs(acc));
        }
      std::sort(mags.begin(), mags.end());
      const double thr = mags[static_cast<std::size_t>(mags.size() * 0.6)];
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
          if (a != b && std::fabs(g[a * n + b]) > thr) g[a * n + b] *= 0.9;
      std::vector<double> ev, vec;
      sym_eig(g, n, ev, vec);
      std::vector<int> order(n);
      std::iota(order.begin(), order.end(), 0);
      std::sort(order.begin(), order.end(), [&](int x, int y) { return ev[x] > ev[y]; });
      Matrix nd(rows, atoms);
      for (index_t i = 0; i < rows; ++i) {
        const int q = order[static_cast<std::size_t>(i)];
        const double sq = std::sqrt(std::max(0.0, ev[q]));
        for (int a = 0; a < n; ++a) nd(i, a) = sq * vec[a * n + q];
      }
      for (index_t j = 0; j < atoms; ++j) {
        double nn = 0.0;
        for (index_t i = 0; i < rows; ++i) nn += nd(i, j) * nd(i, j);
        nn = std::sqrt(nn);
        if (nn > 0)
          for (index_t i = 0; i < rows; ++i) nd(i, j) /= nn;
      }
      d = nd;
      const double mu = coherence(d);
      if (mu < best_mu) {
        best_mu = mu;
        best = d;
      }
    }
  }
  return best;
}

std::vector<index_t> best_support_exhaustive(const Matrix& dictionary, const std::vector<double>& y, int k) {
  std::vector<index_t> cur, best;
  double best_res = std::numeric_limits<double>::infinity();
  std::function<void(index_t)> rec = [&](index_t start) {
    if (static_cast<int>(cur.size()) == k) {
      const double r = residual_of_support(dictionary, y, cur);
      if (r < best_res) {
        best_res = r;
        best = cur;
      }
      return;
    }
    for (index_t j = start; j < dictionary.cols; ++j) {
      cur.push_back(j);
      rec(j + 1);
      cur.pop_back();
    }
  };
  rec(0);
  return best;
}

std::uint16_t half_bits_oracle(double x, bool& overflow) {
  overflow = false;
  const bool neg = std::signbit(x);
  const double ax = std::fabs(x);
  if (ax >= 65520.0) {  // past the midpoint between 65504 and 2^16
    overflow = true;
    return 0;
  }
  // scan every finite non-negative binary16 value for the nearest; ties -> even mantissa
  std::uint16_t best = 0;
  double best_d = std::numeric_limits<double>::infinity();
  for (std::uint32_t bits = 0; bits < 0x7c00; ++bits) {
    const int e = static_cast<int>(bits >> 10), m = static_cast<int>(bits & 0x3ff);
    const double v = e == 0 ? std::ldexp(static_cast<double>(m), -24)
                            : std::ldexp(1.0 + static_cast<double>(m) / 1024.0, e - 15);
    const double dist = std::fabs(v - ax);
    if (dist < best_d || (dist == best_d && (bits & 1) == 0 && (best & 1) == 1)) {
      best_d = dist;
      best = static_cast<std::uint16_t>(bits);
    }
  }
  return static_cast<std::uint16_t>(best | (neg ? 0x8000 : 0));
}

}  // namespace xts::testsupport
