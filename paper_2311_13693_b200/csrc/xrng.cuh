// Counter-based, bit-exact re-statement of the reference RNG for host and
// device.
//
// Reference: /root/reference/proj/include/xts/rng.hpp
//   next_u64  :15-20  splitmix64, state += 0x9e3779b97f4a7c15
//   uniform01 :23     (x >> 11) * 2^-53
//   normal    :26-41  polar method, spare cached, std::log / std::sqrt
//   derive    :46-50  2nd output of Rng(seed ^ (golden * (tag + 0x632b...)))
//
// splitmix64's n-th output is a pure function of (seed, n), so a row stream
// can be evaluated out of order: candidate pair t of a stream consumes
// outputs 2t and 2t+1. That is what lets the ensemble kernel generate one
// matrix row per warp with a ballot/prefix-sum over accepted pairs instead of
// the reference's sequential loop.
//
// Bit-exactness: the reference is built without -march (baseline x86-64), so
// u*u + v*v is two roundings (no FMA); std::log resolves to glibc 2.39's
// __log_fma on FMA+AVX2 hosts. xlog() below replays that variant's exact
// instruction sequence (fused/unfused as objdump shows it) with explicit
// __fma_rn/__dmul_rn/__dadd_rn so nvcc cannot re-associate or contract.
#pragma once
#include <cstdint>
#include <cmath>
#include <cstring>

#include "glibc_log_data.h"

#if defined(__CUDACC__)
#define XHD __host__ __device__ __forceinline__
#else
#define XHD inline
#endif

namespace xtsg {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

XHD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// n-th (0-based) output of a splitmix64 stream seeded with `seed`.
XHD uint64_t stream_at(uint64_t seed, uint64_t n) { return mix64(seed + (n + 1) * kGolden); }

XHD uint64_t derive(uint64_t seed, uint64_t tag) {
  return stream_at(seed ^ (kGolden * (tag + 0x632be59bd9b4e019ULL)), 1);
}

XHD double uniform_from(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

XHD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
XHD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}

// Explicitly rounded primitives: device intrinsics forbid contraction; on the
// host this header is compiled with -ffp-contract=off and std::fma.
#if defined(__CUDA_ARCH__)
#define XFMA(a, b, c) __fma_rn((a), (b), (c))
#define XMUL(a, b) __dmul_rn((a), (b))
#define XADD(a, b) __dadd_rn((a), (b))
#define XSUB(a, b) __dsub_rn((a), (b))
#define XDIV(a, b) __ddiv_rn((a), (b))
#define XSQRT(a) __dsqrt_rn((a))
#else
#define XFMA(a, b, c) std::fma((a), (b), (c))
#define XMUL(a, b) ((a) * (b))
#define XADD(a, b) ((a) + (b))
#define XSUB(a, b) ((a) - (b))
#define XDIV(a, b) ((a) / (b))
#define XSQRT(a) std::sqrt((a))
#endif

struct LogEntry {
  double invc, logc;
};

#if defined(__CUDACC__)
__device__ __constant__ static const LogEntry kLogTabDev[128] = XTSG_LOG_TAB_INIT;
#endif
static const LogEntry kLogTabHost[128] = XTSG_LOG_TAB_INIT;

// glibc 2.39 x86_64 __log_fma for finite x > 0 (the only inputs the polar
// method produces: 0 < s < 1). Subnormal inputs are renormalised like glibc.
XHD double xlog(double x) {
#if defined(__CUDA_ARCH__)
  const LogEntry* tab = kLogTabDev;
#else
  const LogEntry* tab = kLogTabHost;
#endif
  uint64_t ix = as_u64(x);
  if (ix - 0x3fee000000000000ULL < 0x0003090000000000ULL) {
    // |x - 1| small: log1p-style polynomial (B coefficients)
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = XSUB(x, 1.0);
    const double r2 = XMUL(r, r);
    const double r3 = XMUL(r, r2);
    const double p12 = XFMA(r2, XTSG_LOG_B3, XFMA(r, XTSG_LOG_B2, XTSG_LOG_B1));
    const double p45 = XFMA(r2, XTSG_LOG_B6, XFMA(r, XTSG_LOG_B5, XTSG_LOG_B4));
    double q = XFMA(r3, XTSG_LOG_B10, XFMA(r2, XTSG_LOG_B9, XFMA(r, XTSG_LOG_B8, XTSG_LOG_B7)));
    q = XFMA(q, r3, p45);
    q = XFMA(q, r3, p12);
    const double t = XFMA(r, 0x1.0p27, r);
    const double rhi = XFMA(-0x1.0p27, r, t);
    const double rlo = XSUB(r, rhi);
    const double rhi2 = XMUL(rhi, rhi);
    const double hi = XFMA(rhi2, XTSG_LOG_B0, r);
    double lo = XFMA(rhi2, XTSG_LOG_B0, XSUB(r, hi));
    lo = XFMA(XMUL(XTSG_LOG_B0, rlo), XADD(r, rhi), lo);
    const double y = XFMA(q, r3, lo);
    return XADD(hi, y);
  }
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return -INFINITY;
    if (ix == 0x7ff0000000000000ULL) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return NAN;
    ix = as_u64(XMUL(x, 0x1.0p52)) - (52ULL << 52);
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = static_cast<int>((tmp >> 45) & 127);
  const int64_t k = static_cast<int64_t>(tmp) >> 52;
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double z = as_f64(iz);
  const double kd = static_cast<double>(k);
  const double w = XFMA(kd, XTSG_LOG_LN2HI, tab[i].logc);
  const double r = XFMA(z, tab[i].invc, -1.0);
  const double hi = XADD(r, w);
  const double lo = XFMA(kd, XTSG_LOG_LN2LO, XADD(XSUB(w, hi), r));
  const double r2 = XMUL(r, r);
  const double r3 = XMUL(r, r2);
  const double p = XFMA(XFMA(r, XTSG_LOG_A4, XTSG_LOG_A3), r2, XFMA(r, XTSG_LOG_A2, XTSG_LOG_A1));
  const double t = XFMA(r2, XTSG_LOG_A0, lo);
  return XADD(XFMA(r3, p, t), hi);
}

// One polar-method candidate from outputs (2t, 2t+1) of `seed`'s stream.
// Returns true when accepted (0 < s < 1) and writes the two normals.
XHD bool polar_candidate(uint64_t seed, uint64_t t, double& n0, double& n1) {
  const double u = XSUB(2.0 * uniform_from(stream_at(seed, 2 * t)), 1.0);
  const double v = XSUB(2.0 * uniform_from(stream_at(seed, 2 * t + 1)), 1.0);
  const double s = XADD(XMUL(u, u), XMUL(v, v));
  if (s >= 1.0 || s == 0.0) return false;
  const double m = XSQRT(XDIV(-2.0 * xlog(s), s));
  n0 = XMUL(u, m);
  n1 = XMUL(v, m);
  return true;
}

// compression.cpp:19-25: +sqrt(s) w.p. 1/(2s), -sqrt(s) w.p. 1/(2s), else 0.
XHD double three_point(uint64_t x, double s, double root) {
  const double u = uniform_from(x);
  if (u < XDIV(0.5, s)) return root;
  if (u < XDIV(1.0, s)) return -root;
  return 0.0;
}

// Sequential host stream mirroring xts::Rng exactly (used by host code paths).
struct HostRng {
  uint64_t state;
  double spare = 0.0;
  bool have = false;
  explicit HostRng(uint64_t s) : state(s) {}
  uint64_t next() { return mix64(state += kGolden); }
  double uniform() { return uniform_from(next()); }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    for (;;) {
      const double u = XSUB(2.0 * uniform(), 1.0);
      const double v = XSUB(2.0 * uniform(), 1.0);
      const double s = XADD(XMUL(u, u), XMUL(v, v));
      if (s >= 1.0 || s == 0.0) continue;
      const double m = XSQRT(XDIV(-2.0 * xlog(s), s));
      spare = XMUL(v, m);
      have = true;
      return XMUL(u, m);
    }
  }
};

}  // namespace xtsg
