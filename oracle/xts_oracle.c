/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference algorithm for
 * the compression path, used as the parity checker by tests/, smoke() and
 * bench.py's cpu_baseline leg. Never linked into or called by the product.
 *
 * Plain C, fp64, scalar loops. Each function cites the reference it restates
 * (/root/reference/proj/...). Built with -O2 -ffp-contract=off and no -march,
 * like the reference (proj/src/CMakeLists.txt:21), so u*u + v*v rounds twice
 * and log() resolves to the same glibc variant: the RNG is bit-exact.
 * Pinned against the compiled reference (oracle/_ref) and the reference's
 * known-answer tests in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ULL

typedef struct {
  uint64_t state;
  double spare;
  int have;
} orng;

/* rng.hpp:15-20 */
static uint64_t next_u64(orng* r) {
  uint64_t z = (r->state += GOLDEN);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
/* rng.hpp:23 */
static double uniform01(orng* r) { return (double)(next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:26-41 */
static double normal(orng* r) {
  if (r->have) {
    r->have = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * uniform01(r) - 1.0;
    v = 2.0 * uniform01(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double m = sqrt(-2.0 * log(s) / s);
  r->spare = v * m;
  r->have = 1;
  return u * m;
}
static orng mk(uint64_t seed) {
  orng r = {seed, 0.0, 0};
  return r;
}
/* rng.hpp:46-50 */
uint64_t or_derive(uint64_t seed, uint64_t tag) {
  orng r = mk(seed ^ (GOLDEN * (tag + 0x632be59bd9b4e019ULL)));
  next_u64(&r);
  return next_u64(&r);
}

void or_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  orng r = mk(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = next_u64(&r);
}
void or_rng_normal(uint64_t seed, int64_t n, double* out) {
  orng r = mk(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = normal(&r);
}

/* compression.cpp:19-25 */
static double three_point(orng* r, double s) {
  const double u = uniform01(r);
  const double root = sqrt(s);
  if (u < 0.5 / s) return root;
  if (u < 1.0 / s) return -root;
  return 0.0;
}

/* compression.cpp:82-95 (returns -1 on usage error) */
int64_t or_replica_count(const int64_t* dims, const int64_t* red, int64_t slack) {
  for (int m = 0; m < 3; ++m)
    if (red[m] < 3 || red[m] > dims[m]) return -1;
  if (slack < 0) return -1;
  int64_t b = (dims[0] - 2 + red[0] - 3) / (red[0] - 2);
  int64_t b1 = (dims[1] + red[1] - 1) / red[1], b2 = (dims[2] + red[2] - 1) / red[2];
  if (b1 > b) b = b1;
  if (b2 > b) b = b2;
  return b + slack;
}

/* compression.cpp:97-103, column-major fill from one stream */
void or_gen_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  orng r = mk(seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = normal(&r);
}
/* compression.cpp:105-113 */
void or_gen_sparse(int64_t rows, int64_t cols, double s, uint64_t seed, double* out) {
  orng r = mk(seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = three_point(&r, s);
}

/* compression.cpp:40-72: P matrices rows x cols, column-major, back to back.
 * kind: 0 gaussian, 1 sparse (anchor rows always gaussian). */
void or_gen_mode(int64_t rows, int64_t cols, int64_t count, int64_t shared, int kind, double s,
                 uint64_t shared_seed, uint64_t seed, uint64_t tag, double* out) {
  for (int64_t p = 0; p < count; ++p) {
    const uint64_t rep = or_derive(seed, 1000 + 8 * (uint64_t)p + tag);
    double* m = out + p * rows * cols;
    for (int64_t r = 0; r < rows; ++r) {
      const int sh = r < shared;
      orng g = mk(or_derive(sh ? shared_seed : rep, (uint64_t)r));
      for (int64_t j = 0; j < cols; ++j)
        m[r + rows * j] = (sh || kind == 0) ? normal(&g) : three_point(&g, s);
    }
  }
}

/* compression.cpp:51-72 for ONE replica p of one mode, keeping only the
 * columns idx[0..nidx) (ascending): each row's stream is drawn up to the last
 * kept column, exactly as fill_row draws it. out is rows x nidx column-major.
 * Lets the tests check index spaces (10^6 columns) without materialising the
 * whole ensemble, and lets callers spread replicas over threads. */
void or_gen_replica_cols(int64_t rows, int64_t p, int64_t shared, int kind, double s, uint64_t shared_seed,
                         uint64_t seed, uint64_t tag, int64_t nidx, const int64_t* idx, double* out) {
  const uint64_t rep = or_derive(seed, 1000 + 8 * (uint64_t)p + tag);
  const int64_t last = nidx ? idx[nidx - 1] : -1;
  for (int64_t r = 0; r < rows; ++r) {
    const int sh = r < shared;
    orng g = mk(or_derive(sh ? shared_seed : rep, (uint64_t)r));
    int64_t q = 0;
    for (int64_t j = 0; j <= last; ++j) {
      const double x = (sh || kind == 0) ? normal(&g) : three_point(&g, s);
      while (q < nidx && idx[q] == j) out[r + rows * q++] = x;
    }
  }
}

/* naive column-major gemm C = A * B (fixed k order) */
static void gemm_nn(int64_t m, int64_t n, int64_t k, const double* a, const double* b, double* c) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t q = 0; q < k; ++q) acc += a[i + m * q] * b[q + k * j];
      c[i + m * j] = acc;
    }
}

/* compression.cpp:115-200. kind 0/1/2; for two-stage inner_rows[3] must be
 * the llround(alpha*L) etc. computed by the caller. */
void or_make_ensemble(const int64_t* dims, const int64_t* red, int64_t count, int64_t shared, int kind,
                      double s, int inner_kind, double inner_s, const int64_t* inner_rows, uint64_t seed,
                      double* u, double* v, double* w) {
  double* outs[3] = {u, v, w};
  for (int m = 0; m < 3; ++m) {
    const uint64_t sh = or_derive(seed, 101 + (uint64_t)m);
    if (kind != 2) {
      or_gen_mode(red[m], dims[m], count, shared, kind, s, sh, seed, (uint64_t)m, outs[m]);
      continue;
    }
    const int64_t ir = inner_rows[m];
    double* inner = (double*)malloc(sizeof(double) * ir * dims[m]);
    double* outer = (double*)malloc(sizeof(double) * count * red[m] * ir);
    const uint64_t ts = or_derive(seed, 201 + (uint64_t)m);
    if (inner_kind == 1)
      or_gen_sparse(ir, dims[m], inner_s, ts, inner);
    else
      or_gen_gaussian(ir, dims[m], ts, inner);
    or_gen_mode(red[m], ir, count, shared, 0, 1.0, sh, seed, (uint64_t)m, outer);
    for (int64_t p = 0; p < count; ++p)
      gemm_nn(red[m], dims[m], ir, outer + p * red[m] * ir, inner, outs[m] + p * red[m] * dims[m]);
    free(inner);
    free(outer);
  }
}

/* compression.cpp:202-209 + tensor.cpp:32-83: mode 1 -> 2 -> 3 products */
void or_comp(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l, const double* v,
             int64_t m, const double* w, int64_t n, double* y) {
  double* s1 = (double*)calloc((size_t)(l * n2 * n3) + 1, sizeof(double));
  double* s2 = (double*)calloc((size_t)(l * m * n3) + 1, sizeof(double));
  for (int64_t k = 0; k < n3; ++k)
    for (int64_t j = 0; j < n2; ++j)
      for (int64_t a = 0; a < l; ++a) {
        double acc = 0.0;
        for (int64_t i = 0; i < n1; ++i) acc += u[a + l * i] * t[i + n1 * (j + n2 * k)];
        s1[a + l * (j + n2 * k)] = acc;
      }
  for (int64_t k = 0; k < n3; ++k)
    for (int64_t b = 0; b < m; ++b)
      for (int64_t a = 0; a < l; ++a) {
        double acc = 0.0;
        for (int64_t j = 0; j < n2; ++j) acc += v[b + m * j] * s1[a + l * (j + n2 * k)];
        s2[a + l * (b + m * k)] = acc;
      }
  for (int64_t c = 0; c < n; ++c)
    for (int64_t b = 0; b < m; ++b)
      for (int64_t a = 0; a < l; ++a) {
        double acc = 0.0;
        for (int64_t k = 0; k < n3; ++k) acc += w[c + n * k] * s2[a + l * (b + m * k)];
        y[a + l * (b + m * c)] = acc;
      }
  free(s1);
  free(s2);
}

/* tensor.cpp:133-150 (bit-exact loop order) */
void or_reconstruct(const double* a, const double* b, const double* c, int64_t ni, int64_t nj, int64_t nk,
                    int64_t rank, double* out) {
  memset(out, 0, sizeof(double) * ni * nj * nk);
  for (int64_t r = 0; r < rank; ++r)
    for (int64_t k = 0; k < nk; ++k)
      for (int64_t j = 0; j < nj; ++j) {
        const double s = b[j + nj * r] * c[k + nk * r];
        double* slab = out + ni * (j + nj * k);
        for (int64_t i = 0; i < ni; ++i) slab[i] += a[i + ni * r] * s;
      }
}

/* compression.cpp:215-220 */
void or_comp_from_factors(const double* a, const double* b, const double* c, int64_t ni, int64_t nj, int64_t nk,
                          int64_t rank, const double* u, int64_t l, const double* v, int64_t m, const double* w,
                          int64_t n, double* y) {
  double* ua = (double*)malloc(sizeof(double) * l * rank + 8);
  double* vb = (double*)malloc(sizeof(double) * m * rank + 8);
  double* wc = (double*)malloc(sizeof(double) * n * rank + 8);
  gemm_nn(l, rank, ni, u, a, ua);
  gemm_nn(m, rank, nj, v, b, vb);
  gemm_nn(n, rank, nk, w, c, wc);
  or_reconstruct(ua, vb, wc, l, m, n, rank, y);
  free(ua);
  free(vb);
  free(wc);
}

/* test_support.hpp:50-64: raw elementwise Eq. 3 sum */
void or_comp_triple_sum(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                        const double* v, int64_t m, const double* w, int64_t n, double* y) {
  for (int64_t a = 0; a < l; ++a)
    for (int64_t b = 0; b < m; ++b)
      for (int64_t c = 0; c < n; ++c) {
        double acc = 0.0;
        for (int64_t i = 0; i < n1; ++i)
          for (int64_t j = 0; j < n2; ++j)
            for (int64_t k = 0; k < n3; ++k)
              acc += u[a + l * i] * v[b + m * j] * w[c + n * k] * t[i + n1 * (j + n2 * k)];
        y[a + l * (b + m * c)] = acc;
      }
}

/* pipeline.cpp:157-162: dense synthetic factor, one polar stream */
void or_generate_dense(const int64_t* dims, int64_t rank, uint64_t seed, double* a, double* b, double* c) {
  or_gen_gaussian(dims[0], rank, or_derive(seed, 1), a);
  or_gen_gaussian(dims[1], rank, or_derive(seed, 2), b);
  or_gen_gaussian(dims[2], rank, or_derive(seed, 3), c);
}

/* ---- precision model (half.cpp, mixed.cpp) ---------------------------- */

/* double_to_half_bits (half.cpp:10-47); returns -1 for HalfRangeError. */
int32_t or_half_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint32_t sign = (uint32_t)((b >> 63) << 15);
  const uint64_t dexp = (b >> 52) & 0x7ff, dman = b & ((1ULL << 52) - 1);
  if (dexp == 0x7ff) return -1;
  if (dexp == 0) return (int32_t)sign;
  const int e = (int)dexp - 1023;
  if (e >= 16) return -1;
  if (e <= -26) return (int32_t)sign;
  if (e >= -14) {
    uint64_t r = dman >> 42;
    const uint64_t rem = dman & ((1ULL << 42) - 1), hp = 1ULL << 41;
    if (rem > hp || (rem == hp && (r & 1))) ++r;
    int he = e;
    if (r == 1024) { r = 0; ++he; }
    if (he > 15) return -1;
    return (int32_t)(sign | (uint32_t)((he + 15) << 10) | (uint32_t)r);
  }
  const uint64_t full = (1ULL << 52) | dman;
  const int shift = 28 - e;
  uint64_t r = full >> shift;
  const uint64_t rem = full & ((1ULL << shift) - 1), hp = 1ULL << (shift - 1);
  if (rem > hp || (rem == hp && (r & 1))) ++r;
  if (r == 1024) return (int32_t)(sign | (1u << 10));
  return (int32_t)(sign | (uint32_t)r);
}

/* half_bits_to_double (half.cpp:49-60) */
double or_half_value(int32_t bits) {
  const int e = (bits >> 10) & 0x1f, man = bits & 0x3ff;
  double v = e == 0 ? ldexp((double)man, -24) : ldexp((double)(1024 + man), e - 25);
  return (bits >> 15) & 1 ? -v : v;
}

/* round_to_half / fp16_split / fp16_split_stored over n values (mixed.cpp:11-25);
 * mode 0 round, 1 split, 2 stored split. Returns 1 on HalfRangeError. */
int or_split(const double* x, int64_t n, int mode, double* half, double* res) {
  for (int64_t e = 0; e < n; ++e) {
    const int32_t hb = or_half_bits(x[e]);
    if (hb < 0) return 1;
    half[e] = or_half_value(hb);
    if (mode >= 1) {
      double r = x[e] - half[e];
      if (mode == 2) {
        const int32_t rb = or_half_bits(ldexp(r, 11));
        if (rb < 0) return 1;
        r = ldexp(or_half_value(rb), -11);
      }
      res[e] = r;
    }
  }
  return 0;
}

/* half_gemm (mixed.cpp:63-76) applied to one unfolding: out(a,c,b) = sum_x A(c,x) in(a,x,b) */
static void mode_seq(const double* A, int64_t nc, int64_t nx, const double* in, int64_t na, int64_t nb,
                     double* out) {
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t c = 0; c < nc; ++c)
      for (int64_t a = 0; a < na; ++a) {
        double acc = 0.0;
        for (int64_t x = 0; x < nx; ++x) acc += A[c + nc * x] * in[a + na * (x + nx * b)];
        out[a + na * (c + nc * b)] = acc;
      }
}

/* comp_with(t, u, v, w, &half_gemm) (compression.cpp:202-209, mixed.cpp:84-86) */
void or_comp_half(const double* t, int64_t n1, int64_t n2, int64_t n3, const double* u, int64_t l,
                  const double* v, int64_t m, const double* w, int64_t n, double* y) {
  double* s1 = malloc(sizeof(double) * (size_t)(l * n2 * n3 + 1));
  double* s2 = malloc(sizeof(double) * (size_t)(l * m * n3 + 1));
  mode_seq(u, l, n1, t, 1, n2 * n3, s1);
  mode_seq(v, m, n2, s1, l, n3, s2);
  mode_seq(w, n, n3, s2, l * m, 1, y);
  free(s1);
  free(s2);
}

/* comp_mixed (mixed.cpp:88-98) from split parts: five comp_half terms, add_inplace order */
void or_comp_mixed(const double* th, const double* tr, int64_t n1, int64_t n2, int64_t n3, const double* uh,
                   const double* ur, int64_t l, const double* vh, const double* vr, int64_t m, const double* wh,
                   const double* wr, int64_t n, double* y) {
  const int64_t yn = l * m * n;
  double* tmp = malloc(sizeof(double) * (size_t)(yn + 1));
  or_comp_half(th, n1, n2, n3, uh, l, vh, m, wh, n, y);
  const double* terms[4][4] = {{th, ur, vh, wh}, {th, uh, vr, wh}, {th, uh, vh, wr}, {tr, uh, vh, wh}};
  for (int q = 0; q < 4; ++q) {
    or_comp_half(terms[q][0], n1, n2, n3, terms[q][1], l, terms[q][2], m, terms[q][3], n, tmp);
    for (int64_t e = 0; e < yn; ++e) y[e] += tmp[e];
  }
  free(tmp);
}
