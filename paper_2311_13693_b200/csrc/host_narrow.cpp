// Host-side narrowing of f32/f64 slabs to bf16 for the PCIe pipeline of
// Plan::compress_host_narrow (plan.cu). Round to nearest even, NaN quieted:
// bit-identical to the device's __float2bfloat16 (and, for f64, to its
// double -> float -> bf16 staging). Compiled by the host compiler with
// per-ISA clones so the branchless loop vectorises on AVX-512 / AVX2 hosts.
#include <immintrin.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace xtsg {

namespace {

// float -> binary16 bits, round to nearest even (== __float2half_rn): exact
// for normals, subnormals, overflow to inf and NaN
inline uint16_t f2h(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t sign = (u >> 16) & 0x8000u;
  const uint32_t a = u & 0x7fffffffu;
  if (a >= 0x7f800000u) return static_cast<uint16_t>(sign | 0x7c00u | (a > 0x7f800000u ? 0x200u : 0u));
  if (a >= 0x477ff000u) return static_cast<uint16_t>(sign | 0x7c00u);  // rounds to >= 65520: inf
  if (a < 0x38800000u) {  // half subnormal or zero: round a * 2^24 to an integer
    if (a < 0x33000000u) return static_cast<uint16_t>(sign);  // below half of the smallest subnormal
    const uint32_t m = (a & 0x7fffffu) | 0x800000u;
    const int shift = 126 - static_cast<int>(a >> 23);  // 14..24
    uint32_t r = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u), hp = 1u << (shift - 1);
    if (rem > hp || (rem == hp && (r & 1u))) ++r;
    return static_cast<uint16_t>(sign | r);
  }
  const uint32_t r = a + 0xfffu + ((a >> 13) & 1u);  // RNE at bit 13
  return static_cast<uint16_t>(sign | ((r - 0x38000000u) >> 13));
}

template <class T>
inline void narrow_row_h(const T* __restrict__ src, int64_t n, uint16_t* __restrict__ dst) {
  for (int64_t i = 0; i < n; ++i) dst[i] = f2h(static_cast<float>(src[i]));
}

template <class T>
inline void narrow_row(const T* __restrict__ src, int64_t n, uint16_t* __restrict__ dst) {
  for (int64_t i = 0; i < n; ++i) {
    const float f = static_cast<float>(src[i]);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    const uint32_t qnan = (u >> 16) | 0x40u;
    dst[i] = static_cast<uint16_t>((u & 0x7fffffffu) > 0x7f800000u ? qnan : rne);
  }
}

// AVX2: 8 floats -> 8 bf16 per step, RNE + quiet NaN exactly like the scalar
// rule, written with non-temporal 16-byte stores (no read-for-ownership of
// the pinned destination: a third less host-memory traffic)
__attribute__((target("avx2"))) void narrow_row_bf16_avx2(const float* __restrict__ src, int64_t n,
                                                          uint16_t* __restrict__ dst) {
  const __m256i bias = _mm256_set1_epi32(0x7fff), one = _mm256_set1_epi32(1);
  const __m256i absm = _mm256_set1_epi32(0x7fffffff), inf = _mm256_set1_epi32(0x7f800000);
  const __m256i qbit = _mm256_set1_epi32(0x40);
  int64_t i = 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  for (; i + 8 <= n; i += 8) {
    const __m256i u = _mm256_castps_si256(_mm256_loadu_ps(src + i));
    const __m256i hi = _mm256_srli_epi32(u, 16);
    __m256i r = _mm256_srli_epi32(_mm256_add_epi32(_mm256_add_epi32(u, bias), _mm256_and_si256(hi, one)), 16);
    const __m256i nan = _mm256_cmpgt_epi32(_mm256_and_si256(u, absm), inf);
    r = _mm256_blendv_epi8(r, _mm256_or_si256(hi, qbit), nan);
    const __m256i pk = _mm256_permute4x64_epi64(_mm256_packus_epi32(r, r), 0x08);
    const __m128i out = _mm256_castsi256_si128(pk);
    if (aligned) _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), out);
    else _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), out);
  }
  for (; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, src + i, 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    dst[i] = static_cast<uint16_t>((u & 0x7fffffffu) > 0x7f800000u ? ((u >> 16) | 0x40u) : rne);
  }
}

// F16C: 8 floats -> 8 binary16 per vcvtps2ph with round-to-nearest-even
// (IEEE: subnormals, overflow to inf), non-temporal 16-byte stores
__attribute__((target("avx2,f16c"))) void narrow_row_f16_f16c(const float* __restrict__ src, int64_t n,
                                                             uint16_t* __restrict__ dst) {
  int64_t i = 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  for (; i + 8 <= n; i += 8) {
    const __m128i h = _mm256_cvtps_ph(_mm256_loadu_ps(src + i), _MM_FROUND_TO_NEAREST_INT);
    if (aligned) _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), h);
    else _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), h);
  }
  for (; i < n; ++i) dst[i] = f2h(src[i]);
}

bool host_has_f16c() {
  static const bool has = __builtin_cpu_supports("f16c") && __builtin_cpu_supports("avx2");
  return has;
}

// AVX-512: 16 floats -> 16 bf16 per step (same integer RNE rule), 32-byte
// non-temporal stores when aligned
__attribute__((target("avx512f"))) void narrow_row_bf16_avx512(const float* __restrict__ src, int64_t n,
                                                              uint16_t* __restrict__ dst) {
  const __m512i bias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1);
  const __m512i absm = _mm512_set1_epi32(0x7fffffff), inf = _mm512_set1_epi32(0x7f800000);
  const __m512i qbit = _mm512_set1_epi32(0x40);
  int64_t i = 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 31) == 0;
  for (; i + 16 <= n; i += 16) {
    const __m512i u = _mm512_castps_si512(_mm512_loadu_ps(src + i));
    const __m512i hi = _mm512_srli_epi32(u, 16);
    __m512i r = _mm512_srli_epi32(_mm512_add_epi32(_mm512_add_epi32(u, bias), _mm512_and_si512(hi, one)), 16);
    const __mmask16 nan = _mm512_cmpgt_epi32_mask(_mm512_and_si512(u, absm), inf);
    r = _mm512_mask_blend_epi32(nan, r, _mm512_or_si512(hi, qbit));
    const __m256i out = _mm512_cvtepi32_epi16(r);
    if (aligned && ((reinterpret_cast<uintptr_t>(dst + i) & 31) == 0))
      _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), out);
    else
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), out);
  }
  for (; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, src + i, 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    dst[i] = static_cast<uint16_t>((u & 0x7fffffffu) > 0x7f800000u ? ((u >> 16) | 0x40u) : rne);
  }
}

// AVX512-BF16: vcvtneps2bf16 rounds to nearest even in hardware but treats
// subnormal inputs as zero; vectors holding a float subnormal take the
// integer rule instead, so the result stays bit-identical to the device's
__attribute__((target("avx512f,avx512bf16"))) void narrow_row_bf16_hw(const float* __restrict__ src, int64_t n,
                                                                     uint16_t* __restrict__ dst) {
  const __m512i expm = _mm512_set1_epi32(0x7f800000), manm = _mm512_set1_epi32(0x007fffff);
  const __m512i zero = _mm512_setzero_si512();
  int64_t i = 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 31) == 0;
  for (; i + 16 <= n; i += 16) {
    const __m512 x = _mm512_loadu_ps(src + i);
    const __m512i u = _mm512_castps_si512(x);
    const __mmask16 sub = _mm512_cmpeq_epi32_mask(_mm512_and_si512(u, expm), zero) &
                          _mm512_cmpneq_epi32_mask(_mm512_and_si512(u, manm), zero);
    __m256i out;
    if (sub == 0) {
      out = reinterpret_cast<__m256i>(_mm512_cvtneps_pbh(x));
    } else {
      alignas(32) uint16_t tmp[16];
      for (int q = 0; q < 16; ++q) {
        uint32_t w;
        std::memcpy(&w, src + i + q, 4);
        const uint32_t rne = (w + 0x7fffu + ((w >> 16) & 1u)) >> 16;
        tmp[q] = static_cast<uint16_t>((w & 0x7fffffffu) > 0x7f800000u ? ((w >> 16) | 0x40u) : rne);
      }
      out = _mm256_load_si256(reinterpret_cast<const __m256i*>(tmp));
    }
    if (aligned && ((reinterpret_cast<uintptr_t>(dst + i) & 31) == 0))
      _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), out);
    else
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), out);
  }
  for (; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, src + i, 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    dst[i] = static_cast<uint16_t>((u & 0x7fffffffu) > 0x7f800000u ? ((u >> 16) | 0x40u) : rne);
  }
}

bool host_has_avx512bf16() {
  static const bool has = __builtin_cpu_supports("avx512bf16");
  return has;
}

bool host_has_avx512() {
  static const bool has = __builtin_cpu_supports("avx512f");
  return has;
}

bool host_has_avx2() {
  static const bool has = __builtin_cpu_supports("avx2");
  return has;
}

}  // namespace

__attribute__((target_clones("avx512f", "avx2", "default")))
void narrow_rows_f32(const float* x, int64_t ni, int64_t nj, int64_t ld0, int64_t ld1, int64_t k0, int64_t row0,
                     int64_t row1, int64_t ldi, uint16_t* out, bool f16) {
  for (int64_t row = row0; row < row1; ++row) {
    const int64_t j = row % nj, k = k0 + row / nj;
    uint16_t* dst = out + row * ldi;
    if (f16 && host_has_f16c()) narrow_row_f16_f16c(x + j * ld0 + k * ld1, ni, dst);
    else if (f16) narrow_row_h(x + j * ld0 + k * ld1, ni, dst);
    else if (host_has_avx512bf16()) narrow_row_bf16_hw(x + j * ld0 + k * ld1, ni, dst);
    else if (host_has_avx512()) narrow_row_bf16_avx512(x + j * ld0 + k * ld1, ni, dst);
    else if (host_has_avx2()) narrow_row_bf16_avx2(x + j * ld0 + k * ld1, ni, dst);
    else narrow_row(x + j * ld0 + k * ld1, ni, dst);
    for (int64_t i = ni; i < ldi; ++i) dst[i] = 0;
  }
  _mm_sfence();
}

__attribute__((target_clones("avx512f", "avx2", "default")))
void narrow_rows_f64(const double* x, int64_t ni, int64_t nj, int64_t ld0, int64_t ld1, int64_t k0, int64_t row0,
                     int64_t row1, int64_t ldi, uint16_t* out, bool f16) {
  for (int64_t row = row0; row < row1; ++row) {
    const int64_t j = row % nj, k = k0 + row / nj;
    uint16_t* dst = out + row * ldi;
    if (f16) narrow_row_h(x + j * ld0 + k * ld1, ni, dst);
    else narrow_row(x + j * ld0 + k * ld1, ni, dst);
    for (int64_t i = ni; i < ldi; ++i) dst[i] = 0;
  }
}

// Persistent fork-join workers for the narrowing slabs: spawning and joining
// a fresh std::thread per worker per 256 MB slab cost ~0.3 ms of a ~6 ms
// slab. One run at a time (callers serialise on run_mu); the pool is leaked
// on purpose so no joinable thread is destroyed at process exit.
namespace {
class WorkerPool {
 public:
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> rg(run_mu_);
    while (static_cast<int>(th_.size()) < n - 1) {
      const int id = static_cast<int>(th_.size()) + 1;
      th_.emplace_back([this, id] { worker(id); });
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &fn;
      njob_ = n;
      remaining_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return remaining_ == 0; });
    job_ = nullptr;
  }

 private:
  void worker(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f = nullptr;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= njob_) continue;
        f = job_;
      }
      (*f)(id);
      std::lock_guard<std::mutex> g(mu_);
      if (--remaining_ == 0) done_.notify_one();
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* job_ = nullptr;
  int njob_ = 0, remaining_ = 0;
  uint64_t gen_ = 0;
};
}  // namespace

void run_workers(int n, const std::function<void(int)>& fn) {
  static WorkerPool* pool = new WorkerPool;
  if (n <= 1) {
    fn(0);
    return;
  }
  pool->run(n, fn);
}

}  // namespace xtsg
