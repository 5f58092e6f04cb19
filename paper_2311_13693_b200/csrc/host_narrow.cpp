// Host-side narrowing of f32/f64 slabs to bf16 for the PCIe pipeline of
// Plan::compress_host_narrow (plan.cu). Round to nearest even, NaN quieted:
// bit-identical to the device's __float2bfloat16 (and, for f64, to its
// double -> float -> bf16 staging). Compiled by the host compiler with
// per-ISA clones so the branchless loop vectorises on AVX-512 / AVX2 hosts.
#include <cstdint>
#include <cstring>

namespace xtsg {

namespace {

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

}  // namespace

__attribute__((target_clones("avx512f", "avx2", "default")))
void narrow_rows_f32(const float* x, int64_t ni, int64_t nj, int64_t ld0, int64_t ld1, int64_t k0, int64_t row0,
                     int64_t row1, int64_t ldi, uint16_t* out) {
  for (int64_t row = row0; row < row1; ++row) {
    const int64_t j = row % nj, k = k0 + row / nj;
    uint16_t* dst = out + row * ldi;
    narrow_row(x + j * ld0 + k * ld1, ni, dst);
    for (int64_t i = ni; i < ldi; ++i) dst[i] = 0;
  }
}

__attribute__((target_clones("avx512f", "avx2", "default")))
void narrow_rows_f64(const double* x, int64_t ni, int64_t nj, int64_t ld0, int64_t ld1, int64_t k0, int64_t row0,
                     int64_t row1, int64_t ldi, uint16_t* out) {
  for (int64_t row = row0; row < row1; ++row) {
    const int64_t j = row % nj, k = k0 + row / nj;
    uint16_t* dst = out + row * ldi;
    narrow_row(x + j * ld0 + k * ld1, ni, dst);
    for (int64_t i = ni; i < ldi; ++i) dst[i] = 0;
  }
}

}  // namespace xtsg
