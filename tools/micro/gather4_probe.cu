// Probe: TMA tile::gather4 with SWIZZLE_128B into a 1024-B aligned buffer at
// row offsets 0 and 4 (byte offset 512): prints whether the 16-byte chunks land
// where an address-based 128B swizzle puts them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
    uint32_t d0 = (uint32_t)__cvta_generic_to_shared(buf), d1 = d0 + 512;
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(d0), "l"(&tm), "r"(b), "r"(64), "r"(3), "r"(10), "r"(-1), "r"(7)
                 : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(d1), "l"(&tm), "r"(b), "r"(0), "r"(1), "r"(2), "r"(5), "r"(100000)
                 : "memory");
  }
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b) : "memory");
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int R = 20, C = 256;  // rows x cols (cols contiguous), value = row*1000 + col (as u16 mod)
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 1024);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult rc = ((Fn)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  k<<<1, 128>>>(tm, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> out(512);
  cudaMemcpy(out.data(), o, 1024, cudaMemcpyDeviceToHost);
  const int rows[8] = {3, 10, -1, 7, 1, 2, 5, 100000};
  const int cols[8] = {64, 64, 64, 64, 0, 0, 0, 0};
  int bad_addr = 0, bad_rel = 0;
  for (int r = 0; r < 8; ++r)
    for (int ch = 0; ch < 8; ++ch)
      for (int e2 = 0; e2 < 8; ++e2) {
        const int rr = rows[r];
        const uint16_t want = (rr < 0 || rr >= R) ? 0 : (uint16_t)(rr * 256 + cols[r] + ch * 8 + e2);
        // address-based swizzle: physical chunk = ch ^ (row % 8) with row = r (0..7 over the 1024 B)
        if (out[r * 64 + ((ch ^ r) * 8) + e2] != want) ++bad_addr;
        // box-relative swizzle: row index inside each 4-row gather
        if (out[r * 64 + ((ch ^ (r & 3)) * 8) + e2] != want) ++bad_rel;
      }
  printf("address-based swizzle mismatches: %d, box-relative mismatches: %d\n", bad_addr, bad_rel);
  return 0;
}
