// Microbenchmark: single-CTA streaming rate of a cp.async.bulk ring
// (1-D bulk copies global -> shared, mbarrier full/empty ring), as used by
// the large-replica CP-ALS kernel. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_poll(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\nP_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra P_%=;\n}" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(su32(bar)) : "memory");
}

__global__ void ring(const char* src, int64_t total, int chunk, int ns, int copies, long long* out, double* sink, int mode = 0) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const char* base = src + static_cast<int64_t>(blockIdx.x) * total;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], (mode & 2) ? blockDim.x / 32 - 1 : blockDim.x / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nch = total / chunk;
  auto issue = [&](int64_t c) {
    const int st = static_cast<int>(c % ns);
    if (c >= ns) { if (mode & 1) mbar_poll(&empty[st], static_cast<uint32_t>(((c / ns) - 1) & 1)); else mbar_wait(&empty[st], static_cast<uint32_t>(((c / ns) - 1) & 1)); }
    expect_tx(&full[st], chunk);
    const int part = chunk / copies;
    for (int q = 0; q < copies; ++q) bulk(sm + st * chunk + q * part, base + c * chunk + q * part, part, &full[st]);
  };
  long long t0 = clock64();
  double acc = 0.0;
  if (mode & 2) {  // warp 0 = producer, others consume
    if (threadIdx.x == 0) for (int64_t c = 0; c < nch; ++c) issue(c);
    else if (threadIdx.x >= 32)
      for (int64_t c = 0; c < nch; ++c) {
        const int st = static_cast<int>(c % ns);
        if (mode & 1) mbar_poll(&full[st], static_cast<uint32_t>((c / ns) & 1)); else mbar_wait(&full[st], static_cast<uint32_t>((c / ns) & 1));
        acc += reinterpret_cast<const double*>(sm + st * chunk)[threadIdx.x];
        __syncwarp();
        if ((threadIdx.x & 31) == 0) arrive(&empty[st]);
      }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (acc == 12345.0) sink[0] = acc;
    return;
  }
  if (mode & 4) {  // incremental stage / phase bookkeeping (no divisions)
    int pst = 0, pph = 0;  // producer: next stage to fill, its empty parity
    int64_t issued = 0;
    auto issue2 = [&]() {
      if (issued >= ns) mbar_wait(&empty[pst], pph ^ 1);
      expect_tx(&full[pst], chunk);
      bulk(sm + pst * chunk, base + issued * chunk, chunk, &full[pst]);
      ++issued;
      if (++pst == ns) { pst = 0; pph ^= 1; }
    };
    if (threadIdx.x == 0) for (int c = 0; c < ns && c < nch; ++c) issue2();
    int st = 0, ph = 0;
    for (int64_t c = 0; c < nch; ++c) {
      mbar_wait(&full[st], ph);
      acc += reinterpret_cast<const double*>(sm + st * chunk)[threadIdx.x];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) arrive(&empty[st]);
      if (threadIdx.x == 0 && issued < nch) issue2();
      if (++st == ns) { st = 0; ph ^= 1; }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (acc == 12345.0) sink[0] = acc;
    return;
  }
  if (threadIdx.x == 0) for (int c = 0; c < ns && c < nch; ++c) issue(c);
  for (int64_t c = 0; c < nch; ++c) {
    const int st = static_cast<int>(c % ns);
    if (mode & 1) mbar_poll(&full[st], static_cast<uint32_t>((c / ns) & 1)); else mbar_wait(&full[st], static_cast<uint32_t>((c / ns) & 1));
    acc += reinterpret_cast<const double*>(sm + st * chunk)[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) arrive(&empty[st]);
    if (threadIdx.x == 0 && c + ns < nch) issue(c + ns);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}

// burst: thread 0 (or lanes of warp 0) issues n copies of `part` bytes onto one
// barrier, waits once; reports cycles (cold: distinct source ranges per rep)
__global__ void burst(const char* src, int n, int part, int lanes, long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) expect_tx(&bar, n * part);
  __syncwarp();
  if (threadIdx.x < lanes)
    for (int q = threadIdx.x; q < n; q += lanes) bulk(sm + q * part, src + static_cast<int64_t>(q) * part, part, &bar);
  if (threadIdx.x == 0) { mbar_wait(&bar, 0); out[0] = clock64() - t0; }
}

// burst over separate barriers: copy q completes on bar[q]
__global__ void burst2(const char* src, int n, int part, long long* out, int order) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[32];
  if (threadIdx.x == 0) { for (int q = 0; q < n; ++q) mbar_init(&bar[q], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    if (order == 0) {
      for (int q = 0; q < n; ++q) { expect_tx(&bar[q], part); bulk(sm + q * part, src + static_cast<int64_t>(q) * part, part, &bar[q]); }
    } else {
      for (int q = 0; q < n; ++q) expect_tx(&bar[q], part);
      for (int q = 0; q < n; ++q) bulk(sm + q * part, src + static_cast<int64_t>(q) * part, part, &bar[q]);
    }
    for (int q = 0; q < n; ++q) mbar_wait(&bar[q], 0);
    out[0] = clock64() - t0;
  }
}

int main() {
  const int64_t total = 128ll * 128 * 128 * 8;  // one 128^3 fp64 replica
  const int blocks_list[2] = {1, 124};
  char* src;
  cudaMalloc(&src, total * 124);
  cudaMemset(src, 0, total * 124);
  long long* out;
  cudaMallocManaged(&out, 124 * sizeof(long long));
  double* sink;
  cudaMalloc(&sink, 8);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct Cfg { int chunk, ns, copies; } cfgs[] = {{8192, 8, 8}, {8192, 8, 1}, {8192, 16, 1}, {16384, 8, 1}, {32768, 4, 1}, {32768, 6, 1}, {16384, 12, 1}, {8192, 4, 1}};
  for (int mode : {0, 4})
  for (int bi = 0; bi < 1; ++bi)
    for (auto& c : cfgs) {
      const int smem = c.chunk * c.ns;
      cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      printf("mode %d ", mode);
      for (int rep = 0; rep < 2; ++rep) ring<<<blocks_list[bi], 256, smem>>>(src, total, c.chunk, c.ns, c.copies, out, sink, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      double mx = 0;
      for (int b = 0; b < blocks_list[bi]; ++b) mx = out[b] > mx ? out[b] : mx;
      printf("blocks %3d chunk %6d ns %2d copies %d: %.0f cycles, %.2f B/cycle per SM\n", blocks_list[bi], c.chunk, c.ns, c.copies, mx, total / mx);
    }
  for (int order = 0; order < 2; ++order) for (int n : {1, 2, 4, 8, 16, 24}) {
    cudaFuncSetAttribute(burst2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long best = 1ll << 60;
    for (int rep = 0; rep < 5; ++rep) {
      burst2<<<1, 32, 200 * 1024>>>(src + static_cast<int64_t>(rep + 1) * 40 * 1024 * 1024, n, 8192, out, order);
      cudaDeviceSynchronize();
      best = out[0] < best ? out[0] : best;
    }
    if (0) printf("burst2 order %d n %2d: %lld cycles\n", order, n, best);
  }
  for (int part : {8192}) for (int lanes : {1}) for (int n : {1, 2, 4, 8, 16, 24}) {
    const int smem = n * part;
    if (smem > 200 * 1024) continue;
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long best = 1ll << 60;
    for (int rep = 0; rep < 5; ++rep) {
      burst<<<1, 32, 200 * 1024>>>(src + static_cast<int64_t>(rep + 1) * 40 * 1024 * 1024, n, part, lanes, out);
      cudaDeviceSynchronize();
      best = out[0] < best ? out[0] : best;
    }
    if (0) printf("burst part %5d lanes %2d n %2d: %lld cycles\n", part, lanes, n, best);
  }
  return 0;
}
