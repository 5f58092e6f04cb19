// Measured fp32 SIMT FMA peak of this GPU (the bound the SIMT sparse kernel
// would face): 8 independent FFMA chains per thread, 1024 threads x 4 CTAs per
// SM, CUDA-event timed, best of 5. Prints one JSON line.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void __launch_bounds__(1024) fma_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3f + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fmaf(x[q], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 12345.678f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 20000, blocks = sms * 2, threads = 1024;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_kernel<<<blocks, threads>>>(out, 100, 0.999f, 0.001f);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma = double(blocks) * threads * iters * 16.0 * 8.0;
  printf("{\"fp32_fma_tflops\": %.2f, \"fma_per_s\": %.4e, \"sms\": %d, \"ms\": %.3f, \"how\": \"8 independent FFMA chains x 16 unrolled per iteration, %d CTAs x %d threads, best of 5, 2 flop per FMA\"}\n",
         2.0 * fma / (best * 1e-3) / 1e12, fma / (best * 1e-3), sms, best, blocks, threads);
  return 0;
}
