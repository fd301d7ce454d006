// FP32 CUDA-core FMA throughput on this GPU (the compute roof of the
// CUDA-core update / Gram kernels: measure before using it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak tools/fp32_peak.cu
// Each thread runs 16 independent FMA chains; grid = 8 CTAs x 256 threads per
// SM; best of 10 launches, CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma(float *out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 4);
  const int iters = 1 << 16, threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fma<<<blocks, threads>>>(out, 1024, 0.999f, 1e-3f);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_fma<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 16 * (double)iters * threads * blocks;
  printf("{\"fp32_fma_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %d, \"best_ms\": %.3f, "
         "\"nominal_tflops_at_max_clock\": %.2f}\n",
         flops / (best * 1e-3) / 1e12, sms, clk / 1000, best,
         2.0 * 128 * sms * (clk * 1e3) / 1e12);
  return 0;
}
