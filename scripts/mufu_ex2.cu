// Microbenchmark ("MUFU ex2 ~3.25e12 /s, derived, to verify"): throughput of
// ex2.approx.ftz.f32 (the softmax exponential of the attention kernels) and, for scale, of FFMA, on
// every SM.  Each thread runs 8 independent dependency chains so the pipe, not the latency, binds.
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu scripts/mufu_ex2.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -1.0f + 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void ffma_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.5f + 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A83126F;" : "+f"(a[i]));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  float* out;
  cudaMalloc(&out, 4096);
  const int threads = 1024, blocks = sms * 2, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double rate[2];
  for (int k = 0; k < 2; ++k) {
    for (int rep = 0; rep < 2; ++rep) {  // warm-up, then timed
      cudaEventRecord(e0);
      if (k == 0)
        ex2_kernel<<<blocks, threads>>>(out, iters);
      else
        ffma_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    rate[k] = (double)blocks * threads * iters * 8 / (ms * 1e-3);
  }
  const double ghz = clk * 1e-6;
  printf("{\"sms\": %d, \"sm_clock_ghz_max\": %.3f, \"ex2_per_s\": %.4e, \"ex2_per_clk_per_sm_at_max_clock\": %.2f, "
         "\"ffma_per_s\": %.4e, \"ffma_per_clk_per_sm_at_max_clock\": %.2f}\n",
         sms, ghz, rate[0], rate[0] / (sms * ghz * 1e9), rate[1], rate[1] / (sms * ghz * 1e9));
  return 0;
}
