// Microbenchmark: per-SM throughput of the instructions the attention softmax is built from, alone
// and mixed, to learn which share a pipe on sm_100a: ex2.approx.ftz.f32 (MUFU), cvt.rn.bf16x2.f32
// (F2FP), ex2.approx.ftz.bf16x2, fma.rn.f32x2 (FFMA2), and ex2 + cvt mixed 2:1 (the softmax's ratio).
// Each thread runs 8 independent chains so the pipe, not the latency, binds.
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe scripts/pipe_bench.cu && /tmp/pipe
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t b[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = -1.0f + 0.001f * (threadIdx.x + i);
    b[i] = 0x3f803f80u + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "+r"(b[i]) : "f"(a[i]));
      if (MODE == 2) {  // 2 ex2 + 1 cvt (the softmax ratio)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "+r"(b[i]) : "f"(a[i - 1]));
      }
      if (MODE == 3) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b[i]));
      if (MODE == 4) {
        asm volatile("{.reg .b64 t; mov.b64 t, {%0, %1}; fma.rn.f32x2 t, t, t, t; mov.b64 {%0, %1}, t;}"
                     : "+f"(a[i]), "+f"(a[(i + 1) & 7]));
      }
      if (MODE == 5) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b[i]));
    }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)b[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int MODE>
double run(int blocks, int threads, int iters, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)blocks * threads * iters * 8 / (ms * 1e-3);  // instructions (per thread) per second
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4096);
  const int threads = 1024, blocks = sms * 2, iters = 4096;
  const double f = 1.0 / (sms * clk * 1e-6 * 1e9);
  const char* names[6] = {"ex2_f32", "cvt_bf16x2", "ex2_f32+cvt/2 (per ex2)", "ex2_bf16x2", "ffma2", "ex2_f16x2"};
  double r[6];
  r[0] = run<0>(blocks, threads, iters, out);
  r[1] = run<1>(blocks, threads, iters, out);
  r[2] = run<2>(blocks, threads, iters, out);
  r[3] = run<3>(blocks, threads, iters, out);
  r[4] = run<4>(blocks, threads, iters, out);
  r[5] = run<5>(blocks, threads, iters, out);
  printf("{");
  for (int i = 0; i < 6; ++i) printf("%s\"%s_per_clk_per_sm\": %.2f", i ? ", " : "", names[i], r[i] * f);
  printf("}\n");
  return 0;
}
