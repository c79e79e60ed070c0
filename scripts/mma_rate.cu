// Microbenchmark: tcgen05.mma issue-to-completion rate on one SM for the shapes the attention kernels use
// (kind::f16, bf16 in, fp32 accumulate, cta_group::1, M = 128): SS (both operands in shared memory) at
// N = 64 / 128 / 256 and TS (A from TMEM) at N = 64 / 128.  One CTA per SM, one thread issues ITERS chains
// of K = 16 MMAs into one accumulator and commits; cycles / MMA vs the floor M * N / 256 (B300_MICROARCH).
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_11410_b200/csrc \
//   -o /tmp/mma_rate scripts/mma_rate.cu && /tmp/mma_rate
#include <cstdio>

#include "ptx.cuh"

using namespace cadet;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 32768);
    const uint32_t idesc = idesc_bf16(128, N, 0, 0);
    unsigned long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {  // warm-up, then timed
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = smem_desc(sB + k * 32, 16, 1024, SWZ_128B);
          if (TS)
            mma_bf16_ts(tmem + 256, tmem + k * 8, bd, idesc, 1u);
          else
            mma_bf16_ss(tmem + 256, smem_desc(sA + k * 32, 16, 1024, SWZ_128B), bd, idesc, 1u);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, rep & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(unsigned long long* d, int sms) {
  const int iters = 2048;
  cudaFuncSetAttribute(mma_rate_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  mma_rate_kernel<N, TS><<<sms, 128, 66 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const double per = mean / (iters * 8.0), floor = 128.0 * N / 256.0;
  printf("{\"mode\": \"%s\", \"M\": 128, \"N\": %d, \"K\": 16, \"cycles_per_mma\": %.1f, \"floor\": %.1f, \"frac\": %.3f}\n",
         TS ? "TS" : "SS", N, per, floor, floor / per);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 256 * sizeof(unsigned long long));
  run<64, false>(d, sms);
  run<128, false>(d, sms);
  run<256, false>(d, sms);
  run<64, true>(d, sms);
  run<128, true>(d, sms);
  run<256, true>(d, sms);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
