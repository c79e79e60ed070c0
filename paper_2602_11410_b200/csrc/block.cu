// NEXT-3: the normalisations of the pre-norm CADET block (reading R32).
//   rmsnorm_fwd_kernel  Y = X / sqrt(mean(X^2) + eps) * gamma, rstd saved; warp per row, 16-byte loads
//   rmsnorm_bwd_kernel  dX = rstd gamma dY - X rstd^3 mean(X gamma dY) (+ dresid); dgamma partials in
//                       registers over grid-strided rows, one block reduction + atomic per column
// HBM-bound: 2 d B read + 2 d B written per row forward, 6 d B read + 2 d B written backward.
#include "../../include/cadet.h"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {
void set_error(const char* msg);

constexpr float RMS_EPS = 1e-6f;
constexpr int RMS_MAXC = 4;  // 256-column chunks per lane: d <= 1024 (host-checked)

__device__ __forceinline__ void unpack8(const uint4& u, float (&x)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&x)[8]) {
  return make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
}

__global__ void __launch_bounds__(256) rmsnorm_fwd_kernel(const __nv_bfloat16* X, const float* gamma, int T, int d,
                                                          __nv_bfloat16* Y, float* rstd) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= T) return;
  float x[RMS_MAXC][8];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < RMS_MAXC; ++c) {
    const int col = c * 256 + lane * 8;
    if (col < d) {
      unpack8(*reinterpret_cast<const uint4*>(X + (size_t)row * d + col), x[c]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(x[c][e], x[c][e], ss);
    }
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / (float)d + RMS_EPS);
  if (lane == 0) rstd[row] = r;
#pragma unroll
  for (int c = 0; c < RMS_MAXC; ++c) {
    const int col = c * 256 + lane * 8;
    if (col < d) {
      float y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = x[c][e] * r * gamma[col + e];
      *reinterpret_cast<uint4*>(Y + (size_t)row * d + col) = pack8(y);
    }
  }
}

__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const __nv_bfloat16* X, const float* gamma, const float* rstd,
                                                          const __nv_bfloat16* dY, const __nv_bfloat16* dresid, int T,
                                                          int d, __nv_bfloat16* dX, float* dgamma) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float dg[RMS_MAXC][8];
#pragma unroll
  for (int c = 0; c < RMS_MAXC; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) dg[c][e] = 0.f;
  for (int row = blockIdx.x * 8 + w; row < T; row += gridDim.x * 8) {
    float x[RMS_MAXC][8], gy[RMS_MAXC][8];
    float s = 0.f;
    const float r = rstd[row];
#pragma unroll
    for (int c = 0; c < RMS_MAXC; ++c) {
      const int col = c * 256 + lane * 8;
      if (col < d) {
        float dy[8];
        unpack8(*reinterpret_cast<const uint4*>(X + (size_t)row * d + col), x[c]);
        unpack8(*reinterpret_cast<const uint4*>(dY + (size_t)row * d + col), dy);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          gy[c][e] = gamma[col + e] * dy[e];
          s = fmaf(x[c][e], gy[c][e], s);
          dg[c][e] = fmaf(dy[e], x[c][e] * r, dg[c][e]);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float k = r * r * r * s / (float)d;
#pragma unroll
    for (int c = 0; c < RMS_MAXC; ++c) {
      const int col = c * 256 + lane * 8;
      if (col < d) {
        float dx[8], dr[8];
        if (dresid)
          unpack8(*reinterpret_cast<const uint4*>(dresid + (size_t)row * d + col), dr);
#pragma unroll
        for (int e = 0; e < 8; ++e) dx[e] = r * gy[c][e] - x[c][e] * k + (dresid ? dr[e] : 0.f);
        *reinterpret_cast<uint4*>(dX + (size_t)row * d + col) = pack8(dx);
      }
    }
  }
  // dgamma: 8 warps of the block into shared memory (fixed order), one atomic per column
  __shared__ float sh[8][1024];
#pragma unroll
  for (int c = 0; c < RMS_MAXC; ++c) {
    const int col = c * 256 + lane * 8;
    if (col < d)
#pragma unroll
      for (int e = 0; e < 8; ++e) sh[w][col + e] = dg[c][e];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < d; col += blockDim.x) {
    float a = 0.f;
    for (int ww = 0; ww < 8; ++ww) a += sh[ww][col];
    atomicAdd(dgamma + col, a);
  }
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace cadet

using namespace cadet;

extern "C" {

cadet_status cadet_rmsnorm_forward(const void* X, const float* gamma, int32_t T, int32_t d, void* Y, float* rstd,
                                   cadet_stream_t stream) {
  if ((T > 0 && (!X || !Y || !rstd)) || !gamma || T < 0 || d <= 0 || d % 8 || d > 256 * RMS_MAXC) {
    set_error("rmsnorm_forward: bad argument (d % 8 == 0, d <= 1024)");
    return CADET_E_ARG;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 1);
  if (T > 0)
    rmsnorm_fwd_kernel<<<(T + 7) / 8, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(X), gamma, T, d,
                                                   reinterpret_cast<__nv_bfloat16*>(Y), rstd);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return CADET_E_CUDA;
  }
  return CADET_OK;
}

cadet_status cadet_rmsnorm_backward(const void* X, const float* gamma, const float* rstd, const void* dY,
                                    const void* dresid, int32_t T, int32_t d, void* dX, float* dgamma,
                                    cadet_stream_t stream) {
  if ((T > 0 && (!X || !rstd || !dY || !dX)) || !gamma || !dgamma || T < 0 || d <= 0 || d % 8 || d > 256 * RMS_MAXC) {
    set_error("rmsnorm_backward: bad argument (d % 8 == 0, d <= 1024)");
    return CADET_E_ARG;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e0 = cudaMemsetAsync(dgamma, 0, sizeof(float) * d, st);
  if (e0 != cudaSuccess) {
    set_error(cudaGetErrorString(e0));
    return CADET_E_CUDA;
  }
  ProfScope ps(PROF_OTHER, st, 1);
  if (T > 0) {
    const int blocks = min((T + 7) / 8, 8 * sm_count());
    rmsnorm_bwd_kernel<<<blocks, 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(X), gamma, rstd, reinterpret_cast<const __nv_bfloat16*>(dY),
        reinterpret_cast<const __nv_bfloat16*>(dresid), T, d, reinterpret_cast<__nv_bfloat16*>(dX), dgamma);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return CADET_E_CUDA;
  }
  return CADET_OK;
}

}  // extern "C"
