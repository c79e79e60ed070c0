// NEXT-3: the normalisations of the pre-norm CADET block (reading R32).
//   rmsnorm_fwd_kernel  Y = X / sqrt(mean(X^2) + eps) * gamma, rstd saved; warp per row, 16-byte loads
//   rmsnorm_bwd_kernel  dX = rstd gamma dY - X rstd^3 mean(X gamma dY) (+ dresid); dgamma partials in
//                       registers over grid-strided rows, one block reduction + atomic per column
// HBM-bound: 2 d B read + 2 d B written per row forward, 6 d B read + 2 d B written backward.
#include "../../include/cadet.h"
#include "launch.cuh"
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

// Both kernels: 256 threads, gamma staged once per block in shared memory, warps grid-stride over
// rows; each lane keeps its 8-column chunks of a row as raw bf16x8 (uint4) registers and unpacks on
// the fly, so many rows' loads are in flight per SM (the kernels are HBM-bound).
__device__ __forceinline__ void load_row(const __nv_bfloat16* base, int d, int lane, uint4 (&r)[RMS_MAXC]) {
#pragma unroll
  for (int c = 0; c < RMS_MAXC; ++c) {
    const int col = c * 256 + lane * 8;
    r[c] = col < d ? __ldcs(reinterpret_cast<const uint4*>(base + col)) : make_uint4(0, 0, 0, 0);
  }
}

__global__ void __launch_bounds__(256, 2) rmsnorm_fwd_kernel(const __nv_bfloat16* X, const float* gamma, int T, int d,
                                                          __nv_bfloat16* Y, float* rstd) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) float g_s[256 * RMS_MAXC];
  for (int i = threadIdx.x; i < d; i += blockDim.x) g_s[i] = gamma[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = gridDim.x * 8;
  // two rows per warp per iteration: 8 x 16 B loads per lane in flight
  for (int row = blockIdx.x * 8 + (threadIdx.x >> 5); row < T; row += 2 * nw) {
    uint4 xr[2][RMS_MAXC];
    float ss[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (row + h * nw < T) load_row(X + (size_t)(row + h * nw) * d, d, lane, xr[h]);
      else
#pragma unroll
        for (int c = 0; c < RMS_MAXC; ++c) xr[h][c] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ss[h] = 0.f;
#pragma unroll
      for (int c = 0; c < RMS_MAXC; ++c) {
        float x[8];
        unpack8(xr[h][c], x);
#pragma unroll
        for (int e = 0; e < 8; ++e) ss[h] = fmaf(x[e], x[e], ss[h]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss[0] += __shfl_xor_sync(0xffffffffu, ss[0], o);
      ss[1] += __shfl_xor_sync(0xffffffffu, ss[1], o);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rh = row + h * nw;
      if (rh >= T) continue;
      const float r = rsqrtf(ss[h] / (float)d + RMS_EPS);
      if (lane == 0) rstd[rh] = r;
#pragma unroll
      for (int c = 0; c < RMS_MAXC; ++c) {
        const int col = c * 256 + lane * 8;
        if (col < d) {
          float x[8], y[8];
          unpack8(xr[h][c], x);
          const float4 g0 = *reinterpret_cast<const float4*>(g_s + col);
          const float4 g1 = *reinterpret_cast<const float4*>(g_s + col + 4);
          const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) y[e] = x[e] * r * g[e];
          *reinterpret_cast<uint4*>(Y + (size_t)rh * d + col) = pack8(y);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const __nv_bfloat16* X, const float* gamma, const float* rstd,
                                                          const __nv_bfloat16* dY, const __nv_bfloat16* dresid, int T,
                                                          int d, __nv_bfloat16* dX, float* dgamma) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) float g_s[256 * RMS_MAXC];
  __shared__ __align__(16) float dg_s[8][256 * RMS_MAXC];  // per-warp dgamma partials (lane-private columns)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < d; i += blockDim.x) g_s[i] = gamma[i];
  for (int i = lane; i < d; i += 32) dg_s[w][i] = 0.f;
  __syncthreads();
  for (int row = blockIdx.x * 8 + w; row < T; row += gridDim.x * 8) {
    uint4 xr[RMS_MAXC], yr[RMS_MAXC], rr[RMS_MAXC];
    load_row(X + (size_t)row * d, d, lane, xr);
    load_row(dY + (size_t)row * d, d, lane, yr);
    if (dresid) load_row(dresid + (size_t)row * d, d, lane, rr);
    const float r = rstd[row];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < RMS_MAXC; ++c) {
      const int col = c * 256 + lane * 8;
      if (col < d) {
        float x[8], dy[8];
        unpack8(xr[c], x);
        unpack8(yr[c], dy);
        float4* dg = reinterpret_cast<float4*>(&dg_s[w][col]);
        float4 a0 = dg[0], a1 = dg[1];
        const float4 g0 = *reinterpret_cast<const float4*>(g_s + col);
        const float4 g1 = *reinterpret_cast<const float4*>(g_s + col + 4);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) s = fmaf(x[e], g[e] * dy[e], s);
        a0.x = fmaf(dy[0], x[0] * r, a0.x); a0.y = fmaf(dy[1], x[1] * r, a0.y);
        a0.z = fmaf(dy[2], x[2] * r, a0.z); a0.w = fmaf(dy[3], x[3] * r, a0.w);
        a1.x = fmaf(dy[4], x[4] * r, a1.x); a1.y = fmaf(dy[5], x[5] * r, a1.y);
        a1.z = fmaf(dy[6], x[6] * r, a1.z); a1.w = fmaf(dy[7], x[7] * r, a1.w);
        dg[0] = a0;
        dg[1] = a1;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float k = r * r * r * s / (float)d;
#pragma unroll
    for (int c = 0; c < RMS_MAXC; ++c) {
      const int col = c * 256 + lane * 8;
      if (col < d) {
        float x[8], dy[8], dr[8], dx[8];
        unpack8(xr[c], x);
        unpack8(yr[c], dy);
        if (dresid) unpack8(rr[c], dr);
        const float4 g0 = *reinterpret_cast<const float4*>(g_s + col);
        const float4 g1 = *reinterpret_cast<const float4*>(g_s + col + 4);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) dx[e] = r * g[e] * dy[e] - x[e] * k + (dresid ? dr[e] : 0.f);
        *reinterpret_cast<uint4*>(dX + (size_t)row * d + col) = pack8(dx);
      }
    }
  }
  __syncthreads();
  // dgamma: the 8 warps' partials in a fixed order, one atomic per column per block
  for (int col = threadIdx.x; col < d; col += blockDim.x) {
    float a = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) a += dg_s[ww][col];
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
    launch_pdl(rmsnorm_fwd_kernel, dim3(min((T + 15) / 16, 2 * sm_count())), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(X), gamma, T, d,
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
    const int blocks = min((T + 7) / 8, 3 * sm_count());
    launch_pdl(rmsnorm_bwd_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(X), gamma, rstd, reinterpret_cast<const __nv_bfloat16*>(dY),
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
