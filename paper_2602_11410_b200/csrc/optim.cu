// NEXT-4: the optimizer step of the HSDP training step (reading R35).
//   adamw_kernel     fused AdamW over one rank's shard of the flat fp32 master parameters: m, v, the
//                    master and its bf16 compute copy updated in one pass (30 B per parameter)
//   widen_kernel     bf16 -> fp32 (the fp32-consumed parameters, e.g. biases, after the all-gather)
// Both are HBM-bound elementwise passes: 16-byte vector accesses, grid-stride over 4 x SMs blocks.
#include "../../include/cadet.h"
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {
void set_error(const char* msg);

struct AdamArgs {
  float lr, beta1, beta2, eps, decay;  // decay = 1 - lr * weight_decay
  float inv_bc1, inv_bc2;              // 1 / (1 - beta^step), computed on the host in double
};

__device__ __forceinline__ float adam_one(float& p, float& m, float& v, float g, const AdamArgs& a) {
  m = fmaf(a.beta1, m, (1.f - a.beta1) * g);
  v = fmaf(a.beta2, v, (1.f - a.beta2) * g * g);
  const float den = sqrtf(v * a.inv_bc2) + a.eps;
  p = p * a.decay - a.lr * (m * a.inv_bc1) / den;
  return p;
}

__global__ void __launch_bounds__(256) adamw_kernel(const float* __restrict__ g, float* __restrict__ p,
                                                    float* __restrict__ m, float* __restrict__ v,
                                                    __nv_bfloat16* __restrict__ pbf, int64_t n, AdamArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 pp = reinterpret_cast<float4*>(p)[i], mm = reinterpret_cast<float4*>(m)[i],
           vv = reinterpret_cast<float4*>(v)[i];
    adam_one(pp.x, mm.x, vv.x, gg.x, a);
    adam_one(pp.y, mm.y, vv.y, gg.y, a);
    adam_one(pp.z, mm.z, vv.z, gg.z, a);
    adam_one(pp.w, mm.w, vv.w, gg.w, a);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (pbf) reinterpret_cast<uint2*>(pbf)[i] = make_uint2(pack_bf16(pp.x, pp.y), pack_bf16(pp.z, pp.w));
  }
  // ragged tail (n % 4 elements)
  for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam_one(pp, mm, vv, g[i], a);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (pbf) pbf[i] = __float2bfloat16_rn(pp);
  }
}

__global__ void __launch_bounds__(256) widen_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst,
                                                    int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n8 = n >> 3;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    const uint4 u = reinterpret_cast<const uint4*>(src)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    float4* o = reinterpret_cast<float4*>(dst) + 2 * i;
    const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]), c = __bfloat1622float2(h[2]),
                 d = __bfloat1622float2(h[3]);
    o[0] = make_float4(a.x, a.y, b.x, b.y);
    o[1] = make_float4(c.x, c.y, d.x, d.y);
  }
  for (int64_t i = (n8 << 3) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __bfloat162float(src[i]);
}

static int grid_for(int64_t work) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 4 * sms ? 4 * sms : b));
}

static cadet_status launch_err(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return CADET_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  set_error(buf);
  return CADET_E_CUDA;
}

}  // namespace cadet

using namespace cadet;

extern "C" {

void cadet_default_adamw_config(cadet_adamw_config* c) {
  if (!c) return;
  c->lr = 1e-4f;
  c->beta1 = 0.9f;
  c->beta2 = 0.999f;
  c->eps = 1e-8f;
  c->weight_decay = 0.f;
}

cadet_status cadet_adamw_step(const cadet_adamw_config* c, int64_t step, const float* grad, float* param, float* m,
                              float* v, void* param_bf16, int64_t n, cadet_stream_t stream) {
  if (!c || step < 1 || n < 0 || (n > 0 && (!grad || !param || !m || !v)) ||
      ((reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(m) |
        reinterpret_cast<uintptr_t>(v)) & 15) ||
      (reinterpret_cast<uintptr_t>(param_bf16) & 7)) {
    set_error("adamw_step: bad argument (step >= 1, non-null 16-byte-aligned fp32 buffers, 8-byte-aligned bf16)");
    return CADET_E_ARG;
  }
  if (n == 0) return CADET_OK;
  AdamArgs a;
  a.lr = c->lr;
  a.beta1 = c->beta1;
  a.beta2 = c->beta2;
  a.eps = c->eps;
  a.decay = (float)(1.0 - (double)c->lr * (double)c->weight_decay);
  a.inv_bc1 = (float)(1.0 / (1.0 - pow((double)c->beta1, (double)step)));
  a.inv_bc2 = (float)(1.0 / (1.0 - pow((double)c->beta2, (double)step)));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 1);
  launch_pdl(adamw_kernel, dim3(grid_for(n / 4 + 1)), dim3(256), 0, st, grad, param, m, v, reinterpret_cast<__nv_bfloat16*>(param_bf16),
                                                    n, a);
  return launch_err("adamw_step");
}

cadet_status cadet_bf16_to_f32(const void* src, float* dst, int64_t n, cadet_stream_t stream) {
  if (n < 0 || (n > 0 && (!src || !dst)) || (reinterpret_cast<uintptr_t>(src) & 15) ||
      (reinterpret_cast<uintptr_t>(dst) & 15)) {
    set_error("bf16_to_f32: bad argument (16-byte-aligned buffers)");
    return CADET_E_ARG;
  }
  if (n == 0) return CADET_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 1);
  launch_pdl(widen_kernel, dim3(grid_for(n / 8 + 1)), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(src), dst, n);
  return launch_err("bf16_to_f32");
}

}  // extern "C"
