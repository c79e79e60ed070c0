// Elementwise / reduction kernels of the hot path that are HBM-bound (no tensor cores):
//   (RoPE angles alpha_i = dt_row theta_i, theta_i = (phi_min / dt_max) base^(2i/hd), are
//    evaluated on the fly by the kernels that rotate: no (cos, sin) table exists in HBM)
//   gate_rope_fwd_kernel    A4: Qr = RoPE(Q * sigma(Zq)), Kr = RoPE(K * sigma(Zk))
//   rope_apply_kernel       RoPE without interaction gate (ablation path)
//   rope_gate_bwd_kernel    A11: dQt = R(-alpha) dQr; g = sigma(Zq); u = dQt*Q*g*(1-g); r = dQt*g
//   gather_rows_kernel      H_r = H[rows] (A7 operand)
//   head_init / head_dz / head_dhid   A7/A8 routed BCE (Eq. 9) and the tower backward
//   add_kernel              Y = O (+ resid) when the output projection is ablated
#include "misc.cuh"
#include <algorithm>
#include <cuda_fp16.h>
#include <string.h>
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {


// alpha = dt * theta in fp64, reduced mod 2 pi in fp64 (|k| <= ~1e3: the 2 pi rounding error
// k * 2.4e-16 is negligible), then MUFU sincos on r in [-pi, pi] (abs err ~5e-7).
__device__ __forceinline__ void rope_cs(double dt, double th, float& c, float& s) {
  const double ang = dt * th;
  const double k = rint(ang * 0.15915494309189535);
  const float r = (float)fma(-k, 6.283185307179586, ang);
  __sincosf(r, &s, &c);
}

// alpha = dt theta in compensated fp32: dt = dth + dtl (exact), theta = thh + thl; p + lo = dt theta to
// ~2^-40 relative; reduction by 2 pi = 6.2831855f - 1.7484556e-7f (two FMAs), then MUFU sincos
__device__ __forceinline__ void rope_cs_f(float dth, float dtl, float thh, float thl, float& c, float& s) {
  const float p = dth * thh;
  const float lo = fmaf(dth, thl, fmaf(dtl, thh, fmaf(dth, thh, -p)));
  const float k = rintf(p * 0.15915494f);
  float r = fmaf(-k, 6.28318548202514648f, p);
  r = fmaf(-k, -1.7484556e-7f, r) + lo;
  __sincosf(r, &s, &c);
}
// (cos, sin) of pairs i0 .. i0 + N - 1 of `row` (time rebased to the row's sequence start)
template <int N>
__device__ __forceinline__ void rope_row_cs(const RopeOTF& rp, int row, int i0, float (&c)[N], float (&s)[N]) {
  const float2 d = rp.dt[row];  // one load: the plan rebased and split the row's time
  const float dth = d.x, dtl = d.y;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float2 th = rp.theta[i0 + e];
    rope_cs_f(dth, dtl, th.x, th.y, c[e], s[e]);
  }
}

// one thread per (row, pair of columns)
__global__ void rope_apply_kernel(const __nv_bfloat16* in, __nv_bfloat16* out, int T, int d, int hd, RopeOTF rp) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t pairs = (size_t)T * d / 2;
  if (idx >= pairs) return;
  const int row = (int)(idx / (d / 2));
  const int c = (int)(idx % (d / 2)) * 2;
  const float2 v = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(in)[idx]);
  float cv[1] = {1.f}, sv[1] = {0.f};
  if (rp.on) rope_row_cs<1>(rp, row, (c % hd) / 2, cv, sv);
  reinterpret_cast<__nv_bfloat162*>(out)[idx] =
      __floats2bfloat162_rn(v.x * cv[0] - v.y * sv[0], v.x * sv[0] + v.y * cv[0]);
}

// A4 after the gate GEMMs (Z_q = Q W_qg, Z_k = K W_kg stored bf16): Qr = RoPE_t(Q * sigma(Z_q)) and
// Kr = RoPE_t(K * sigma(Z_k)) in one HBM pass (Eq. 5 + P:274); one thread per (row, 8 columns), Q
// and K together so the row's angles are evaluated once; rp.on = 0: no RoPE.
__global__ void __launch_bounds__(256) gate_rope_fwd_kernel(const __nv_bfloat16* Q, const __nv_bfloat16* K,
                                                            const __nv_bfloat16* Gq, const __nv_bfloat16* Gk,
                                                            RopeOTF rp, __nv_bfloat16* Qr, __nv_bfloat16* Kr,
                                                            int T, int d, int hd, float* tapQ, float* tapK) {
  pdl_trigger();
  pdl_wait();
  const int per_row = d / 8;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * per_row) return;
  const int row = idx / per_row, c0 = (idx - row * per_row) * 8;
  const size_t off = (size_t)row * d + c0;
  float cv[4] = {1.f, 1.f, 1.f, 1.f}, sv[4] = {0.f, 0.f, 0.f, 0.f};
  if (rp.on) rope_row_cs<4>(rp, row, (c0 % hd) / 2, cv, sv);  // the 8-column group never crosses a head edge
  const __nv_bfloat16* src[2] = {Q, K};
  const __nv_bfloat16* gate[2] = {Gq, Gk};
  __nv_bfloat16* dst[2] = {Qr, Kr};
  float* tap[2] = {tapQ, tapK};
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const uint4 xu = *reinterpret_cast<const uint4*>(src[w] + off);
    const uint4 gu = *reinterpret_cast<const uint4*>(gate[w] + off);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xu);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu);
    uint32_t o[4];
    float f[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __bfloat1622float2(x2[e]), z = __bfloat1622float2(g2[e]);
      const float a = x.x * sigmoid_fast(z.x), b = x.y * sigmoid_fast(z.y);
      f[2 * e] = a * cv[e] - b * sv[e];
      f[2 * e + 1] = a * sv[e] + b * cv[e];
      o[e] = pack_bf16(f[2 * e], f[2 * e + 1]);
    }
    *reinterpret_cast<uint4*>(dst[w] + off) = make_uint4(o[0], o[1], o[2], o[3]);
    if (tap[w]) {  // parity tap: the fp32 value before its bf16 rounding
      float4* t4 = reinterpret_cast<float4*>(tap[w] + off);
      t4[0] = make_float4(f[0], f[1], f[2], f[3]);
      t4[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
  }
}

// dr: fp32 (dQr accumulator) or bf16 (dKr).  gate (Z) bf16 may be null (no interaction gate):
// then out_u is unused and out_r (bf16 if r_bf16) receives dQt directly.
// One thread = 8 consecutive columns (4 pairs) of one row: 16-byte accesses, (cos, sin) from the
// row's RoPE angles evaluated on the fly (rp.on = 0: no RoPE).
struct RgSide {
  const void* dr;
  const __nv_bfloat16* Xq;
  const __nv_bfloat16* Z;
  __nv_bfloat16* out_u;
  void* out_r;
  float* tap_u;  // parity taps (nullable): fp32 u and r before their bf16 rounding
  float* tap_r;
};
struct RgSides {
  RgSide s[2];
};
// Both sides of A11 (Q, K) in one thread: the row's (cos, sin) are evaluated once for the two sides (the
// MUFU sincos work was half of this kernel's issue slots), and all of the thread's loads (up to six 16-byte
// chunks) are issued before any arithmetic.  nsides = 1: the single-side entry point.
template <bool TAPS>
__global__ void __launch_bounds__(256) rope_gate_bwd_kernel(RgSides sides, int nsides, int dr_f32, int r_bf16, int T,
                                                            int d, int hd, RopeOTF rp) {
  pdl_trigger();
  pdl_wait();
  const int per_row = d / 8;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)T * per_row) return;
  const int row = (int)(idx / per_row);
  const int c0 = (int)(idx % per_row) * 8;
  const size_t off = (size_t)row * d + c0;
  // loads of both sides first
  uint4 dru[2][2], zu[2], xu[2];
#pragma unroll
  for (int sd = 0; sd < 2; ++sd) {
    if (sd >= nsides) break;
    const RgSide& S = sides.s[sd];
    if (dr_f32) {
      dru[sd][0] = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(S.dr) + off)[0];
      dru[sd][1] = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(S.dr) + off)[1];
    } else {
      dru[sd][0] = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(S.dr) + off);
    }
    if (S.Z) {
      zu[sd] = *reinterpret_cast<const uint4*>(S.Z + off);
      xu[sd] = *reinterpret_cast<const uint4*>(S.Xq + off);
    }
  }
  float cv[4] = {1.f, 1.f, 1.f, 1.f}, sv[4] = {0.f, 0.f, 0.f, 0.f};
  if (rp.on) rope_row_cs<4>(rp, row, (c0 % hd) / 2, cv, sv);  // the 8-column group never crosses a head edge
#pragma unroll
  for (int sd = 0; sd < 2; ++sd) {
    if (sd >= nsides) break;
    const RgSide& S = sides.s[sd];
    float g[8];
    if (dr_f32) {
      const float* f = reinterpret_cast<const float*>(&dru[sd][0]);
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] = f[e];
    } else {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&dru[sd][0]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h2[e]);
        g[2 * e] = f.x;
        g[2 * e + 1] = f.y;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // R(-alpha)
      const float x0 = g[2 * e], x1 = g[2 * e + 1];
      g[2 * e] = x0 * cv[e] + x1 * sv[e];
      g[2 * e + 1] = x1 * cv[e] - x0 * sv[e];
    }
    float r[8];
    if (S.Z) {
      const __nv_bfloat162* z2 = reinterpret_cast<const __nv_bfloat162*>(&zu[sd]);
      const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xu[sd]);
      uint32_t uo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 z = __bfloat1622float2(z2[e]);
        const float2 x = __bfloat1622float2(x2[e]);
        const float g0 = sigmoid_fast(z.x), g1 = sigmoid_fast(z.y);
        const float u0 = g[2 * e] * x.x * g0 * (1.f - g0), u1 = g[2 * e + 1] * x.y * g1 * (1.f - g1);
        __nv_bfloat162 v = __floats2bfloat162_rn(u0, u1);
        uo[e] = *reinterpret_cast<uint32_t*>(&v);
        if constexpr (TAPS) {
          if (S.tap_u) *reinterpret_cast<float2*>(S.tap_u + off + 2 * e) = make_float2(u0, u1);
        }
        r[2 * e] = g[2 * e] * g0;
        r[2 * e + 1] = g[2 * e + 1] * g1;
      }
      *reinterpret_cast<uint4*>(S.out_u + off) = make_uint4(uo[0], uo[1], uo[2], uo[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = g[e];
    }
    if constexpr (TAPS) {
      if (S.tap_r) {
        float4* t4 = reinterpret_cast<float4*>(S.tap_r + off);
        t4[0] = make_float4(r[0], r[1], r[2], r[3]);
        t4[1] = make_float4(r[4], r[5], r[6], r[7]);
      }
    }
    if (r_bf16) {
      uint32_t ro[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 v = __floats2bfloat162_rn(r[2 * e], r[2 * e + 1]);
        ro[e] = *reinterpret_cast<uint32_t*>(&v);
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(S.out_r) + off) = make_uint4(ro[0], ro[1], ro[2], ro[3]);
    } else {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(S.out_r) + off);
      o[0] = make_float4(r[0], r[1], r[2], r[3]);
      o[1] = make_float4(r[4], r[5], r[6], r[7]);
    }
  }
}

// bf16 16-byte chunk -> fp16 (the towers' GEMMs run on fp16 operands, R27)
__device__ __forceinline__ uint4 bf16x8_to_f16x8(const uint4 u) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
  uint4 o;
  uint32_t* w = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(b[e]);
    const __half2 h = __floats2half2_rn(f.x, f.y);
    w[e] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return o;
}

__global__ void bf16_to_f16_kernel(const uint4* src, uint4* dst, size_t n8) {
  pdl_trigger();
  pdl_wait();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = bf16x8_to_f16x8(src[i]);
}

__global__ void gather_rows_kernel(const uint8_t* H, const int32_t* rows, int n, int T, int row_bytes, uint8_t* out,
                                   uint32_t* err, int to_f16) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  int src = rows[r];
  if (src < 0 || src >= T) {
    if (lane == 0) atomicOr(err, ERRBIT_OFFSETS);
    src = 0;
  }
  const uint4* s = reinterpret_cast<const uint4*>(H + (size_t)src * row_bytes);
  uint4* o = reinterpret_cast<uint4*>(out + (size_t)r * row_bytes);
  if (to_f16)
    for (int c = lane; c < row_bytes / 16; c += 32) o[c] = bf16x8_to_f16x8(s[c]);
  else
    for (int c = lane; c < row_bytes / 16; c += 32) o[c] = s[c];
}

__global__ void head_init_kernel(float* logits, const float* b2, int n, int K) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * K) logits[i] = b2[i % K];
}

// Routed BCE (Eq. 9): loss = sum softplus(z_k) - y z_k; dz = sigma(z_k) - y on the realised tower.
__global__ void head_dz_kernel(const float* logits, const int32_t* bucket, const float* label, int n, int K,
                               float* dz, float* loss_sum, float* db2, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float l = 0.f, g = 0.f;
  int k = 0;
  if (i < n) {
    k = bucket[i];
    if (k < 0 || k >= K) {
      atomicOr(err, ERRBIT_BUCKET);
      k = min(max(k, 0), K - 1);
    }
    const float z = logits[(size_t)i * K + k];
    const float y = label[i];
    l = fmaxf(z, 0.f) + log1pf(__expf(-fabsf(z))) - y * z;
    g = 1.f / (1.f + __expf(-z)) - y;
    if (!isfinite(l)) atomicOr(err, ERRBIT_NONFINITE);
    dz[i] = g;
  }
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(loss_sum, l);
  for (int kk = 0; kk < K; ++kk) {  // db2[k] = sum of dz over rows routed to tower k (warp-reduced)
    float gk = (i < n && k == kk) ? g : 0.f;
    for (int o = 16; o > 0; o >>= 1) gk += __shfl_xor_sync(0xffffffffu, gk, o);
    if ((threadIdx.x & 31) == 0 && gk != 0.f) atomicAdd(db2 + kk, gk);
  }
}

// dhid[i, c] = dz_i * w2[c] * 1[pre > 0] on the realised tower, 0 elsewhere (S:260 isolation);
// column sums db1[c] += dhid, dw2[c] += dz_i * relu(pre[i, c]).  Thread = 8 consecutive columns
// (one tower: dh % 8 == 0) with 16-byte accesses; block = 32 x 8 threads (256 columns x 8 row
// groups), rows strided over blockIdx.y.
__global__ void __launch_bounds__(256) head_dhid_kernel(const __nv_bfloat16* pre, const float* dz, const int32_t* bucket,
                                                        const float* w2, int n, int K, int dh, __nv_bfloat16* dhid,
                                                        __nv_bfloat16* dhid_lo, float* db1, float* dw2) {
  pdl_trigger();
  pdl_wait();
  const int N = K * dh;
  const int c0 = (blockIdx.x * 32 + threadIdx.x) * 8;
  float s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.f;
  if (c0 < N) {
    const int k = c0 / dh;
    float w[8];
    const float4 wa = *reinterpret_cast<const float4*>(w2 + c0), wb = *reinterpret_cast<const float4*>(w2 + c0 + 4);
    w[0] = wa.x, w[1] = wa.y, w[2] = wa.z, w[3] = wa.w, w[4] = wb.x, w[5] = wb.y, w[6] = wb.z, w[7] = wb.w;
    for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < n; i += gridDim.y * blockDim.y) {
      const int b = min(max(bucket[i], 0), K - 1);
      uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
      if (b == k) {
        const float z = dz[i];
        const uint4 pu = *reinterpret_cast<const uint4*>(pre + (size_t)i * N + c0);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pu);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 pr = __bfloat1622float2(p2[e]);
          const float g0 = pr.x > 0.f ? z * w[2 * e] : 0.f, g1 = pr.y > 0.f ? z * w[2 * e + 1] : 0.f;
          s1[2 * e] += g0;
          s1[2 * e + 1] += g1;
          s2[2 * e] += z * fmaxf(pr.x, 0.f);
          s2[2 * e + 1] += z * fmaxf(pr.y, 0.f);
          if (dhid_lo) {  // bf16 hi + lo split: the GEMM operand keeps ~16 bits (R27)
            const __nv_bfloat162 h = __floats2bfloat162_rn(g0, g1);
            const float2 hf = __bfloat1622float2(h);
            const __nv_bfloat162 l = __floats2bfloat162_rn(g0 - hf.x, g1 - hf.y);
            hi[e] = *reinterpret_cast<const uint32_t*>(&h);
            lo[e] = *reinterpret_cast<const uint32_t*>(&l);
          } else {        // one fp16 operand (11-bit mantissa; R27)
            const __half2 h = __floats2half2_rn(g0, g1);
            hi[e] = *reinterpret_cast<const uint32_t*>(&h);
          }
        }
      }
      *reinterpret_cast<uint4*>(dhid + (size_t)i * N + c0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      if (dhid_lo) *reinterpret_cast<uint4*>(dhid_lo + (size_t)i * N + c0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
  __shared__ float sh1[8][257], sh2[8][257];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    sh1[threadIdx.y][threadIdx.x * 8 + e] = s1[e];
    sh2[threadIdx.y][threadIdx.x * 8 + e] = s2[e];
  }
  __syncthreads();
  // 256 threads reduce the 256 columns over the 8 row groups
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int c = blockIdx.x * 256 + t;
  if (c < N) {
    float a = 0.f, b = 0.f;
    for (int y = 0; y < 8; ++y) {
      a += sh1[y][t];
      b += sh2[y][t];
    }
    atomicAdd(db1 + c, a);
    atomicAdd(dw2 + c, b);
  }
}

__global__ void add_bf16_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* out, size_t n2) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  float2 x = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(a)[i]);
  if (b) {
    const float2 y = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(b)[i]);
    x.x += y.x;
    x.y += y.y;
  }
  reinterpret_cast<__nv_bfloat162*>(out)[i] = __floats2bfloat162_rn(x.x, x.y);
}

// ---------------------------------------------------------------- launchers
static inline unsigned blocks(size_t n, unsigned b) { return (unsigned)((n + b - 1) / b); }

cudaError_t rope_apply_launch(const void* in, void* out, int T, int d, int hd, const RopeOTF& rp, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  const size_t pairs = (size_t)T * d / 2;
  if (pairs)
    launch_pdl(rope_apply_kernel, dim3(blocks(pairs, 256)), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(in),
                                                         reinterpret_cast<__nv_bfloat16*>(out), T, d, hd, rp);
  return cudaGetLastError();
}
cudaError_t rope_gate_bwd_launch2(const void* const* dr, const void* const* Xq, const void* const* Z,
                                  void* const* out_u, void* const* out_r, int nsides, int dr_f32, int r_bf16, int T,
                                  int d, int hd, const RopeOTF& rp, cudaStream_t st, float* const* tap_u,
                                  float* const* tap_r) {
  if (nsides < 1 || nsides > 2) return cudaErrorInvalidValue;
  RgSides sides;
  for (int i = 0; i < 2; ++i) {
    const int k = i < nsides ? i : 0;
    sides.s[i] = RgSide{dr[k], reinterpret_cast<const __nv_bfloat16*>(Xq[k]), reinterpret_cast<const __nv_bfloat16*>(Z[k]),
                        reinterpret_cast<__nv_bfloat16*>(out_u[k]), out_r[k], tap_u ? tap_u[k] : nullptr,
                        tap_r ? tap_r[k] : nullptr};
  }
  ProfScope ps(PROF_OTHER, st, 1);
  const size_t work = (size_t)T * d / 8;
  if (work)
    launch_pdl(((tap_u && (tap_u[0] || tap_u[nsides - 1])) || (tap_r && (tap_r[0] || tap_r[nsides - 1])))
                   ? rope_gate_bwd_kernel<true> : rope_gate_bwd_kernel<false>, dim3(blocks(work, 256)),
               dim3(256), 0, st, sides, nsides, dr_f32, r_bf16, T, d, hd, rp);
  return cudaGetLastError();
}
cudaError_t rope_gate_bwd_launch(const void* dr, int dr_f32, const void* Xq, const void* Z, void* out_u, void* out_r,
                                 int r_bf16, int T, int d, int hd, const RopeOTF& rp, cudaStream_t st) {
  return rope_gate_bwd_launch2(&dr, &Xq, &Z, &out_u, &out_r, 1, dr_f32, r_bf16, T, d, hd, rp, st);
}
cudaError_t gate_rope_fwd_launch(const void* Q, const void* K, const void* Gq, const void* Gk, const RopeOTF& rp,
                                 void* Qr, void* Kr, int T, int d, int hd, cudaStream_t st, float* tapQ,
                                 float* tapK) {
  ProfScope ps(PROF_OTHER, st, 1);
  const size_t work = (size_t)T * d / 8;
  if (work >= (size_t)INT32_MAX) return cudaErrorInvalidValue;
  if (work)
    launch_pdl(gate_rope_fwd_kernel, dim3(blocks(work, 256)), dim3(256), 0, st,
               reinterpret_cast<const __nv_bfloat16*>(Q), reinterpret_cast<const __nv_bfloat16*>(K),
               reinterpret_cast<const __nv_bfloat16*>(Gq), reinterpret_cast<const __nv_bfloat16*>(Gk), rp,
               reinterpret_cast<__nv_bfloat16*>(Qr), reinterpret_cast<__nv_bfloat16*>(Kr), T, d, hd, tapQ, tapK);
  return cudaGetLastError();
}
cudaError_t gather_rows_launch(const void* H, const int32_t* rows, int n, int T, int d, void* out, uint32_t* err,
                               cudaStream_t st, int to_f16) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0)
    launch_pdl(gather_rows_kernel, dim3(blocks(n, 8)), dim3(256), 0, st, reinterpret_cast<const uint8_t*>(H), rows, n,
               T, d * 2, reinterpret_cast<uint8_t*>(out), err, to_f16);
  return cudaGetLastError();
}
cudaError_t bf16_to_f16_launch(const void* src, void* dst, size_t n, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n % 8) return cudaErrorInvalidValue;
  if (n) {
    const size_t b = (n / 8 + 255) / 256;
    launch_pdl(bf16_to_f16_kernel, dim3((unsigned)(b > 1184 ? 1184 : b)), dim3(256), 0, st,
               reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n / 8);
  }
  return cudaGetLastError();
}
cudaError_t head_init_launch(float* logits, const float* b2, int n, int K, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0) launch_pdl(head_init_kernel, dim3(blocks((size_t)n * K, 256)), dim3(256), 0, st, logits, b2, n, K);
  return cudaGetLastError();
}
cudaError_t head_dz_launch(const float* logits, const int32_t* bucket, const float* label, int n, int K, float* dz,
                           float* loss_sum, float* db2, uint32_t* err, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0) launch_pdl(head_dz_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, logits, bucket, label, n, K, dz, loss_sum, db2, err);
  return cudaGetLastError();
}
cudaError_t head_dhid_launch(const void* pre, const float* dz, const int32_t* bucket, const float* w2, int n, int K,
                             int dh, void* dhid, void* dhid_lo, float* db1, float* dw2, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0) {
    dim3 blk(32, 8);
    dim3 grd((K * dh + 255) / 256, (unsigned)min(128, (n + 7) / 8));
    launch_pdl(head_dhid_kernel, dim3(grd), dim3(blk), 0, st, reinterpret_cast<const __nv_bfloat16*>(pre), dz, bucket, w2, n, K, dh,
                                          reinterpret_cast<__nv_bfloat16*>(dhid),
                                          reinterpret_cast<__nv_bfloat16*>(dhid_lo), db1, dw2);
  }
  return cudaGetLastError();
}
__global__ void slab_reduce_kernel(const float4* slabs, int nsplit, size_t n4, float4* out) {
  pdl_trigger();
  pdl_wait();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = slabs[i];
    for (int s = 1; s < nsplit; ++s) {
      const float4 b = slabs[(size_t)s * n4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    out[i] = a;
  }
}
cudaError_t slab_reduce_launch(const float* slabs, int nsplit, size_t n, float* out, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n % 4 || nsplit < 1) return cudaErrorInvalidValue;
  if (n)
    launch_pdl(slab_reduce_kernel, dim3((unsigned)std::min<size_t>(blocks(n / 4, 256), 148 * 8)), dim3(256), 0, st,
               reinterpret_cast<const float4*>(slabs), nsplit, n / 4, reinterpret_cast<float4*>(out));
  return cudaGetLastError();
}
// context buckets: bucket = #{j : pos > boundary_j}; pos < 1 is a routing error
__global__ void bucketize_kernel(const int32_t* pos, int n, Bounds bd, int32_t* out, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = pos[i];
  int k = 0;
  if (p < 1) {
    atomicOr(err, ERRBIT_BUCKET);
  } else {
    for (int j = 0; j < bd.nb; ++j) k += p > bd.b[j] ? 1 : 0;
  }
  out[i] = k;
}
cudaError_t bucketize_launch(const int32_t* pos, int n, const Bounds& bd, int32_t* out, uint32_t* err,
                             cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0) launch_pdl(bucketize_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, pos, n, bd, out, err);
  return cudaGetLastError();
}
cudaError_t add_bf16_launch(const void* a, const void* b, void* out, size_t n, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (n)
    launch_pdl(add_bf16_kernel, dim3(blocks(n / 2, 256)), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(a),
                                                         reinterpret_cast<const __nv_bfloat16*>(b),
                                                         reinterpret_cast<__nv_bfloat16*>(out), n / 2);
  return cudaGetLastError();
}


struct ZeroSpans {
  void* p[8];
  unsigned long long n[8];
  int count;
};
__global__ void __launch_bounds__(256) zero_many_kernel(ZeroSpans z) {
  pdl_trigger();
  pdl_wait();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int s = 0; s < z.count; ++s) {
    uint4* q = reinterpret_cast<uint4*>(z.p[s]);
    const size_t n16 = (reinterpret_cast<uintptr_t>(z.p[s]) & 15) ? 0 : z.n[s] / 16;  // unaligned: bytewise
    for (size_t i = tid; i < n16; i += stride) q[i] = make_uint4(0u, 0u, 0u, 0u);
    for (size_t i = n16 * 16 + tid; i < z.n[s]; i += stride) reinterpret_cast<uint8_t*>(z.p[s])[i] = 0;
  }
}
cudaError_t zero_many_launch(const ZeroSpan* spans, int n, cudaStream_t st) {
  ZeroSpans z;
  z.count = 0;
  size_t total = 0;
  for (int i = 0; i < n && z.count < 8; ++i) {
    if (!spans[i].ptr || !spans[i].bytes) continue;
    z.p[z.count] = spans[i].ptr;
    z.n[z.count] = spans[i].bytes;
    total += spans[i].bytes;
    ++z.count;
  }
  if (z.count == 0) return cudaSuccess;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const size_t b = (total / 16 + 255) / 256;
  const int grid = (int)(b < 1 ? 1 : (b > (size_t)4 * sms ? (size_t)4 * sms : b));
  ProfScope ps(PROF_OTHER, st, 1);
  launch_pdl(zero_many_kernel, dim3(grid), dim3(256), 0, st, z);
  return cudaGetLastError();
}

}  // namespace cadet
