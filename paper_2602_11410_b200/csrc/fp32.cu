// CADET_FP32 parity mode (north star: "1e-4 for an fp32 mode"; SURVEY 8(c) protocol ii): the whole
// gated layer (A2-A12, Eqs. 3-7), the attention core and the towers (Eqs. 8-9)
// on fp32 tensors end to end.
//
//  * every projection / gradient GEMM is a 3xTF32 tcgen05 GEMM: each fp32 operand x is split once
//    into hi = tf32(x) and lo = x - hi (split_tf32_kernel, which also lays every operand out K-major),
//    and C = A_hi B_hi + A_hi B_lo + A_lo B_hi runs as ONE 3-segment kind::tf32 accumulation in TMEM
//    (gemm.cu), relative error ~2^-21 per product instead of 2^-8 for bf16 operands;
//  * gates, RoPE (angles in fp64 from int64 rebased times) and their adjoints are exact fp32
//    elementwise kernels (expf, fp64 sincos);
//  * the attention core runs in fp32 FMA arithmetic (warp per query row / key row, online softmax,
//    the plan's per-row visible prefix + diagonal + PAIR_PREV cell; fully masked keys never visited):
//    P and dS stay fp32 instead of becoming MMA operands.
// Parity / validation mode only: performance is not a goal here (the bf16 path is the product).
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>

#include "../../include/cadet.h"
#include "fp32.cuh"
#include "gemm.cuh"
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {

namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
inline unsigned nblk(size_t n, int b) { return (unsigned)((n + b - 1) / b); }
__device__ __forceinline__ float sig_exact(float z) { return 1.0f / (1.0f + expf(-z)); }
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
}  // namespace

// ------------------------------------------------------------------ 3xTF32 operand split
// src [rows][cols] fp32 (row stride ld_src) -> hi, lo with hi = tf32 round-to-nearest(x), lo = x - hi
// (exact), stored [rows][ldo] (trans = 0) or [cols][ldo] (trans = 1); 32 x 32 tiles through smem.
__global__ void split_tf32_kernel(const float* __restrict__ src, int rows, int cols, int ld_src, int trans,
                                  float* __restrict__ hi, float* __restrict__ lo, int ldo) {
  pdl_trigger();
  pdl_wait();
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;
    tile[k][tx] = (r < rows && c < cols) ? src[(size_t)r * ld_src + c] : 0.f;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    float x;
    int orow, ocol;
    if (!trans) {
      x = tile[k][tx];
      orow = r0 + k;
      ocol = c0 + tx;
      if (orow >= rows || ocol >= cols) continue;
    } else {
      x = tile[tx][k];
      orow = c0 + k;
      ocol = r0 + tx;
      if (orow >= cols || ocol >= rows) continue;
    }
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    const float hf = __uint_as_float(h);
    hi[(size_t)orow * ldo + ocol] = hf;
    lo[(size_t)orow * ldo + ocol] = x - hf;
  }
}

size_t gemm3x_scratch_bytes(int M, int N, int K) {
  const size_t kp = (size_t)(K + 3) / 4 * 4;
  return 2 * a256((size_t)M * kp * 4) + 2 * a256((size_t)N * kp * 4);
}

__global__ void fill_rows_f32_kernel(float* C, const float* src, size_t n) {  // C = src (or 0)
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) C[i] = src ? src[i] : 0.f;
}

// C[M, N] (+)= op(A) op(B): C = op(A) op(B) + resid (resid may be null, or C itself to accumulate),
// op(A) [M, K] = A stored [M][K] (or [K][M] if a_t), op(B) [K, N] = B stored [K][N] (or [N][K] if b_t:
// the g W^T case); C row-major [M][N].  scratch >= gemm3x_scratch_bytes(M, N, K).
// Accuracy: the tensor cores' fp32 accumulation truncates (measured: biased toward zero, ~2^-23 of the
// running sum per MMA instruction once the products carry 22 significant bits), so one TMEM
// accumulator over K = 1024 in three segments (384 instructions) drifts ~1e-5 relative.  Each unit
// therefore accumulates at most 4 k-blocks (16 instructions) and the partial sums are added into C with
// fp32 atomics (round to nearest): ~1e-6 relative at K = 1024.
cudaError_t gemm3x(int M, int N, int K, const float* A, int a_t, const float* B, int b_t, float* C,
                   const float* resid, void* scratch, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const size_t MN = (size_t)M * N;
  cudaError_t e = cudaSuccess;
  if (resid != C) {
    ProfScope ps(PROF_OTHER, st, 1);
    e = launch_pdl(fill_rows_f32_kernel, dim3(nblk(MN, 256)), dim3(256), 0, st, C, resid, MN);
  }
  if (K <= 0 || e != cudaSuccess) return e;
  const int kp = (K + 3) / 4 * 4;
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  float* Ah = reinterpret_cast<float*>(p);
  p += a256((size_t)M * kp * 4);
  float* Al = reinterpret_cast<float*>(p);
  p += a256((size_t)M * kp * 4);
  float* Bh = reinterpret_cast<float*>(p);
  p += a256((size_t)N * kp * 4);
  float* Bl = reinterpret_cast<float*>(p);
  {
    ProfScope ps(PROF_OTHER, st, 2);
    // A -> [M][kp]: stored [M][K] (no transpose) or [K][M] (transpose)
    const int ar = a_t ? K : M, ac = a_t ? M : K;
    e = launch_pdl(split_tf32_kernel, dim3(nblk(ac, 32), nblk(ar, 32)), dim3(256), 0, st, A, ar, ac, ac, a_t, Ah, Al,
                   kp);
    // B -> [N][kp]: stored [N][K] (b_t: no transpose) or [K][N] (transpose)
    const int br = b_t ? N : K, bc = b_t ? K : N;
    if (e == cudaSuccess)
      e = launch_pdl(split_tf32_kernel, dim3(nblk(bc, 32), nblk(br, 32)), dim3(256), 0, st, B, br, bc, bc, b_t ? 0 : 1,
                     Bh, Bl, kp);
    if (e != cudaSuccess) return e;
  }
  GemmProblem g;
  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.nseg = 3;
  g.tf32 = 1;
  const float* as[3] = {Ah, Ah, Al};
  const float* bs[3] = {Bh, Bl, Bh};
  for (int s = 0; s < 3; ++s) {
    g.K[s] = K;
    g.A[s] = OperandDesc{as[s], M, K, 0, kp};
    g.B[s] = OperandDesc{bs[s], N, K, 0, kp};
  }
  const int kb_total = 3 * ((K + 31) / 32);
  g.split_k = (kb_total + 3) / 4;
  g.epi.mode = EPI_ATOMIC;
  g.epi.out = C;
  g.epi.out_f32 = 1;
  g.epi.ldo = N;
  return gemm_launch(&g, 1, 128, st);
}

// ------------------------------------------------------------------ elementwise (exact fp32)
// RoPE angle of (row, pair i): alpha = (t_row - t_seqstart) theta_i, theta_i = (phi_min / dt_max)
// base^(2i / hd) (R5), fp64 throughout (R21: int64 rebasing keeps it shift invariant)
struct RopeK {
  const int64_t* t;
  const int32_t* row_seq;
  const int32_t* cu;
  double phi_min, base, dt_max;
  int on;
};
__device__ __forceinline__ void rope_cs64(const RopeK& r, int row, int i, int hd, float& c, float& s) {
  if (!r.on) {
    c = 1.f;
    s = 0.f;
    return;
  }
  const int sq = r.row_seq[row];
  const double dt = sq >= 0 ? (double)(r.t[row] - r.t[r.cu[sq]]) : 0.0;
  const double th = (r.phi_min / r.dt_max) * pow(r.base, 2.0 * i / (double)hd);
  double sn, cs;
  sincos(dt * th, &sn, &cs);
  c = (float)cs;
  s = (float)sn;
}

// out = x * sigma(z)   (Eq. 4 / Eq. 5 gates)
__global__ void gate_f32_kernel(const float* x, const float* z, float* out, size_t n) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i] * sig_exact(z[i]);
}
// Qr = RoPE(Q * sigma(Z)) (z null: no gate), thread per (row, adjacent pair) (R3, R4)
__global__ void gate_rope_f32_kernel(const float* x, const float* z, float* out, int T, int d, int hd, RopeK rk) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)T * d / 2) return;
  const int row = (int)(idx / (d / 2)), c = (int)(idx % (d / 2)) * 2;
  const size_t o = (size_t)row * d + c;
  float a = x[o], b = x[o + 1];
  if (z) {
    a *= sig_exact(z[o]);
    b *= sig_exact(z[o + 1]);
  }
  float cs, sn;
  rope_cs64(rk, row, (c % hd) / 2, hd, cs, sn);
  out[o] = a * cs - b * sn;
  out[o + 1] = a * sn + b * cs;
}
// A11: dT = R(-alpha) dr; with the gate: u = dT * x * g (1 - g), r = dT * g (g = sigma(z)); else r = dT
__global__ void rope_gate_bwd_f32_kernel(const float* dr, const float* x, const float* z, float* u, float* r, int T,
                                         int d, int hd, RopeK rk) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)T * d / 2) return;
  const int row = (int)(idx / (d / 2)), c = (int)(idx % (d / 2)) * 2;
  const size_t o = (size_t)row * d + c;
  float cs, sn;
  rope_cs64(rk, row, (c % hd) / 2, hd, cs, sn);
  const float g0 = dr[o] * cs + dr[o + 1] * sn, g1 = dr[o + 1] * cs - dr[o] * sn;
  if (z) {
    const float s0 = sig_exact(z[o]), s1 = sig_exact(z[o + 1]);
    u[o] = g0 * x[o] * s0 * (1.f - s0);
    u[o + 1] = g1 * x[o + 1] * s1 * (1.f - s1);
    r[o] = g0 * s0;
    r[o + 1] = g1 * s1;
  } else {
    r[o] = g0;
    r[o + 1] = g1;
  }
}
// A12: u = dXt * X * g (1 - g), r = dXt * g (+ dresid), g = sigma(Zx)
__global__ void gate_bwd_f32_kernel(const float* dxt, const float* x, const float* z, const float* dres, float* u,
                                    float* r, size_t n) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float g = sig_exact(z[i]);
  u[i] = dxt[i] * x[i] * g * (1.f - g);
  r[i] = dxt[i] * g + (dres ? dres[i] : 0.f);
}
__global__ void add_f32_kernel(const float* a, const float* b, float* out, size_t n) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + (b ? b[i] : 0.f);
}
// D[h][i] = sum_k dO[i][h hd + k] O[i][h hd + k]   (A10 preprocess)
__global__ void rowdot_f32_kernel(const float* dO, const float* O, float* D, int T, int H, int hd) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)T * H) return;
  const int row = (int)(idx / H), h = (int)(idx % H);
  const float* a = dO + (size_t)row * H * hd + h * hd;
  const float* b = O + (size_t)row * H * hd + h * hd;
  float s = 0.f;
  for (int k = 0; k < hd; ++k) s = fmaf(a[k], b[k], s);
  D[(size_t)h * T + row] = s;
}

// ------------------------------------------------------------------ attention core, fp32 (Eq. 7)
// Visible keys of real row i of sequence s (global indices, the plan's exact encoding of the mask,
// DESIGN R24): the prefix [cu[s], kv_end[i]), then i - 1 if the row's PAIR_PREV bit is set and i - 1
// lies past the prefix, then the diagonal i (R8).
struct F32Attn {
  const float *Q, *K, *V, *O, *dO, *lse, *D;
  float *Oout, *lse_out, *dQ, *dK, *dV;
  const int32_t *kv_end, *row_seq, *cu;
  const uint8_t* row_pp;
  int T, H, hd;
  float scale;
};
struct RowKeys {
  int a, npre, pp, i, n;
};
__device__ __forceinline__ RowKeys row_keys(const F32Attn& p, int i) {
  RowKeys r;
  const int s = p.row_seq[i];
  r.a = p.cu[s];
  const int ke = p.kv_end[i];
  r.npre = max(ke - r.a, 0);
  r.pp = (p.row_pp[i] && i - 1 >= ke && i - 1 >= r.a) ? 1 : 0;
  r.i = i;
  r.n = r.npre + r.pp + 1;
  return r;
}
__device__ __forceinline__ int key_at(const RowKeys& r, int idx) {
  return idx < r.npre ? r.a + idx : ((idx == r.npre && r.pp) ? r.i - 1 : r.i);
}
__device__ __forceinline__ bool visible(const F32Attn& p, int i, int j) {
  return j < p.kv_end[i] || i == j || (p.row_pp[i] && j == i - 1);
}
__device__ __forceinline__ float dot_row(const float* a_smem, const float* b, int hd) {
  float s = 0.f;
  for (int k = 0; k < hd; k += 4) {
    const float4 v = *reinterpret_cast<const float4*>(b + k);
    s = fmaf(a_smem[k], v.x, s);
    s = fmaf(a_smem[k + 1], v.y, s);
    s = fmaf(a_smem[k + 2], v.z, s);
    s = fmaf(a_smem[k + 3], v.w, s);
  }
  return s;
}

// forward: warp per (query row, head); lanes score 32 keys at a time; lane owns output dims lane + 32 c
__global__ void __launch_bounds__(128) attn_fwd_f32_kernel(F32Attn p) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) float qs[4][128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + w, h = blockIdx.y, hd = p.hd, d = p.H * hd;
  if (i >= p.T) return;
  float* Orow = p.Oout + (size_t)i * d + h * hd;
  if (p.row_seq[i] < 0) {  // pad row: O = 0, LSE = 0 (R17)
    for (int c = lane; c < hd; c += 32) Orow[c] = 0.f;
    if (lane == 0) p.lse_out[(size_t)h * p.T + i] = 0.f;
    return;
  }
  for (int c = lane; c < hd; c += 32) qs[w][c] = p.Q[(size_t)i * d + h * hd + c];
  __syncwarp();
  const RowKeys rk = row_keys(p, i);
  float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < rk.n; base += 32) {
    const int idx = base + lane;
    const bool ok = idx < rk.n;
    const int j = ok ? key_at(rk, idx) : i;
    const float sc = ok ? dot_row(qs[w], p.K + (size_t)j * d + h * hd, hd) * p.scale : -INFINITY;
    const float mn = fmaxf(m, warp_max(sc));
    const float pr = ok ? expf(sc - mn) : 0.f;
    const float corr = expf(m - mn);
    l = l * corr + warp_sum(pr);
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] *= corr;
    const int cnt = min(32, rk.n - base);
    for (int jj = 0; jj < cnt; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, pr, jj);
      const int kj = __shfl_sync(0xffffffffu, j, jj);
      const float* vr = p.V + (size_t)kj * d + h * hd;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane + 32 * c < hd) o[c] = fmaf(pj, vr[lane + 32 * c], o[c]);
    }
    m = mn;
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (lane + 32 * c < hd) Orow[lane + 32 * c] = o[c] * inv;
  if (lane == 0) p.lse_out[(size_t)h * p.T + i] = m + logf(l);
}

// backward dQ: warp per (query row, head): dS_ij = P_ij (dO_i . V_j - D_i); dQ_i = scale sum_j dS_ij K_j
__global__ void __launch_bounds__(128) attn_bwd_dq_f32_kernel(F32Attn p) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) float qs[4][128];
  __shared__ __align__(16) float gs[4][128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + w, h = blockIdx.y, hd = p.hd, d = p.H * hd;
  if (i >= p.T) return;
  float* out = p.dQ + (size_t)i * d + h * hd;
  if (p.row_seq[i] < 0) {
    for (int c = lane; c < hd; c += 32) out[c] = 0.f;
    return;
  }
  for (int c = lane; c < hd; c += 32) {
    qs[w][c] = p.Q[(size_t)i * d + h * hd + c];
    gs[w][c] = p.dO[(size_t)i * d + h * hd + c];
  }
  __syncwarp();
  const RowKeys rk = row_keys(p, i);
  const float L = p.lse[(size_t)h * p.T + i], Di = p.D[(size_t)h * p.T + i];
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < rk.n; base += 32) {
    const int idx = base + lane;
    const bool ok = idx < rk.n;
    const int j = ok ? key_at(rk, idx) : i;
    float ds = 0.f;
    if (ok) {
      const float pr = expf(dot_row(qs[w], p.K + (size_t)j * d + h * hd, hd) * p.scale - L);
      ds = pr * (dot_row(gs[w], p.V + (size_t)j * d + h * hd, hd) - Di);
    }
    const int cnt = min(32, rk.n - base);
    for (int jj = 0; jj < cnt; ++jj) {
      const float dj = __shfl_sync(0xffffffffu, ds, jj);
      const int kj = __shfl_sync(0xffffffffu, j, jj);
      const float* kr = p.K + (size_t)kj * d + h * hd;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane + 32 * c < hd) acc[c] = fmaf(dj, kr[lane + 32 * c], acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (lane + 32 * c < hd) out[lane + 32 * c] = acc[c] * p.scale;
}

// backward dK, dV: warp per (key row j, head), scanning the rows i >= j of its sequence that see j
// (no atomics: each dK_j / dV_j row is written once)
__global__ void __launch_bounds__(128) attn_bwd_dkv_f32_kernel(F32Attn p) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) float ks[4][128];
  __shared__ __align__(16) float vs[4][128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + w, h = blockIdx.y, hd = p.hd, d = p.H * hd;
  if (j >= p.T) return;
  float* dk = p.dK + (size_t)j * d + h * hd;
  float* dv = p.dV + (size_t)j * d + h * hd;
  const int s = p.row_seq[j];
  if (s < 0) {
    for (int c = lane; c < hd; c += 32) dk[c] = dv[c] = 0.f;
    return;
  }
  for (int c = lane; c < hd; c += 32) {
    ks[w][c] = p.K[(size_t)j * d + h * hd + c];
    vs[w][c] = p.V[(size_t)j * d + h * hd + c];
  }
  __syncwarp();
  const int e = p.cu[s + 1];
  float ak[4] = {0.f, 0.f, 0.f, 0.f}, av[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i0 = j; i0 < e; i0 += 32) {
    const int i = i0 + lane;
    float pr = 0.f, ds = 0.f;
    if (i < e && visible(p, i, j)) {
      pr = expf(dot_row(ks[w], p.Q + (size_t)i * d + h * hd, hd) * p.scale - p.lse[(size_t)h * p.T + i]);
      ds = pr * (dot_row(vs[w], p.dO + (size_t)i * d + h * hd, hd) - p.D[(size_t)h * p.T + i]);
    }
    const int cnt = min(32, e - i0);
    for (int ii = 0; ii < cnt; ++ii) {
      const float pi = __shfl_sync(0xffffffffu, pr, ii), di = __shfl_sync(0xffffffffu, ds, ii);
      if (pi == 0.f && di == 0.f) continue;  // warp-uniform: masked row
      const float* qr = p.Q + (size_t)(i0 + ii) * d + h * hd;
      const float* gr = p.dO + (size_t)(i0 + ii) * d + h * hd;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane + 32 * c < hd) {
          ak[c] = fmaf(di, qr[lane + 32 * c], ak[c]);
          av[c] = fmaf(pi, gr[lane + 32 * c], av[c]);
        }
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (lane + 32 * c < hd) {
      dk[lane + 32 * c] = ak[c] * p.scale;
      dv[lane + 32 * c] = av[c];
    }
}

static F32Attn f32attn(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v) {
  F32Attn p;
  memset(&p, 0, sizeof(p));
  p.kv_end = v.kv_end;
  p.row_seq = v.row_seq;
  p.row_pp = v.row_pp;
  p.cu = b->cu_seqlens;
  p.T = b->total_tokens;
  p.H = c->n_heads;
  p.hd = c->head_dim;
  p.scale = (float)(1.0 / sqrt((double)c->head_dim));
  return p;
}

cudaError_t attn_fwd_f32(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v, const float* Qr,
                         const float* Kr, const float* V, float* O, float* lse, cudaStream_t st) {
  F32Attn p = f32attn(c, b, v);
  p.Q = Qr;
  p.K = Kr;
  p.V = V;
  p.Oout = O;
  p.lse_out = lse;
  if (p.T == 0) return cudaSuccess;
  ProfScope ps(PROF_ATTN_FWD, st, 1);
  return launch_pdl(attn_fwd_f32_kernel, dim3(nblk(p.T, 4), p.H), dim3(128), 0, st, p);
}

cudaError_t attn_bwd_f32(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v, const float* Qr,
                         const float* Kr, const float* V, const float* O, const float* lse, const float* dO, float* D,
                         float* dQ, float* dK, float* dV, cudaStream_t st) {
  F32Attn p = f32attn(c, b, v);
  p.Q = Qr;
  p.K = Kr;
  p.V = V;
  p.O = O;
  p.lse = lse;
  p.dO = dO;
  p.D = D;
  p.dQ = dQ;
  p.dK = dK;
  p.dV = dV;
  if (p.T == 0) return cudaSuccess;
  ProfScope ps(PROF_ATTN_BWD, st, 3);
  cudaError_t e = launch_pdl(rowdot_f32_kernel, dim3(nblk((size_t)p.T * p.H, 256)), dim3(256), 0, st, dO, O, D, p.T,
                             p.H, p.hd);
  if (e == cudaSuccess) e = launch_pdl(attn_bwd_dq_f32_kernel, dim3(nblk(p.T, 4), p.H), dim3(128), 0, st, p);
  if (e == cudaSuccess) e = launch_pdl(attn_bwd_dkv_f32_kernel, dim3(nblk(p.T, 4), p.H), dim3(128), 0, st, p);
  return e;
}

// ------------------------------------------------------------------ the gated layer in fp32
static RopeK ropek(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v) {
  RopeK r;
  r.t = b->timestamps_ms;
  r.row_seq = v.row_seq;
  r.cu = b->cu_seqlens;
  r.phi_min = c->rope_phi_min;
  r.base = c->rope_base;
  r.dt_max = (double)c->rope_delta_t_max_ms;
  r.on = c->use_rope;
  return r;
}

static size_t fsz(int T, int d) { return a256((size_t)T * d * 4); }

size_t f32_saved_bytes(const cadet_attn_config* c, int T) {
  return 10 * fsz(T, c->d_model) + a256((size_t)4 * c->n_heads * T);
}
// plan | D [H, T] | 13 fp32 [T, d] backward temporaries | 3xTF32 split scratch
size_t f32_layer_ws_bytes(const cadet_attn_config* c, int n, int T) {
  const int d = c->d_model;
  const size_t scratch = std::max(gemm3x_scratch_bytes(T, d, d), gemm3x_scratch_bytes(d, d, T));
  return plan_bytes(n, T, T) + a256((size_t)4 * c->n_heads * T) + 13 * fsz(T, d) + scratch;
}

struct F32Saved {
  float *Zx, *Xt, *Q, *K, *Zq, *Zk, *Qr, *Kr, *V, *O, *lse;
};
static F32Saved carve_saved_f32(void* saved, const cadet_attn_config* c, int T) {
  uint8_t* p = reinterpret_cast<uint8_t*>(saved);
  F32Saved S;
  float** sl[10] = {&S.Zx, &S.Xt, &S.Q, &S.K, &S.Zq, &S.Zk, &S.Qr, &S.Kr, &S.V, &S.O};
  for (int i = 0; i < 10; ++i) *sl[i] = reinterpret_cast<float*>(p + i * fsz(T, c->d_model));
  S.lse = reinterpret_cast<float*>(p + 10 * fsz(T, c->d_model));
  return S;
}
struct F32Ws {
  float* D;
  float *dO, *dQr, *dKr, *dV, *uq, *rq, *uk, *rk, *dQ, *dK, *dXt, *ux, *rx;
  void* scratch;
};
static F32Ws carve_ws_f32(void* ws, const cadet_attn_config* c, int n, int T) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws) + plan_bytes(n, T, T);
  F32Ws W;
  W.D = reinterpret_cast<float*>(p);
  p += a256((size_t)4 * c->n_heads * T);
  float** sl[13] = {&W.dO, &W.dQr, &W.dKr, &W.dV, &W.uq, &W.rq, &W.uk, &W.rk, &W.dQ, &W.dK, &W.dXt, &W.ux, &W.rx};
  for (int i = 0; i < 13; ++i) {
    *sl[i] = reinterpret_cast<float*>(p);
    p += fsz(T, c->d_model);
  }
  W.scratch = p;
  return W;
}

cudaError_t layer_forward_f32(const cadet_attn_config* c, const cadet_batch* b, const cadet_attn_weights* w,
                              const float* X, float* Y, const float* resid, void* saved, void* ws, cudaStream_t st) {
  const int T = b->total_tokens, d = c->d_model, n = b->n_seqs, hd = c->head_dim;
  const size_t N = (size_t)T * d;
  PlanView v = plan_carve(ws, n, T, T);
  F32Saved S = carve_saved_f32(saved, c, T);
  F32Ws W = carve_ws_f32(ws, c, n, T);
  const RopeK rk = ropek(c, b, v);
  cudaError_t e = cudaSuccess;
  // A2 (Eq. 4): Xt = X * sigma(X W_xg)
  const float* Xt = X;
  if (c->use_rep_gate) {
    e = gemm3x(T, d, d, X, 0, (const float*)w->W_xg, 0, S.Zx, nullptr, W.scratch, st);
    if (e == cudaSuccess) e = launch_pdl(gate_f32_kernel, dim3(nblk(N, 256)), dim3(256), 0, st, X, (const float*)S.Zx, S.Xt, N);
    Xt = S.Xt;
  } else {
    e = cudaMemcpyAsync(S.Xt, X, N * 4, cudaMemcpyDeviceToDevice, st);
  }
  // A3 (Eq. 3; R2)
  const void* Wqkv[3] = {w->W_q, w->W_k, w->W_v};
  float* qkv[3] = {S.Q, S.K, S.V};
  for (int i = 0; i < 3 && e == cudaSuccess; ++i)
    e = gemm3x(T, d, d, Xt, 0, (const float*)Wqkv[i], 0, qkv[i], nullptr, W.scratch, st);
  // A4 (Eq. 5 + RoPE P:274)
  if (c->use_int_gate) {
    if (e == cudaSuccess) e = gemm3x(T, d, d, S.Q, 0, (const float*)w->W_qg, 0, S.Zq, nullptr, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(T, d, d, S.K, 0, (const float*)w->W_kg, 0, S.Zk, nullptr, W.scratch, st);
  }
  if (e == cudaSuccess)
    e = launch_pdl(gate_rope_f32_kernel, dim3(nblk(N / 2, 256)), dim3(256), 0, st, (const float*)S.Q,
                   (const float*)(c->use_int_gate ? S.Zq : nullptr), S.Qr, T, d, hd, rk);
  if (e == cudaSuccess)
    e = launch_pdl(gate_rope_f32_kernel, dim3(nblk(N / 2, 256)), dim3(256), 0, st, (const float*)S.K,
                   (const float*)(c->use_int_gate ? S.Zk : nullptr), S.Kr, T, d, hd, rk);
  // A5 (Eq. 7)
  if (e == cudaSuccess) e = attn_fwd_f32(c, b, v, S.Qr, S.Kr, S.V, S.O, S.lse, st);
  // A6
  if (e == cudaSuccess) {
    if (c->use_out_proj)
      e = gemm3x(T, d, d, S.O, 0, (const float*)w->W_o, 0, Y, resid, W.scratch, st);
    else
      e = launch_pdl(add_f32_kernel, dim3(nblk(N, 256)), dim3(256), 0, st, (const float*)S.O, resid, Y, N);
  }
  if (e == cudaSuccess) e = zero_pad_rows_launch(Y, d * 4, T, b->cu_seqlens, n, st);
  return e;
}

cudaError_t layer_backward_f32(const cadet_attn_config* c, const cadet_batch* b, const cadet_attn_weights* w,
                               const float* X, const void* saved, const float* dY, float* dX, const float* dresid,
                               const cadet_attn_grads* g, void* ws, cudaStream_t st, void* const* grad_events) {
  const int T = b->total_tokens, d = c->d_model, n = b->n_seqs, hd = c->head_dim;
  const size_t N = (size_t)T * d;
  PlanView v = plan_carve(ws, n, T, T);
  F32Saved S = carve_saved_f32(const_cast<void*>(saved), c, T);
  F32Ws W = carve_ws_f32(ws, c, n, T);
  const RopeK rk = ropek(c, b, v);
  cudaError_t e = cudaSuccess;
  auto mark = [&](int i) {
    if (e == cudaSuccess && grad_events && grad_events[i]) e = cudaEventRecord((cudaEvent_t)grad_events[i], st);
  };
  const size_t wb = (size_t)d * d * 4;
  float* gws[7] = {g->dW_xg, g->dW_q, g->dW_k, g->dW_v, g->dW_qg, g->dW_kg, g->dW_o};
  for (int i = 0; i < 7 && e == cudaSuccess; ++i)  // ablated groups are reported as zero
    if (gws[i]) e = cudaMemsetAsync(gws[i], 0, wb, st);
  // A9: dO = dY W_o^T ; dW_o = O^T dY
  const float* dO = dY;
  if (c->use_out_proj && e == cudaSuccess) {
    e = gemm3x(T, d, d, dY, 0, (const float*)w->W_o, 1, W.dO, nullptr, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(d, d, T, S.O, 1, dY, 0, g->dW_o, nullptr, W.scratch, st);
    dO = W.dO;
  }
  mark(0);
  // A10
  if (e == cudaSuccess) e = attn_bwd_f32(c, b, v, S.Qr, S.Kr, S.V, S.O, S.lse, dO, W.D, W.dQr, W.dKr, W.dV, st);
  // A11: R(-alpha) + interaction-gate backward
  const float* dQ = W.rq;
  const float* dK = W.rk;
  const int ig = c->use_int_gate;
  if (e == cudaSuccess)
    e = launch_pdl(rope_gate_bwd_f32_kernel, dim3(nblk(N / 2, 256)), dim3(256), 0, st, (const float*)W.dQr,
                   (const float*)S.Q, (const float*)(ig ? S.Zq : nullptr), W.uq, W.rq, T, d, hd, rk);
  if (e == cudaSuccess)
    e = launch_pdl(rope_gate_bwd_f32_kernel, dim3(nblk(N / 2, 256)), dim3(256), 0, st, (const float*)W.dKr,
                   (const float*)S.K, (const float*)(ig ? S.Zk : nullptr), W.uk, W.rk, T, d, hd, rk);
  if (ig) {
    if (e == cudaSuccess) e = gemm3x(T, d, d, W.uq, 0, (const float*)w->W_qg, 1, W.dQ, W.rq, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(T, d, d, W.uk, 0, (const float*)w->W_kg, 1, W.dK, W.rk, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(d, d, T, S.Q, 1, W.uq, 0, g->dW_qg, nullptr, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(d, d, T, S.K, 1, W.uk, 0, g->dW_kg, nullptr, W.scratch, st);
    dQ = W.dQ;
    dK = W.dK;
  }
  mark(1);
  // A12: dXt = dQ W_q^T + dK W_k^T + dV W_v^T ; dW_{q,k,v} = Xt^T d{Q,K,V}
  const float* Xt = S.Xt;
  if (e == cudaSuccess) e = gemm3x(T, d, d, dQ, 0, (const float*)w->W_q, 1, W.dXt, nullptr, W.scratch, st);
  if (e == cudaSuccess) e = gemm3x(T, d, d, dK, 0, (const float*)w->W_k, 1, W.dXt, W.dXt, W.scratch, st);
  if (e == cudaSuccess) e = gemm3x(T, d, d, W.dV, 0, (const float*)w->W_v, 1, W.dXt, W.dXt, W.scratch, st);
  if (e == cudaSuccess) e = gemm3x(d, d, T, Xt, 1, dQ, 0, g->dW_q, nullptr, W.scratch, st);
  if (e == cudaSuccess) e = gemm3x(d, d, T, Xt, 1, dK, 0, g->dW_k, nullptr, W.scratch, st);
  if (e == cudaSuccess) e = gemm3x(d, d, T, Xt, 1, W.dV, 0, g->dW_v, nullptr, W.scratch, st);
  mark(2);
  if (c->use_rep_gate) {  // u_x = dXt X g (1 - g), r_x = dXt g (+ dresid); dX = r_x + u_x W_xg^T; dW_xg = X^T u_x
    if (e == cudaSuccess)
      e = launch_pdl(gate_bwd_f32_kernel, dim3(nblk(N, 256)), dim3(256), 0, st, (const float*)W.dXt, X,
                     (const float*)S.Zx, dresid, W.ux, W.rx, N);
    if (e == cudaSuccess) e = gemm3x(T, d, d, W.ux, 0, (const float*)w->W_xg, 1, dX, W.rx, W.scratch, st);
    if (e == cudaSuccess) e = gemm3x(d, d, T, X, 1, W.ux, 0, g->dW_xg, nullptr, W.scratch, st);
  } else if (e == cudaSuccess) {
    e = launch_pdl(add_f32_kernel, dim3(nblk(N, 256)), dim3(256), 0, st, (const float*)W.dXt, dresid, dX, N);
  }
  mark(3);
  if (e == cudaSuccess) e = zero_pad_rows_launch(dX, d * 4, T, b->cu_seqlens, n, st);
  return e;
}

// ------------------------------------------------------------------ towers (Eqs. 8-9) in fp32
__global__ void gather_f32_kernel(const float* H, const int32_t* rows, int n, int T, int d, float* out, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * d) return;
  const int i = (int)(idx / d), c = (int)(idx % d);
  int r = rows[i];
  if (r < 0 || r >= T) {
    if (c == 0) atomicOr(err, ERRBIT_OFFSETS);
    r = 0;
  }
  out[idx] = H[(size_t)r * d + c];
}
// routed BCE with logits (Eq. 9): loss += softplus(z_k) - y z_k, dz[i, k] = sigma(z_k) - y on k = bucket[i]
__global__ void head_dz_f32_kernel(const float* logits, const int32_t* bucket, const float* label, int n, int K,
                                   float* dz, float* loss, float* db2, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = bucket[i];
  if (k < 0 || k >= K) {
    atomicOr(err, ERRBIT_BUCKET);
    k = min(max(k, 0), K - 1);
  }
  const float z = logits[(size_t)i * K + k], y = label[i];
  const float l = fmaxf(z, 0.f) + log1pf(expf(-fabsf(z))) - y * z;
  if (!isfinite(l)) atomicOr(err, ERRBIT_NONFINITE);
  const float gz = 1.f / (1.f + expf(-z)) - y;
  for (int kk = 0; kk < K; ++kk) dz[(size_t)i * K + kk] = kk == k ? gz : 0.f;
  atomicAdd(loss, l);
  atomicAdd(db2 + k, gz);
}
// dhid[i, c] = dz[i, c / dh] w2[c] 1[pre > 0]; db1[c] += dhid; dw2[c] += dz relu(pre)
__global__ void head_dhid_f32_kernel(const float* pre, const float* dz, const float* w2, int n, int K, int dh,
                                     float* dhid, float* db1, float* dw2) {
  pdl_trigger();
  pdl_wait();
  const int N = K * dh;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * N) return;
  const int i = (int)(idx / N), c = (int)(idx % N);
  const float z = dz[(size_t)i * K + c / dh], pr = pre[idx];
  const float g = pr > 0.f ? z * w2[c] : 0.f;
  dhid[idx] = g;
  if (g != 0.f) atomicAdd(db1 + c, g);
  if (pr > 0.f && z != 0.f) atomicAdd(dw2 + c, z * pr);
}
// db2[k] = sum_i dz[i, k] (towers backward from given logit gradients)
__global__ void head_db2_f32_kernel(const float* dz, int n, int K, float* db2) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < (size_t)n * K && dz[idx] != 0.f) atomicAdd(db2 + idx % K, dz[idx]);
}
// towers' epilogue: pre += b1; logits[i, k] = b2[k] + sum_{c in tower k} relu(pre[i, c]) w2[c]; warp per row
__global__ void head_post_f32_kernel(float* pre, const float* b1, const float* w2, const float* b2, int n, int K,
                                     int dh, float* logits) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  float* row = pre + (size_t)i * K * dh;
  for (int k = 0; k < K; ++k) {
    float acc = 0.f;
    for (int c = k * dh + lane; c < (k + 1) * dh; c += 32) {
      const float v = row[c] + b1[c];
      row[c] = v;
      acc = fmaf(fmaxf(v, 0.f), w2[c], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) logits[(size_t)i * K + k] = b2[k] + acc;
  }
}
// dHs[rows[i]] += src[i] (rows outside [0, T) were latched by the gather and are skipped)
__global__ void scatter_add_f32_kernel(const float* src, const int32_t* rows, int n, int T, int d, float* dHs) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * d) return;
  const int i = (int)(idx / d), c = (int)(idx % d), r = rows[i];
  if (r >= 0 && r < T) atomicAdd(dHs + (size_t)r * d + c, src[idx]);
}
__global__ void head_init_f32_kernel(float* logits, const float* b2, int n, int K) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * K) logits[i] = b2[i % K];
}

size_t f32_heads_ws_bytes(const cadet_head_config* h, int n) {
  const int d = h->d_model, N = h->K * h->d_hidden;
  size_t s = std::max(gemm3x_scratch_bytes(n, N, d), gemm3x_scratch_bytes(d, N, n));
  s = std::max(s, gemm3x_scratch_bytes(n, d, N));
  return 256 + a256((size_t)n * d * 4) + 2 * a256((size_t)n * N * 4) + a256((size_t)n * h->K * 4) + s;
}
struct F32HeadWs {
  uint32_t* err;
  float *Hr, *pre, *dhid, *dz;
  void* scratch;
};
static F32HeadWs carve_heads_f32(void* ws, const cadet_head_config* h, int n) {
  const int d = h->d_model, N = h->K * h->d_hidden;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  F32HeadWs W;
  W.err = reinterpret_cast<uint32_t*>(p);
  p += 256;
  W.Hr = reinterpret_cast<float*>(p);
  p += a256((size_t)n * d * 4);
  W.pre = reinterpret_cast<float*>(p);
  p += a256((size_t)n * N * 4);
  W.dhid = reinterpret_cast<float*>(p);
  p += a256((size_t)n * N * 4);
  W.dz = reinterpret_cast<float*>(p);
  p += a256((size_t)n * h->K * 4);
  W.scratch = p;
  return W;
}

cudaError_t heads_forward_f32(const cadet_head_config* h, const cadet_head_weights* w, const float* Hs,
                              const int32_t* rows, int n, float* logits, float* pre_out, void* ws, cudaStream_t st) {
  const int d = h->d_model, N = h->K * h->d_hidden;
  F32HeadWs W = carve_heads_f32(ws, h, n);
  float* pre = pre_out ? pre_out : W.pre;
  cudaError_t e = launch_pdl(gather_f32_kernel, dim3(nblk((size_t)n * d, 256)), dim3(256), 0, st, Hs, rows, n,
                             1 << 30, d, W.Hr, W.err);
  if (e == cudaSuccess)
  // pre = H_r W1 (3xTF32), then pre += b1 and logits = b2 + relu(pre) . w2 per tower (Eq. 8)
  if (e == cudaSuccess) e = gemm3x(n, N, d, W.Hr, 0, (const float*)w->W1, 0, pre, nullptr, W.scratch, st);
  if (e == cudaSuccess)
    e = launch_pdl(head_post_f32_kernel, dim3(nblk(n, 4)), dim3(128), 0, st, pre, w->b1, w->w2, w->b2, n, h->K,
                   h->d_hidden, logits);
  return e;
}

// dz given (dz_in, [n, K]) or the routed BCE of Eq. 9 (bucket / label / loss)
cudaError_t heads_backward_f32(const cadet_head_config* h, const cadet_head_weights* w, const float* Hs,
                               const int32_t* rows, int n, int T, const float* pre, const float* dz_in,
                               const float* logits, const int32_t* bucket, const float* label, float* loss,
                               int accumulate, float* dHs, const cadet_head_grads* g, void* ws, cudaStream_t st) {
  const int d = h->d_model, N = h->K * h->d_hidden;
  F32HeadWs W = carve_heads_f32(ws, h, n);
  cudaError_t e = cudaSuccess;
  const void* zs[5] = {g->dW1, g->db1, g->dw2, g->db2, accumulate ? nullptr : dHs};
  const size_t zb[5] = {(size_t)d * N * 4, (size_t)N * 4, (size_t)N * 4, (size_t)h->K * 4, (size_t)T * d * 4};
  for (int i = 0; i < 5 && e == cudaSuccess; ++i)
    if (zs[i]) e = cudaMemsetAsync(const_cast<void*>(zs[i]), 0, zb[i], st);
  if (loss && e == cudaSuccess) e = cudaMemsetAsync(loss, 0, 4, st);
  if (n == 0) return e;
  const float* dz = dz_in;
  if (!dz && e == cudaSuccess) {
    e = launch_pdl(head_dz_f32_kernel, dim3(nblk(n, 256)), dim3(256), 0, st, logits, bucket, label, n, h->K, W.dz,
                   loss, g->db2, W.err);
    dz = W.dz;
  } else if (e == cudaSuccess) {  // db2 = column sums of the given dz
    e = launch_pdl(head_db2_f32_kernel, dim3(nblk((size_t)n * h->K, 256)), dim3(256), 0, st, dz, n, h->K, g->db2);
  }
  if (e == cudaSuccess)
    e = launch_pdl(head_dhid_f32_kernel, dim3(nblk((size_t)n * N, 256)), dim3(256), 0, st, pre, dz, w->w2, n, h->K,
                   h->d_hidden, W.dhid, g->db1, g->dw2);
  if (e == cudaSuccess)
    e = launch_pdl(gather_f32_kernel, dim3(nblk((size_t)n * d, 256)), dim3(256), 0, st, Hs, rows, n, T, d, W.Hr, W.err);
  // dW1 = H_r^T dhid
  if (e == cudaSuccess) e = gemm3x(d, N, n, W.Hr, 1, W.dhid, 0, g->dW1, nullptr, W.scratch, st);
  // dH_r = dhid W1^T (into the H_r slot, no longer needed), then dHs[rows] += dH_r
  if (e == cudaSuccess) e = gemm3x(n, d, N, W.dhid, 0, (const float*)w->W1, 1, W.Hr, nullptr, W.scratch, st);
  if (e == cudaSuccess)
    e = launch_pdl(scatter_add_f32_kernel, dim3(nblk((size_t)n * d, 256)), dim3(256), 0, st, (const float*)W.Hr, rows,
                   n, T, d, dHs);
  return e;
}

}  // namespace cadet
