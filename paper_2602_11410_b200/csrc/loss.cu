// NEXT-2: the full training loss of PAPER.md Eqs. 10-12.
//   routed_logits_kernel   z_t = logits[t, k_t]: the logit the pairwise term compares (R29)
//   compact_kernel         positives / negatives of the batch in index order (deterministic)
//   pair_kernel            RankNet partial sums: thread = local sample, blockIdx.y = slice of the
//                          opposite-label list staged through shared memory
//   pair_finalize_kernel   dL_pair/dz per local sample, per-sample loss share (positives only)
//   full_loss_kernel       Eq. 11 logit gradients: routed BCE (+ pairwise) on the towers, aux tasks
//   head_dhid_full_kernel  tower backward from a full dz [n, K] (aux heads; towers with extra terms)
// Fixed-order reductions everywhere except the per-block loss atomics of full_loss_kernel.
#include <string.h>

#include "../../include/cadet.h"
#include "misc.cuh"
#include <cuda_fp16.h>
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {

__global__ void routed_logits_kernel(const float* logits, int K, const int32_t* bucket, int n, float* z) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = logits[(size_t)i * K + min(max(bucket[i], 0), K - 1)];
}

// One block: positives and negatives of label_all in index order (block scan per 1024-chunk):
// their logits (zp, zn) or, for the local samples, their indices (ip, in_).
__global__ void __launch_bounds__(1024) compact_kernel(const float* z_all, const float* y_all, int n_all, float* zp,
                                                       float* zn, int* counts, int* ip = nullptr, int* in_ = nullptr) {
  pdl_trigger();
  pdl_wait();
  __shared__ int sh[1024];
  int np = 0, nn = 0;
  for (int base = 0; base < n_all; base += 1024) {
    const int i = base + threadIdx.x;
    const bool v = i < n_all;
    const bool pos = v && y_all[i] > 0.5f;
    sh[threadIdx.x] = pos ? 1 : 0;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int x = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += x;
      __syncthreads();
    }
    const int incl = sh[threadIdx.x];
    const int tot = sh[1023];
    const int excl = incl - (pos ? 1 : 0);
    if (v) {
      if (ip) {
        if (pos)
          ip[np + excl] = i;
        else
          in_[nn + (i - base) - excl] = i;
      } else {
        if (pos)
          zp[np + excl] = z_all[i];
        else
          zn[nn + (i - base) - excl] = z_all[i];
      }
    }
    const int cnt = min(1024, n_all - base);
    np += tot;
    nn += cnt - tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[0] = np;
    counts[1] = nn;
  }
}

constexpr int PAIR_TILE = 2048;

// Partial sums over slice blockIdx.y of the opposite-label list; blockIdx.z = 0: local positives
// (thread = one of them, sweeping the batch's negatives), 1: local negatives (sweeping positives),
// so every warp runs one uniform loop:
//   positive i: g = sum_j sigma(z_j - z_i), l = sum_j softplus(z_j - z_i) over negatives j
//   negative i: g = sum_j sigma(z_i - z_j) over positives j (no loss: counted once, on positives)
__global__ void __launch_bounds__(256) pair_kernel(const float* z, int n, const int* ip, const int* in_,
                                                   const int* counts_loc, const float* zp, const float* zn,
                                                   const int* counts, float* part_g, float* part_l) {
  pdl_trigger();
  pdl_wait();
  __shared__ float tile[PAIR_TILE];
  const int side = blockIdx.z;
  const int nloc = counts_loc[side];
  if ((int)(blockIdx.x * blockDim.x) >= nloc) return;  // whole block beyond this side's samples
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < nloc;
  const int i = valid ? (side == 0 ? ip[t] : in_[t]) : 0;
  const float zi = valid ? z[i] : 0.f;
  const float* list = side == 0 ? zn : zp;
  const int len = side == 0 ? counts[1] : counts[0];
  const int S = gridDim.y, sidx = blockIdx.y;
  const int per = (len + S - 1) / S;
  const int j0 = min(len, sidx * per), j1 = min(len, j0 + per);
  float g = 0.f, l = 0.f;
  for (int t0 = j0; t0 < j1; t0 += PAIR_TILE) {
    const int tn = min(PAIR_TILE, j1 - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < tn; k += blockDim.x) tile[k] = list[t0 + k];
    __syncthreads();
    if (side == 0) {
      for (int k = 0; k < tn; ++k) {
        const float x = tile[k] - zi;                        // z_j- - z_i+
        const float e = __expf(-fabsf(x));
        const float r = __fdividef(1.f, 1.f + e);
        g += x >= 0.f ? r : e * r;                           // sigma(x)
        l += fmaxf(x, 0.f) + __logf(1.f + e);               // softplus(x)
      }
    } else {
      for (int k = 0; k < tn; ++k) {
        const float x = zi - tile[k];                        // z_i- - z_j+
        const float e = __expf(-fabsf(x));
        const float r = __fdividef(1.f, 1.f + e);
        g += x >= 0.f ? r : e * r;
      }
    }
  }
  if (valid) {
    part_g[(size_t)sidx * n + i] = g;
    part_l[(size_t)sidx * n + i] = side == 0 ? l : 0.f;
  }
}

__global__ void pair_finalize_kernel(const float* y, int n, const int* counts, const float* part_g,
                                     const float* part_l, int S, float* dz, float* lsample) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int np = counts[0], nn = counts[1];
  const float c = (np > 0 && nn > 0) ? 1.f / ((float)np * (float)nn) : 0.f;
  float g = 0.f, l = 0.f;
  for (int s = 0; s < S; ++s) {
    g += part_g[(size_t)s * n + i];
    l += part_l[(size_t)s * n + i];
  }
  dz[i] = (y[i] > 0.5f ? -c : c) * g;
  lsample[i] = c * l;
}

// Fixed-order single-block sum (deterministic).
__global__ void __launch_bounds__(1024) sum_kernel(const float* v, int n, float* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sh[1024];
  float a = 0.f;
  for (int i = threadIdx.x; i < n; i += 1024) a += v[i];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

struct LossArgs {
  float lambda_ctx, lambda_pair;
  float lambda_aux[8];
  int32_t aux_kind[8];
  int32_t J, K, n;
};

__global__ void __launch_bounds__(256) full_loss_kernel(LossArgs a, const float* logits, const int32_t* bucket,
                                                        const float* label, const float* dz_pair, const float* aux_out,
                                                        const float* aux_label, float* losses, float* dz_ctx,
                                                        float* dz_aux) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[9][8];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float lt[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) lt[t] = 0.f;
  if (i < a.n) {
    const int b = min(max(bucket[i], 0), a.K - 1);
    const float zr = logits[(size_t)i * a.K + b], y = label[i];
    for (int k = 0; k < a.K; ++k) dz_ctx[(size_t)i * a.K + k] = 0.f;
    const float sg = 1.f / (1.f + __expf(-zr));
    dz_ctx[(size_t)i * a.K + b] = a.lambda_ctx * (sg - y) + (dz_pair ? a.lambda_pair * dz_pair[i] : 0.f);
    lt[0] = fmaxf(zr, 0.f) + log1pf(__expf(-fabsf(zr))) - y * zr;
    for (int j = 0; j < a.J; ++j) {
      const float za = aux_out[(size_t)i * a.J + j], ya = aux_label[(size_t)i * a.J + j];
      float g, l;
      if (a.aux_kind[j] == 0) {
        g = 1.f / (1.f + __expf(-za)) - ya;
        l = fmaxf(za, 0.f) + log1pf(__expf(-fabsf(za))) - ya * za;
      } else {
        g = 2.f * (za - ya);
        l = (za - ya) * (za - ya);
      }
      dz_aux[(size_t)i * a.J + j] = a.lambda_aux[j] * g;
      lt[1 + j] = l;
    }
  }
  // block reduction of the 1 + J loss terms, one atomic per block and term
  for (int t = 0; t < 1 + a.J; ++t) {
    float v = lt[t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 1 + a.J) {
    float v = 0.f;
    for (int w = 0; w < 8; ++w) v += red[threadIdx.x][w];
    atomicAdd(losses + threadIdx.x, v);
  }
}

__global__ void loss_total_kernel(LossArgs a, const float* pair_share, float* losses) {
  pdl_trigger();
  pdl_wait();
  const float lp = pair_share ? *pair_share : 0.f;
  losses[a.J + 1] = lp;
  float t = a.lambda_ctx * losses[0] + a.lambda_pair * lp;
  for (int j = 0; j < a.J; ++j) t += a.lambda_aux[j] * losses[1 + j];
  losses[a.J + 2] = t;
}

// Tower backward from a full dz [n, K]: dhid = dz[i, k(c)] w2[c] 1[pre > 0] (bf16 hi + lo, R27),
// db1 += dhid, dw2 += dz relu(pre); thread = 8 consecutive columns (dh % 8 == 0).
__global__ void __launch_bounds__(256) head_dhid_full_kernel(const __nv_bfloat16* pre, const float* dz, const float* w2,
                                                             int n, int K, int dh, __nv_bfloat16* dhid,
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
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = w2[c0 + e];
    for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < n; i += gridDim.y * blockDim.y) {
      const float z = dz[(size_t)i * K + k];
      const uint4 pu = *reinterpret_cast<const uint4*>(pre + (size_t)i * N + c0);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pu);
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 pr = __bfloat1622float2(p2[e]);
        const float g0 = pr.x > 0.f ? z * w[2 * e] : 0.f, g1 = pr.y > 0.f ? z * w[2 * e + 1] : 0.f;
        s1[2 * e] += g0;
        s1[2 * e + 1] += g1;
        s2[2 * e] += z * fmaxf(pr.x, 0.f);
        s2[2 * e + 1] += z * fmaxf(pr.y, 0.f);
        if (dhid_lo) {  // bf16 hi + lo (R27)
          const __nv_bfloat162 h = __floats2bfloat162_rn(g0, g1);
          const float2 hf = __bfloat1622float2(h);
          const __nv_bfloat162 l = __floats2bfloat162_rn(g0 - hf.x, g1 - hf.y);
          hi[e] = *reinterpret_cast<const uint32_t*>(&h);
          lo[e] = *reinterpret_cast<const uint32_t*>(&l);
        } else {        // one fp16 operand (R27)
          const __half2 h = __floats2half2_rn(g0, g1);
          hi[e] = *reinterpret_cast<const uint32_t*>(&h);
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

// db2[k] = sum_i dz[i, k] (one block per tower, fixed order).
__global__ void __launch_bounds__(1024) dz_colsum_kernel(const float* dz, int n, int K, float* db2) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sh[1024];
  const int k = blockIdx.x;
  float a = 0.f;
  for (int i = threadIdx.x; i < n; i += 1024) a += dz[(size_t)i * K + k];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) db2[k] = sh[0];
}

static inline unsigned blocks(size_t n, unsigned b) { return (unsigned)((n + b - 1) / b); }
static inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static int pair_splits(int n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int bx = (n + 255) / 256;
  int s = (4 * sms + bx - 1) / (bx > 0 ? bx : 1);
  return s < 1 ? 1 : (s > 64 ? 64 : s);
}

cudaError_t head_dhid_full_launch(const void* pre, const float* dz, const float* w2, int n, int K, int dh, void* dhid,
                                  void* dhid_lo, float* db1, float* dw2, float* db2, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 2);
  if (n > 0) {
    dim3 blk(32, 8);
    dim3 grd((K * dh + 255) / 256, (unsigned)min(128, (n + 7) / 8));
    launch_pdl(head_dhid_full_kernel, dim3(grd), dim3(blk), 0, st, reinterpret_cast<const __nv_bfloat16*>(pre), dz, w2, n, K, dh,
                                               reinterpret_cast<__nv_bfloat16*>(dhid),
                                               reinterpret_cast<__nv_bfloat16*>(dhid_lo), db1, dw2);
    launch_pdl(dz_colsum_kernel, dim3(K), dim3(1024), 0, st, dz, n, K, db2);
  }
  return cudaGetLastError();
}

}  // namespace cadet

using namespace cadet;

namespace cadet {
void set_error(const char* msg);
}

extern "C" {

void cadet_default_loss_config(cadet_loss_config* lc, int32_t J) {
  if (!lc) return;
  memset(lc, 0, sizeof(*lc));
  lc->J = J < 0 ? 0 : (J > 8 ? 8 : J);
  lc->lambda_ctx = 1.0f;
  lc->lambda_pair = 0.1f;
  for (int j = 0; j < 8; ++j) {
    lc->lambda_aux[j] = 0.1f;
    lc->aux_kind[j] = j == 0 ? 0 : 1;
  }
}

cadet_status cadet_routed_logits(const float* logits, int32_t K, const int32_t* bucket, int32_t n, float* z_out,
                                 cadet_stream_t stream) {
  if (!logits || !bucket || !z_out || K < 1 || n < 0) {
    set_error("routed_logits: bad argument");
    return CADET_E_ARG;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 1);
  if (n > 0) launch_pdl(routed_logits_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, logits, K, bucket, n, z_out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return CADET_E_CUDA;
  }
  return CADET_OK;
}

size_t cadet_pairwise_workspace_bytes(int32_t n, int32_t n_all) {
  if (n < 0 || n_all < 0) return 0;
  const int S = pair_splits(n);
  return 256 + 2 * a256((size_t)n_all * 4) + 2 * a256((size_t)S * n * 4) + a256((size_t)n * 4) +
         2 * a256((size_t)n * 4) + 256;
}

cadet_status cadet_pairwise_loss(const float* z, const float* label, int32_t n, const float* z_all,
                                 const float* label_all, int32_t n_all, float* loss_share, float* dz_pair, void* ws,
                                 size_t ws_bytes, cadet_stream_t stream) {
  if (!z || !label || !z_all || !label_all || !loss_share || !dz_pair || !ws || n < 0 || n_all < n) {
    set_error("pairwise_loss: bad argument");
    return CADET_E_ARG;
  }
  const size_t need = cadet_pairwise_workspace_bytes(n, n_all);
  if (ws_bytes < need) {
    set_error("pairwise_loss: workspace too small");
    return CADET_E_WORKSPACE;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 5);
  const int S = pair_splits(n);
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  int* counts = reinterpret_cast<int*>(p);
  float* zp = reinterpret_cast<float*>(p + 256);
  float* zn = zp + a256((size_t)n_all * 4) / 4;
  float* part_g = zn + a256((size_t)n_all * 4) / 4;
  float* part_l = part_g + a256((size_t)S * n * 4) / 4;
  float* lsample = part_l + a256((size_t)S * n * 4) / 4;
  int* ip = reinterpret_cast<int*>(lsample + a256((size_t)n * 4) / 4);
  int* in_ = ip + a256((size_t)n * 4) / 4;
  int* counts_loc = in_ + a256((size_t)n * 4) / 4;
  cudaError_t e = cudaMemsetAsync(loss_share, 0, 4, st);
  if (n_all > 0 && e == cudaSuccess) {
    launch_pdl(compact_kernel, dim3(1), dim3(1024), 0, st, z_all, label_all, n_all, zp, zn, counts, (int*)nullptr,
               (int*)nullptr);
    if (n > 0) {
      launch_pdl(compact_kernel, dim3(1), dim3(1024), 0, st, z, label, n, nullptr, nullptr, counts_loc, ip, in_);
      launch_pdl(pair_kernel, dim3(dim3(blocks(n, 256), S, 2)), dim3(256), 0, st, z, n, ip, in_, counts_loc, zp, zn, counts, part_g,
                                                             part_l);
      launch_pdl(pair_finalize_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, label, n, counts, part_g, part_l, S, dz_pair, lsample);
      launch_pdl(sum_kernel, dim3(1), dim3(1024), 0, st, lsample, n, loss_share);
    }
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return CADET_E_CUDA;
  }
  return CADET_OK;
}

cadet_status cadet_full_loss_grads(const cadet_loss_config* lc, const float* logits, int32_t K, const int32_t* bucket,
                                   const float* label, const float* dz_pair, const float* pair_share,
                                   const float* aux_out, const float* aux_label, int32_t n, float* losses,
                                   float* dz_ctx, float* dz_aux, cadet_stream_t stream) {
  if (!lc || !logits || !bucket || !label || !losses || !dz_ctx || K < 1 || n < 0 || lc->J < 0 || lc->J > 8 ||
      (lc->J > 0 && (!aux_out || !aux_label || !dz_aux))) {
    set_error("full_loss_grads: bad argument");
    return CADET_E_ARG;
  }
  LossArgs a;
  memset(&a, 0, sizeof(a));
  a.lambda_ctx = lc->lambda_ctx;
  a.lambda_pair = lc->lambda_pair;
  for (int j = 0; j < 8; ++j) {
    a.lambda_aux[j] = lc->lambda_aux[j];
    a.aux_kind[j] = lc->aux_kind[j];
  }
  a.J = lc->J;
  a.K = K;
  a.n = n;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ProfScope ps(PROF_OTHER, st, 2);
  cudaError_t e = cudaMemsetAsync(losses, 0, sizeof(float) * (lc->J + 3), st);
  if (e == cudaSuccess && n > 0)
    launch_pdl(full_loss_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, a, logits, bucket, label, dz_pair, aux_out, aux_label, losses,
                                                     dz_ctx, dz_aux);
  if (e == cudaSuccess) launch_pdl(loss_total_kernel, dim3(1), dim3(1), 0, st, a, pair_share, losses);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return CADET_E_CUDA;
  }
  return CADET_OK;
}

}  // extern "C"
