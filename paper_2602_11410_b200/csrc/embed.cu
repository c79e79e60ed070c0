// NEXT-3 input embeddings (Eq. 1; "embeddings summed per token (id embeddings + type
// embedding)"): every token's input row is the sum of one row of each of F embedding tables,
// picked by the token's F integer ids (token type, ad id, request feature, action / context id; an id
// < 0 means the field is absent for that token kind).
//
//   embed_fwd_kernel   X[t] = sum_f E_f[ids[t, f]] (fp32 sum, one bf16 rounding); rows >= n_valid are 0
//   embed_bwd_*        dE_f[v] = sum over tokens t with ids[t, f] = v of dX[t], DETERMINISTIC:
//       - small tables (V <= 16): each CTA sums its token slice per (id, column) in registers in token
//         order, partials [CTA][V][d] are then summed over CTAs in CTA order;
//       - large tables: 64-bit fixed-point atomics (value * 2^24, two's complement): integer addition
//         is associative, so the result does not depend on the order the atomics land in (resolution
//         6e-8 absolute per contribution, range +-5e11), then one pass converts to fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>

#include "../../include/cadet.h"
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {
namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
inline unsigned nblk(size_t n, int b) { return (unsigned)((n + b - 1) / b); }
constexpr int SMALL_V = 16;
constexpr int SMALL_CTAS = 296;  // 2 waves of one 128 KB CTA per SM
constexpr float FIX_SCALE = 16777216.f;  // 2^24
struct Tables {
  const __nv_bfloat16* E[CADET_EMBED_MAX_TABLES];
  int32_t V[CADET_EMBED_MAX_TABLES];
};
}  // namespace

// thread = (row, 8 columns)
__global__ void embed_fwd_kernel(Tables tb, int F, const int32_t* ids, int T, const int32_t* n_valid, int d,
                                 __nv_bfloat16* X, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = d / 8;
  if (idx >= (size_t)T * per_row) return;
  const int t = (int)(idx / per_row), c0 = (int)(idx % per_row) * 8;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int nv = n_valid ? *n_valid : T;
  if (t < nv) {
    for (int f = 0; f < F; ++f) {
      const int v = ids[(size_t)t * F + f];
      if (v < 0) continue;
      if (v >= tb.V[f]) {
        if (c0 == 0) atomicOr(err, ERRBIT_BUCKET);
        continue;
      }
      const uint4 u = *reinterpret_cast<const uint4*>(tb.E[f] + (size_t)v * d + c0);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(h[e]);
        acc[2 * e] += x.x;
        acc[2 * e + 1] += x.y;
      }
    }
  }
  uint4 o;
  o.x = pack_bf16(acc[0], acc[1]);
  o.y = pack_bf16(acc[2], acc[3]);
  o.z = pack_bf16(acc[4], acc[5]);
  o.w = pack_bf16(acc[6], acc[7]);
  *reinterpret_cast<uint4*>(X + (size_t)t * d + c0) = o;
}

// all small tables (V <= 16) in ONE pass over dX: CTA b sums its token slice [b chunk, (b + 1) chunk) in
// token order into registers acc[slot][4] (thread = 4 columns; slot = the table's row offset + id, at most
// SMALL_SLOTS rows over all small tables), then stores them as partials [CTA][SMALL_SLOTS][d]
constexpr int SMALL_SLOTS = 32;
constexpr int SMALL_TABLES = 4;  // tables sharing the pass
struct SmallSet {
  int32_t n, f[CADET_EMBED_MAX_TABLES], V[CADET_EMBED_MAX_TABLES], off[CADET_EMBED_MAX_TABLES];
};
__global__ void __launch_bounds__(256) embed_bwd_small_kernel(const int32_t* ids, int F, SmallSet ss, int T,
                                                               const int32_t* n_valid, int d,
                                                               const __nv_bfloat16* dX, float* part) {
  pdl_trigger();
  pdl_wait();
  // per-CTA accumulator rows in shared memory, [SMALL_SLOTS][1024 columns]; thread = 4 columns, so every
  // float4 of the accumulator has exactly one owner: no races, tokens added in token order
  extern __shared__ float4 accs[];
  const int nv = n_valid ? min(*n_valid, T) : T;
  const int chunk = (nv + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * chunk, t1 = min(nv, t0 + chunk);
  for (int cb = 0; cb < d; cb += 1024) {
    const int c0 = cb + threadIdx.x * 4;
    const bool on = c0 < d;
    for (int k = 0; k < SMALL_SLOTS; ++k) accs[k * 256 + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    // 8 tokens per round: their dX slices and ids are all requested before any is accumulated
    for (int tb = t0; tb < t1 && on; tb += 8) {
      uint2 u[8];
      int slot[8][SMALL_TABLES];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = tb + q;
        u[q] = t < t1 ? *reinterpret_cast<const uint2*>(dX + (size_t)t * d + c0) : make_uint2(0u, 0u);
#pragma unroll
        for (int j = 0; j < SMALL_TABLES; ++j) {
          const int v = (t < t1 && j < ss.n) ? ids[(size_t)t * F + ss.f[j]] : -1;
          slot[q][j] = (v >= 0 && v < ss.V[j]) ? ss.off[j] + v : -1;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[q].x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[q].y));
#pragma unroll
        for (int j = 0; j < SMALL_TABLES; ++j) {
          if (slot[q][j] < 0) continue;
          float4& r = accs[slot[q][j] * 256 + threadIdx.x];
          r.x += a.x;
          r.y += a.y;
          r.z += b.x;
          r.w += b.y;
        }
      }
    }
    if (on)
      for (int k = 0; k < SMALL_SLOTS; ++k)
        *reinterpret_cast<float4*>(part + ((size_t)blockIdx.x * SMALL_SLOTS + k) * d + c0) = accs[k * 256 + threadIdx.x];
  }
}
// dE_f[v, c] = sum over CTAs b (in order) of part[b, off_f + v, c]
__global__ void embed_bwd_small_reduce_kernel(const float* part, int nb, int slot0, int V, int d, float* dE) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)V * d) return;
  float s = 0.f;
  for (int b = 0; b < nb; ++b) s += part[((size_t)b * SMALL_SLOTS + slot0) * d + i];
  dE[i] = s;
}
// large table: 64-bit fixed-point atomics; thread = (row, 8 columns)
__global__ void embed_bwd_fixed_kernel(const int32_t* ids, int F, int f, int V, int T, const int32_t* n_valid, int d,
                                       const __nv_bfloat16* dX, unsigned long long* acc) {
  pdl_trigger();
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = d / 8;
  const int nv = n_valid ? min(*n_valid, T) : T;
  if (idx >= (size_t)nv * per_row) return;
  const int t = (int)(idx / per_row), c0 = (int)(idx % per_row) * 8;
  const int v = ids[(size_t)t * F + f];
  if (v < 0 || v >= V) return;
  const uint4 u = *reinterpret_cast<const uint4*>(dX + (size_t)t * d + c0);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  unsigned long long* a = acc + (size_t)v * d + c0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(h[e]);
    if (x.x != 0.f) atomicAdd(a + 2 * e, (unsigned long long)__float2ll_rn(x.x * FIX_SCALE));
    if (x.y != 0.f) atomicAdd(a + 2 * e + 1, (unsigned long long)__float2ll_rn(x.y * FIX_SCALE));
  }
}
__global__ void embed_fixed_to_f32_kernel(const unsigned long long* acc, size_t n, float* dE) {
  pdl_trigger();
  pdl_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dE[i] = (float)((double)(long long)acc[i] * (1.0 / 16777216.0));
}

static size_t small_part_bytes(int d) { return a256((size_t)SMALL_CTAS * 32 * d * 4); }

size_t embed_ws_bytes(const cadet_embed_config* c) {
  size_t fixed = 0;
  for (int f = 0; f < c->n_tables; ++f)  // (tables not in the shared small pass use the fixed-point path)
    fixed = std::max(fixed, a256((size_t)c->vocab[f] * c->d_model * 8));
  return 256 + small_part_bytes(c->d_model) + fixed;
}

cudaError_t embed_forward_launch(const cadet_embed_config* c, const void* const* tables, const int32_t* ids, int T,
                                 const int32_t* n_valid, void* X, void* ws, cudaStream_t st) {
  Tables tb;
  memset(&tb, 0, sizeof(tb));
  for (int f = 0; f < c->n_tables; ++f) {
    tb.E[f] = reinterpret_cast<const __nv_bfloat16*>(tables[f]);
    tb.V[f] = c->vocab[f];
  }
  ProfScope ps(PROF_OTHER, st, 1);
  const size_t work = (size_t)T * c->d_model / 8;
  if (!work) return cudaSuccess;
  return launch_pdl(embed_fwd_kernel, dim3(nblk(work, 256)), dim3(256), 0, st, tb, c->n_tables, ids, T, n_valid,
                    c->d_model, reinterpret_cast<__nv_bfloat16*>(X), reinterpret_cast<uint32_t*>(ws));
}

cudaError_t embed_backward_launch(const cadet_embed_config* c, const int32_t* ids, int T, const int32_t* n_valid,
                                  const void* dX, float* const* dtables, void* ws, cudaStream_t st) {
  const int d = c->d_model, F = c->n_tables;
  const __nv_bfloat16* g = reinterpret_cast<const __nv_bfloat16*>(dX);
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + 256);
  unsigned long long* fix = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + 256 +
                                                                  small_part_bytes(d));
  ProfScope ps(PROF_OTHER, st, 2 * F);
  cudaError_t e = cudaSuccess;
  SmallSet ss;
  memset(&ss, 0, sizeof(ss));
  int slots = 0;
  for (int f = 0; f < F; ++f)  // small tables share one pass while their rows fit SMALL_SLOTS registers
    if (c->vocab[f] <= SMALL_V && slots + c->vocab[f] <= SMALL_SLOTS && ss.n < SMALL_TABLES) {
      ss.f[ss.n] = f;
      ss.V[ss.n] = c->vocab[f];
      ss.off[ss.n] = slots;
      slots += c->vocab[f];
      ++ss.n;
    }
  if (ss.n > 0) {
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(embed_bwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               SMALL_SLOTS * 256 * 16);
      attr = e == cudaSuccess;
    }
    if (e == cudaSuccess)
      e = launch_pdl(embed_bwd_small_kernel, dim3(SMALL_CTAS), dim3(256), SMALL_SLOTS * 256 * 16, st, ids, F, ss, T,
                     n_valid, d, g, part);
    for (int j = 0; j < ss.n && e == cudaSuccess; ++j)
      e = launch_pdl(embed_bwd_small_reduce_kernel, dim3(nblk((size_t)ss.V[j] * d, 256)), dim3(256), 0, st,
                     (const float*)part, SMALL_CTAS, ss.off[j], ss.V[j], d, dtables[ss.f[j]]);
  }
  for (int f = 0; f < F && e == cudaSuccess; ++f) {
    bool done = false;
    for (int j = 0; j < ss.n; ++j) done = done || ss.f[j] == f;
    if (done) continue;
    const int V = c->vocab[f];
    e = cudaMemsetAsync(fix, 0, (size_t)V * d * 8, st);
    if (e == cudaSuccess)
      e = launch_pdl(embed_bwd_fixed_kernel, dim3(nblk((size_t)T * d / 8, 256)), dim3(256), 0, st, ids, F, f, V, T,
                     n_valid, d, g, fix);
    if (e == cudaSuccess)
      e = launch_pdl(embed_fixed_to_f32_kernel, dim3(nblk((size_t)V * d, 256)), dim3(256), 0, st,
                     (const unsigned long long*)fix, (size_t)V * d, dtables[f]);
  }
  return e;
}

}  // namespace cadet
