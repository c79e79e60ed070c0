// Persistent warp-specialised tcgen05 GEMM (bf16 in, fp32 accumulate in TMEM) with the
// CADET epilogues fused (rows A2-A4, A6, A7, A9, A11, A12).
//
//   warp 0      : TMA producer (one elected lane), 128B-swizzled K- or MN-major tiles
//   warp 1      : tcgen05.mma issuer (one elected lane), M=128 x N=BN x K=16 per instruction
//   warp 2      : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..11 : epilogue, thread = accumulator row (TMEM lane), tcgen05.ld 32 columns at a time;
//                 two warps per TMEM lane quarter split the 32-column slices
//
// C[M,N] = sum_seg A_seg[M,K_seg] . B_seg[K_seg,N], tiles 128 x BN x 64, split-K optional.
#include "gemm.cuh"
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"
#include <string.h>

namespace cadet {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int GEMM_THREADS = 384;  // 4 non-epilogue warps + 8 epilogue warps

struct KProb {
  int32_t M, N, nseg, kb_total, split_k, m_tiles, n_tiles, unit_begin;
  int32_t kb[GEMM_MAX_SEG];
  int32_t a_mn[GEMM_MAX_SEG], b_mn[GEMM_MAX_SEG];
  int32_t f16, tf32;
  EpiParams epi;
};

struct GemmKParams {
  CUtensorMap mA[GEMM_MAX_PROB][GEMM_MAX_SEG];
  CUtensorMap mB[GEMM_MAX_PROB][GEMM_MAX_SEG];
  KProb p[GEMM_MAX_PROB];
  int32_t nprob, total_units;
  int32_t bm;  // M tile of a unit: 128 (one CTA) or 256 (CTA pair, cta_group::2)
};

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;        // [8 epilogue warps][4 KB] row transposes
  static constexpr int BAR_OFF = STG_OFF + 8 * 4096;
  static constexpr int SMEM = BAR_OFF + 1024 + 256;
};

struct Unit {
  int p, m0, n0, kb_lo, kb_hi, ks;
};

__device__ __forceinline__ Unit decode_unit(const GemmKParams& P, int u) {
  int p = 0;
  while (p + 1 < P.nprob && u >= P.p[p + 1].unit_begin) ++p;
  const KProb& q = P.p[p];
  int local = u - q.unit_begin;
  // split-K: K-slice outermost, so the m x n tiles of one K-slice run together and that slice of
  // both operands stays L2-resident (weight gradients read each activation row block once)
  const int mn = q.m_tiles * q.n_tiles;
  const int ks = local / mn;
  local -= ks * mn;
  const int nt = local % q.n_tiles;
  const int mt = local / q.n_tiles;
  Unit r;
  r.p = p;
  r.m0 = mt * P.bm;
  r.n0 = nt;  // tile index; callers multiply by BN
  r.kb_lo = (int)(((long long)ks * q.kb_total) / q.split_k);
  r.kb_hi = (int)(((long long)(ks + 1) * q.kb_total) / q.split_k);
  r.ks = ks;
  return r;
}

__device__ __forceinline__ void kb_to_seg(const KProb& q, int kb, int& seg, int& kk) {
  seg = 0;
  while (seg + 1 < q.nseg && kb >= q.kb[seg]) {
    kb -= q.kb[seg];
    ++seg;
  }
  kk = kb;
}

// The k-block walk of one unit with the per-segment fields in registers: the producer / MMA loops
// otherwise re-read them from parameter space after every mbarrier wait (the waits clobber memory),
// a dependent chain of constant loads per k-block that made short-K GEMMs (d 352) issue-bound.
struct SegCursor {
  int seg, kk, left;  // left: k-blocks before the next segment (the last segment never advances)
  uint32_t a_mn, b_mn;
  __device__ __forceinline__ void load(const KProb& q) {
    a_mn = (uint32_t)q.a_mn[seg];
    b_mn = (uint32_t)q.b_mn[seg];
  }
  __device__ __forceinline__ void init(const KProb& q, int kb) {
    kb_to_seg(q, kb, seg, kk);
    left = seg + 1 < q.nseg ? q.kb[seg] - kk : 0x7fffffff;
    load(q);
  }
  __device__ __forceinline__ void next(const KProb& q) {
    ++kk;
    if (--left == 0) {
      ++seg;
      kk = 0;
      left = seg + 1 < q.nseg ? q.kb[seg] : 0x7fffffff;
      load(q);
    }
  }
};

// ---------------------------------------------------------------- epilogue helpers
// Epilogue mode sets (compile time): each GEMM launch instantiates only the epilogues of its
// problems, so e.g. a plain store does not carry the gate + RoPE epilogue's registers.
__host__ __device__ constexpr uint32_t MB(int m) { return 1u << m; }
constexpr uint32_t MODES_ALL = MB(EPI_STORE) | MB(EPI_GATE) | MB(EPI_GATE_BWD) | MB(EPI_ATOMIC) |
                               MB(EPI_HEAD) | MB(EPI_GELU) | MB(EPI_GELU_BWD);

// exact GELU u Phi(u) and its derivative (R33)
__device__ __forceinline__ float gelu_f(float u) { return 0.5f * u * (1.f + erff(u * 0.7071067811865476f)); }
__device__ __forceinline__ float gelu_grad_f(float u) {
  return 0.5f * (1.f + erff(u * 0.7071067811865476f)) + u * 0.3989422804014327f * ex2_ftz(-0.7213475204444817f * u * u);
}
#define HAS_MODE(m) ((MODES & MB(m)) != 0u)
__device__ __forceinline__ void load_bf16x32(const void* base, float (&x)[32]) {
  const uint4* p = reinterpret_cast<const uint4*>(base);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = p[q];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      x[q * 8 + e * 2] = f.x;
      x[q * 8 + e * 2 + 1] = f.y;
    }
  }
}
__device__ __forceinline__ void load_f32x32(const void* base, float (&x)[32]) {
  const float4* p = reinterpret_cast<const float4*>(base);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 v = p[q];
    x[q * 4] = v.x;
    x[q * 4 + 1] = v.y;
    x[q * 4 + 2] = v.z;
    x[q * 4 + 3] = v.w;
  }
}
__device__ __forceinline__ void load_any32(const void* base, int is_f32, size_t off, float (&x)[32]) {
  if (is_f32)
    load_f32x32(reinterpret_cast<const float*>(base) + off, x);
  else
    load_bf16x32(reinterpret_cast<const __nv_bfloat16*>(base) + off, x);
}
__device__ __forceinline__ void store_any32(void* base, int is_f32, size_t off, const float (&x)[32]) {
  if (is_f32) {
    float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + off);
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = make_float4(x[q * 4], x[q * 4 + 1], x[q * 4 + 2], x[q * 4 + 3]);
  } else {
    uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + off);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(x[q * 8 + 0], x[q * 8 + 1]);
      u.y = pack_bf16(x[q * 8 + 2], x[q * 8 + 3]);
      u.z = pack_bf16(x[q * 8 + 4], x[q * 8 + 5]);
      u.w = pack_bf16(x[q * 8 + 6], x[q * 8 + 7]);
      p[q] = u;
    }
  }
}

template <uint32_t MODES>
__device__ __forceinline__ void run_epilogue(const EpiParams& e, int row, int M, int n0c, float (&v)[32]) {
  if (row >= M) return;
  int orow = row;
  if (e.row_map) {
    orow = e.row_map[row];
    if (orow < 0 || (e.row_map_max > 0 && orow >= e.row_map_max)) return;
  }
  const size_t off = (size_t)orow * e.ldo + n0c;
  const size_t in_off = (size_t)row * e.ldo + n0c;
  switch (e.mode) {
    case EPI_STORE: if constexpr (HAS_MODE(EPI_STORE)) {
      if (e.resid) {
        float r[32];
        load_any32(e.resid, e.resid_f32, e.resid_at_out ? off : in_off, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += r[j];
      }
      store_any32(e.out, e.out_f32, off, v);
    } break;
    case EPI_GATE: if constexpr (HAS_MODE(EPI_GATE)) {
      if (e.aux) store_any32(e.aux, e.aux_f32, in_off, v);
      float x[32];
      load_bf16x32(reinterpret_cast<const __nv_bfloat16*>(e.src) + in_off, x);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = x[j] * sigmoid_fast(v[j]);
      store_any32(e.out, e.out_f32, off, v);
    } break;
    case EPI_GATE_BWD: if constexpr (HAS_MODE(EPI_GATE_BWD)) {
      float z[32], x[32];
      load_any32(e.aux, e.aux_f32, in_off, z);
      load_bf16x32(reinterpret_cast<const __nv_bfloat16*>(e.src) + in_off, x);
      float r[32];
      if (e.resid) {
        load_any32(e.resid, e.resid_f32, in_off, r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0.f;
      }
      float u[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float g = sigmoid_fast(z[j]);
        u[j] = v[j] * x[j] * g * (1.0f - g);
        r[j] += v[j] * g;
      }
      store_any32(e.out, e.out_f32, off, u);
      store_any32(e.out2, e.out2_f32, off, r);
    } break;
    case EPI_ATOMIC: if constexpr (HAS_MODE(EPI_ATOMIC)) {
      float* o = reinterpret_cast<float*>(e.out) + off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        atomicAdd(reinterpret_cast<float4*>(o) + q, make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]));
    } break;
    case EPI_GELU: if constexpr (HAS_MODE(EPI_GELU)) {
      if (e.aux) store_any32(e.aux, e.aux_f32, in_off, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
      store_any32(e.out, e.out_f32, off, v);
    } break;
    case EPI_GELU_BWD: if constexpr (HAS_MODE(EPI_GELU_BWD)) {
      float u[32];
      load_any32(e.aux, e.aux_f32, in_off, u);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(u[j]);
      store_any32(e.out, e.out_f32, off, v);
    } break;
    case EPI_HEAD: if constexpr (HAS_MODE(EPI_HEAD)) {
      // a 32-column slice covers at most two towers when dh % 32 != 0 (dh >= 32)
      const int k0 = n0c / e.hd;
      const int split = (k0 + 1) * e.hd - n0c;  // first column of tower k0 + 1 inside the slice
      float part0 = 0.f, part1 = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float pre = v[j] + e.b1[n0c + j];
        v[j] = pre;
        const float c = fmaxf(pre, 0.f) * e.w2[n0c + j];
        if (j < split)
          part0 += c;
        else
          part1 += c;
      }
      if (e.aux) store_any32(e.aux, e.aux_f32, in_off, v);
      atomicAdd(e.logits + (size_t)row * e.n_towers + k0, part0);
      if (split < 32) atomicAdd(e.logits + (size_t)row * e.n_towers + k0 + 1, part1);
    } break;
    default:
      break;
  }
}

__device__ __forceinline__ void warp_store_rows(uint32_t stg, void* base, int is_f32, size_t off0, size_t ld,
                                                int rows_valid, const float (&v)[32]) {
  if (!is_f32) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
    warp_store_rows_bf16(stg, w, reinterpret_cast<__nv_bfloat16*>(base) + off0, ld, rows_valid, 32);
  } else {
    uint32_t u[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(v[j]);
    warp_store_rows_f32(stg, u, 1.0f, reinterpret_cast<float*>(base) + off0, ld, rows_valid, 32);
  }
}

// Primary epilogue input (bf16 only), loaded one slice ahead by the epilogue loop: src for the
// gates, resid for a store, aux (the saved pre-activation) for the gate backward.
__device__ __forceinline__ const void* epi_primary(const EpiParams& e) {
  if (e.row_map) return nullptr;
  switch (e.mode) {
    case EPI_GATE:
      return e.src;
    case EPI_STORE:
      return e.resid ? (e.resid_f32 ? nullptr : e.resid) : e.dot_src;
    case EPI_GATE_BWD:
    case EPI_GELU_BWD:
      return e.aux_f32 ? nullptr : e.aux;
    default:
      return nullptr;
  }
}

template <uint32_t MODES>
__device__ __forceinline__ void run_epilogue_warp(const EpiParams& e, int row0, int M, int n0c, float (&v)[32],
                                                  uint32_t stg, const uint4* pre = nullptr, int ks = 0) {
  const int lane = threadIdx.x & 31;
  if (e.row_map) {
    run_epilogue<MODES>(e, row0 + lane, M, n0c, v);
    return;
  }
  const int rows_valid = M - row0;
  if (rows_valid <= 0) return;
  const size_t off0 = (size_t)row0 * e.ldo + n0c;
  switch (e.mode) {
    case EPI_STORE: if constexpr (HAS_MODE(EPI_STORE)) {
      if (e.resid) {
        float r[32];
        if (pre)
          warp_sts_rows_bf16(stg, *reinterpret_cast<const uint4(*)[4]>(pre), r);
        else
          warp_load_rows(stg, e.resid, e.resid_f32, off0, e.ldo, rows_valid, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += r[j];
      }
      if (e.dot_out) {  // per-(row, head) partial of rowsum(acc * dot_src)
        float x[32];
        if (pre && !e.resid)
          warp_sts_rows_bf16(stg, *reinterpret_cast<const uint4(*)[4]>(pre), x);
        else
          warp_load_rows(stg, e.dot_src, 0, off0, e.ldo, rows_valid, x);
        // a 32-column slice covers at most two heads (hd >= 32): split the sum at the head edge
        const int h0 = n0c / e.hd, split = (h0 + 1) * e.hd - n0c;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < split)
            s0 = fmaf(v[j], x[j], s0);
          else
            s1 = fmaf(v[j], x[j], s1);
        }
        if (lane < rows_valid) {
          atomicAdd(e.dot_out + (size_t)h0 * e.dot_T + row0 + lane, s0);
          if (split < 32) atomicAdd(e.dot_out + (size_t)(h0 + 1) * e.dot_T + row0 + lane, s1);
        }
      }
      if constexpr (HAS_MODE(EPI_TAPS)) {
        if (e.tap) warp_store_rows(stg, e.tap, 1, off0, e.ldo, rows_valid, v);
      }
      warp_store_rows(stg, e.out, e.out_f32, off0, e.ldo, rows_valid, v);
    } break;
    case EPI_GATE: if constexpr (HAS_MODE(EPI_GATE)) {
      if (e.aux) warp_store_rows(stg, e.aux, e.aux_f32, off0, e.ldo, rows_valid, v);
      if constexpr (HAS_MODE(EPI_TAPS)) {
        if (e.tap2) warp_store_rows(stg, e.tap2, 1, off0, e.ldo, rows_valid, v);
      }
      float x[32];
      if (pre)
        warp_sts_rows_bf16(stg, *reinterpret_cast<const uint4(*)[4]>(pre), x);
      else
        warp_load_rows(stg, e.src, 0, off0, e.ldo, rows_valid, x);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = x[j] * sigmoid_fast(v[j]);
      if constexpr (HAS_MODE(EPI_TAPS)) {
        if (e.tap) warp_store_rows(stg, e.tap, 1, off0, e.ldo, rows_valid, v);
      }
      warp_store_rows(stg, e.out, e.out_f32, off0, e.ldo, rows_valid, v);
    } break;
    case EPI_GATE_BWD: if constexpr (HAS_MODE(EPI_GATE_BWD)) {
      float z[32], x[32], r[32];
      if (pre)
        warp_sts_rows_bf16(stg, *reinterpret_cast<const uint4(*)[4]>(pre), z);
      else
        warp_load_rows(stg, e.aux, e.aux_f32, off0, e.ldo, rows_valid, z);
      warp_load_rows(stg, e.src, 0, off0, e.ldo, rows_valid, x);
      if (e.resid) {
        warp_load_rows(stg, e.resid, e.resid_f32, off0, e.ldo, rows_valid, r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float g = sigmoid_fast(z[j]);
        const float vj = v[j];
        v[j] = vj * x[j] * g * (1.0f - g);
        r[j] += vj * g;
      }
      if constexpr (HAS_MODE(EPI_TAPS)) {
        if (e.tap) warp_store_rows(stg, e.tap, 1, off0, e.ldo, rows_valid, v);
        if (e.tap2) warp_store_rows(stg, e.tap2, 1, off0, e.ldo, rows_valid, r);
      }
      warp_store_rows(stg, e.out, e.out_f32, off0, e.ldo, rows_valid, v);
      warp_store_rows(stg, e.out2, e.out2_f32, off0, e.ldo, rows_valid, r);
    } break;
    case EPI_ATOMIC: if constexpr (HAS_MODE(EPI_ATOMIC)) {
      if (e.split_stride) {  // deterministic mode: split ks stores its partial into its own slab
        warp_store_rows(stg, reinterpret_cast<float*>(e.out) + (size_t)ks * e.split_stride, 1, off0, e.ldo, rows_valid, v);
        break;
      }
      // split-K partials: transpose through the stage, then fp32 vector reductions that cover 4 rows
      // x 128 B per instruction (instead of 32 rows x 16 B)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        sts_u4(stg + lane * 128 + ((j ^ (lane & 7)) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
               __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
      __syncwarp();
      float* base = reinterpret_cast<float*>(e.out) + off0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = i * 4 + (lane >> 3), j = lane & 7;
        const uint4 u = lds_u4(stg + row * 128 + ((j ^ (row & 7)) << 4));
        if (row < rows_valid)
          atomicAdd(reinterpret_cast<float4*>(base + (size_t)row * e.ldo + j * 4),
                    make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w)));
      }
      __syncwarp();
    } break;
    case EPI_HEAD: if constexpr (HAS_MODE(EPI_HEAD)) {
      // pre = acc + b1 (saved through the warp transpose), logits[row, k] += relu(pre) . w2; a
      // 32-column slice covers at most two towers when dh % 32 != 0 (dh >= 32)
      const int k0 = n0c / e.hd;
      const int split = (k0 + 1) * e.hd - n0c;
      const float4* b4 = reinterpret_cast<const float4*>(e.b1 + n0c);
      const float4* w4 = reinterpret_cast<const float4*>(e.w2 + n0c);
      float part0 = 0.f, part1 = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 bb = b4[q], ww = w4[q];
        const float bv[4] = {bb.x, bb.y, bb.z, bb.w}, wv[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = 4 * q + k;
          v[j] += bv[k];
          const float c = fmaxf(v[j], 0.f) * wv[k];
          if (j < split)
            part0 += c;
          else
            part1 += c;
        }
      }
      if (e.aux) warp_store_rows(stg, e.aux, e.aux_f32, off0, e.ldo, rows_valid, v);
      if (lane < rows_valid) {
        atomicAdd(e.logits + (size_t)(row0 + lane) * e.n_towers + k0, part0);
        if (split < 32) atomicAdd(e.logits + (size_t)(row0 + lane) * e.n_towers + k0 + 1, part1);
      }
    } break;
    case EPI_GELU: if constexpr (HAS_MODE(EPI_GELU)) {
      if (e.aux) warp_store_rows(stg, e.aux, e.aux_f32, off0, e.ldo, rows_valid, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
      warp_store_rows(stg, e.out, e.out_f32, off0, e.ldo, rows_valid, v);
    } break;
    case EPI_GELU_BWD: if constexpr (HAS_MODE(EPI_GELU_BWD)) {
      float u[32];
      if (pre)
        warp_sts_rows_bf16(stg, *reinterpret_cast<const uint4(*)[4]>(pre), u);
      else
        warp_load_rows(stg, e.aux, e.aux_f32, off0, e.ldo, rows_valid, u);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(u[j]);
      warp_store_rows(stg, e.out, e.out_f32, off0, e.ldo, rows_valid, v);
    } break;
    default:
      break;
  }
}

// ---------------------------------------------------------------- kernel
template <int BN, uint32_t MODES>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_kernel(const __grid_constant__ GemmKParams P) {
  using C = GemmCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < P.nprob; ++p)
      for (int s = 0; s < P.p[p].nseg; ++s) {
        tma_prefetch(&P.mA[p][s]);
        tma_prefetch(&P.mB[p][s]);
      }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first
  pdl_wait();  // operands / epilogue inputs are the previous kernels' outputs

  // registers: warpgroup 0 (TMA, MMA, allocator, idle) gives 104 per thread to the epilogue warpgroups
  if (warp == 0) {
    // ============================ TMA producer
    setmaxnreg_dec<64>();
    if (elect_one()) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < P.total_units; u += gridDim.x) {
        const Unit U = decode_unit(P, u);
        const KProb& q = P.p[U.p];
        const int n0 = U.n0 * BN;
        const int bke = q.tf32 ? BK / 2 : BK;  // a 128-byte K row: 64 bf16 / 32 fp32
        SegCursor sc;
        sc.init(q, U.kb_lo);
        for (int kb = U.kb_lo; kb < U.kb_hi; ++kb, ++it, sc.next(q)) {
          const uint32_t stage = it % C::STAGES, use = it / C::STAGES;
          if (use > 0) mbar_wait(&empty[stage], (use - 1) & 1);
          const int k0 = sc.kk * bke;
          const CUtensorMap* mA = &P.mA[U.p][sc.seg];
          const CUtensorMap* mB = &P.mB[U.p][sc.seg];
          uint8_t* sA = smem + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + C::A_BYTES;
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          if (!sc.a_mn) {
            tma_load_2d(sA, mA, &full[stage], k0, U.m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(sA + j * 8192, mA, &full[stage], U.m0 + 64 * j, k0);
          }
          if (!sc.b_mn) {
            tma_load_2d(sB, mB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, mB, &full[stage], n0 + 64 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    setmaxnreg_dec<64>();
    if (elect_one()) {
      uint32_t it = 0, tc = 0;
      for (int u = blockIdx.x; u < P.total_units; u += gridDim.x, ++tc) {
        const Unit U = decode_unit(P, u);
        const KProb& q = P.p[U.p];
        const uint32_t buf = tc & 1, use = tc >> 1;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        const bool tf32 = q.tf32 != 0;
        const uint32_t fmask = q.f16 ? ~((7u << 7) | (7u << 10)) : ~0u;  // F16: format 0
        SegCursor sc;
        sc.init(q, U.kb_lo);
        for (int kb = U.kb_lo; kb < U.kb_hi; ++kb, ++it, sc.next(q)) {
          const uint32_t stage = it % C::STAGES, suse = it / C::STAGES;
          mbar_wait(&full[stage], suse & 1);
          tc_fence_after();
          const uint32_t a_mn = sc.a_mn, b_mn = sc.b_mn;
          const uint32_t sA = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sB = sA + C::A_BYTES;
          if (tf32) {  // K-major fp32 tiles: 4 x (K = 8) per 128-byte row, same 32-byte descriptor steps
            const uint32_t idesc = idesc_tf32(BM, BN);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_tf32_ss(d_tmem, smem_desc(sA + k * 32, 16, 1024, SWZ_128B), smem_desc(sB + k * 32, 16, 1024, SWZ_128B),
                          idesc, (kb > U.kb_lo || k > 0) ? 1u : 0u);
          } else {
            const uint32_t idesc = idesc_bf16(BM, BN, a_mn, b_mn) & fmask;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = a_mn ? smem_desc(sA + k * 2048, 8192, 1024, SWZ_128B)
                                       : smem_desc(sA + k * 32, 16, 1024, SWZ_128B);
              const uint64_t bd = b_mn ? smem_desc(sB + k * 2048, 8192, 1024, SWZ_128B)
                                       : smem_desc(sB + k * 32, 16, 1024, SWZ_128B);
              mma_bf16_ss(d_tmem, ad, bd, idesc, (kb > U.kb_lo || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[stage]);
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<64>();
  } else {
    // ============================ epilogue
    setmaxnreg_inc<216>();
    const uint32_t quarter = warp & 3;
    const int half = (warp - 4) >> 2;  // warps 4-7 take even 32-column slices, 8-11 odd ones
    const uint32_t stg = smem_u32(smem + C::STG_OFF) + (warp - 4) * 4096;
    uint32_t tc = 0;
    for (int u = blockIdx.x; u < P.total_units; u += gridDim.x, ++tc) {
      const Unit U = decode_unit(P, u);
      const KProb& q = P.p[U.p];
      // the epilogue parameters in registers for the whole tile (parameter-space reads would be
      // repeated after every TMEM / barrier wait, which clobber memory)
      const EpiParams e = q.epi;
      const int qM = q.M, qN = q.N;
      const uint32_t buf = tc & 1, use = tc >> 1;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int row0 = U.m0 + quarter * 32;
      const int n0 = U.n0 * BN;
      // the primary epilogue input of slice c + 2 is requested before slice c is processed
      const void* pb = epi_primary(e);
      uint4 g[4];
      auto issue = [&](int c) {
        const int n0c = n0 + c * 32;
        if (c < BN / 32 && n0c < qN && row0 < qM && pb)
          warp_ldg_rows_bf16(pb, (size_t)row0 * e.ldo + n0c, e.ldo, qM - row0, g);
      };
      issue(half);
      for (int c = half; c < BN / 32; c += 2) {
        const int n0c = n0 + c * 32;
        if (n0c >= qN) break;
        uint4 cur[4] = {g[0], g[1], g[2], g[3]};
        issue(c + 2);
        uint32_t r[32];
        tmem_ld32(tmem_addr(tmem_base, quarter, buf * BN + c * 32), r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        run_epilogue_warp<MODES>(e, row0, qM, n0c, v, stg, pb ? cur : nullptr, U.ks);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

// ---------------------------------------------------------------- CTA-pair kernel (cta_group::2)
// Two CTAs of a cluster compute one 256 x 256 tile: CTA r holds A rows [128 r, 128 r + 128) and B
// columns [128 r, 128 r + 128) of the tile in its shared memory; the leader issues M=256 N=256
// tcgen05.mma.cta_group::2, each CTA's TMEM receives its 128 rows x 256 columns.  Per SM and
// k-block this streams 32 KB (vs 48 KB for a 128 x 256 one-CTA tile): half the B traffic, which
// is what bounds the d x d projections through L2.
struct PairCfg {
  static constexpr int STAGES = 6;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = 128 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 512;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = STG_OFF + 8 * 4096;
  static constexpr int SMEM = BAR_OFF + 1024 + 256;
};

template <uint32_t MODES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ GemmKParams P) {
  using C = PairCfg;
  constexpr int BN = 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);  // 8 epilogue warps in each CTA of the pair
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < P.nprob; ++p)
      for (int s = 0; s < P.p[p].nseg; ++s) {
        tma_prefetch(&P.mA[p][s]);
        tma_prefetch(&P.mB[p][s]);
      }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first
  pdl_wait();  // operands / epilogue inputs are the previous kernels' outputs
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0) {
    // ============================ TMA producer (both CTAs; bytes land on the leader's barrier)
    setmaxnreg_dec<64>();
    if (elect_one()) {
      uint32_t it = 0;
      for (int u = cid; u < P.total_units; u += ncl) {
        const Unit U = decode_unit(P, u);
        const KProb& q = P.p[U.p];
        const int n0 = U.n0 * BN + 128 * (int)rank;
        const int m0 = U.m0 + 128 * (int)rank;
        SegCursor sc;
        sc.init(q, U.kb_lo);
        for (int kb = U.kb_lo; kb < U.kb_hi; ++kb, ++it, sc.next(q)) {
          const uint32_t stage = it % C::STAGES, use = it / C::STAGES;
          if (use > 0) mbar_wait(&empty[stage], (use - 1) & 1);
          const int k0 = sc.kk * BK;
          const CUtensorMap* mA = &P.mA[U.p][sc.seg];
          const CUtensorMap* mB = &P.mB[U.p][sc.seg];
          uint8_t* sA = smem + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + C::A_BYTES;
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          if (!sc.a_mn) {
            tma_load_2d_pair(sA, mA, fb, k0, m0);
          } else {
            tma_load_2d_pair(sA, mA, fb, m0, k0);
            tma_load_2d_pair(sA + 8192, mA, fb, m0 + 64, k0);
          }
          if (!sc.b_mn) {
            tma_load_2d_pair(sB, mB, fb, k0, n0);
          } else {
            tma_load_2d_pair(sB, mB, fb, n0, k0);
            tma_load_2d_pair(sB + 8192, mB, fb, n0 + 64, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer (leader CTA only)
    setmaxnreg_dec<64>();
    if (leader && elect_one()) {
      uint32_t it = 0, tc = 0;
      for (int u = cid; u < P.total_units; u += ncl, ++tc) {
        const Unit U = decode_unit(P, u);
        const KProb& q = P.p[U.p];
        const uint32_t buf = tc & 1, use = tc >> 1;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        const uint32_t fmask = q.f16 ? ~((7u << 7) | (7u << 10)) : ~0u;  // F16: format 0
        SegCursor sc;
        sc.init(q, U.kb_lo);
        for (int kb = U.kb_lo; kb < U.kb_hi; ++kb, ++it, sc.next(q)) {
          const uint32_t stage = it % C::STAGES, suse = it / C::STAGES;
          mbar_wait(&full[stage], suse & 1);
          tc_fence_after();
          const uint32_t a_mn = sc.a_mn, b_mn = sc.b_mn;
          const uint32_t idesc = idesc_bf16(256, BN, a_mn, b_mn) & fmask;
          const uint32_t sA = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sB = sA + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = a_mn ? smem_desc(sA + k * 2048, 8192, 1024, SWZ_128B)
                                     : smem_desc(sA + k * 32, 16, 1024, SWZ_128B);
            const uint64_t bd = b_mn ? smem_desc(sB + k * 2048, 8192, 1024, SWZ_128B)
                                     : smem_desc(sB + k * 32, 16, 1024, SWZ_128B);
            mma_bf16_ss_pair(d_tmem, ad, bd, idesc, (kb > U.kb_lo || k > 0) ? 1u : 0u);
          }
          mma_commit_pair_mc(&empty[stage], 0x3);
        }
        mma_commit_pair_mc(&tfull[buf], 0x3);
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<64>();
  } else {
    // ============================ epilogue (both CTAs: 128 rows x 256 columns each)
    setmaxnreg_inc<216>();
    const uint32_t quarter = warp & 3;
    const int half = (warp - 4) >> 2;
    const uint32_t stg = smem_u32(smem + C::STG_OFF) + (warp - 4) * 4096;
    const uint32_t te_remote = mapa_shared(smem_u32(&tempty[0]), 0);
    uint32_t tc = 0;
    for (int u = cid; u < P.total_units; u += ncl, ++tc) {
      const Unit U = decode_unit(P, u);
      const KProb& q = P.p[U.p];
      // the epilogue parameters in registers for the whole tile (parameter-space reads would be
      // repeated after every TMEM / barrier wait, which clobber memory)
      const EpiParams e = q.epi;
      const int qM = q.M, qN = q.N;
      const uint32_t buf = tc & 1, use = tc >> 1;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int row0 = U.m0 + 128 * (int)rank + quarter * 32;
      const int n0 = U.n0 * BN;
      // the primary epilogue input of slice c + 2 is requested before slice c is processed
      const void* pb = epi_primary(e);
      uint4 g[4];
      auto issue = [&](int c) {
        const int n0c = n0 + c * 32;
        if (c < BN / 32 && n0c < qN && row0 < qM && pb)
          warp_ldg_rows_bf16(pb, (size_t)row0 * e.ldo + n0c, e.ldo, qM - row0, g);
      };
      issue(half);
      for (int c = half; c < BN / 32; c += 2) {
        const int n0c = n0 + c * 32;
        if (n0c >= qN) break;
        uint4 cur[4] = {g[0], g[1], g[2], g[3]};
        issue(c + 2);
        uint32_t r[32];
        tmem_ld32(tmem_addr(tmem_base, quarter, buf * BN + c * 32), r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        run_epilogue_warp<MODES>(e, row0, qM, n0c, v, stg, pb ? cur : nullptr, U.ks);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[buf]);
        else
          mbar_arrive_cluster(te_remote + buf * 8);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
}

// ---------------------------------------------------------------- host
static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool make_operand_map(CUtensorMap* m, const OperandDesc& o, int box_rows_kmajor, int tf32) {
  const uint64_t ld = o.ld > 0 ? (uint64_t)o.ld : (uint64_t)o.cols;
  if (tf32) {  // fp32 K-major: 32-element (128-byte) K boxes, TMA zero-fills the K tail
    if (o.mn_major || (ld * 4) % 16) return false;
    uint64_t dims[2] = {(uint64_t)o.cols, (uint64_t)o.rows};
    uint64_t strides[1] = {ld * 4};
    uint32_t box[2] = {32, (uint32_t)box_rows_kmajor};
    return encode_map(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, o.ptr, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  uint64_t dims[2] = {(uint64_t)o.cols, (uint64_t)o.rows};
  uint64_t strides[1] = {ld * 2};
  uint32_t box[2];
  if (!o.mn_major) {
    box[0] = 64;
    box[1] = (uint32_t)box_rows_kmajor;
  } else {
    box[0] = 64;
    box[1] = 64;
  }
  return encode_bf16_map(m, o.ptr, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <uint32_t MODES>
static cudaError_t launch_pair(const GemmKParams& P, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(gemm_pair_kernel<MODES>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int pairs = num_sms() / 2;
  if (P.total_units < pairs) pairs = P.total_units;
  ProfScope ps(PROF_GEMM, stream, 1);
  {
    const cudaError_t e = launch_pdl(gemm_pair_kernel<MODES>, dim3(2 * pairs), dim3(GEMM_THREADS), PairCfg::SMEM,
                                     stream, P);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// the mode sets the layer launches get their own instantiation; anything else runs the all-modes one
static cudaError_t launch_pair_modes(const GemmKParams& P, uint32_t modes, cudaStream_t stream) {
  if (modes & MB(EPI_TAPS)) return launch_pair<MODES_ALL | MB(EPI_TAPS)>(P, stream);  // parity taps
  switch (modes) {
    case MB(EPI_STORE): return launch_pair<MB(EPI_STORE)>(P, stream);
    case MB(EPI_GATE): return launch_pair<MB(EPI_GATE)>(P, stream);
    case MB(EPI_STORE) | MB(EPI_ATOMIC): return launch_pair<MB(EPI_STORE) | MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_GATE_BWD) | MB(EPI_ATOMIC): return launch_pair<MB(EPI_GATE_BWD) | MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_ATOMIC): return launch_pair<MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_HEAD): return launch_pair<MB(EPI_HEAD)>(P, stream);
    case MB(EPI_GELU): return launch_pair<MB(EPI_GELU)>(P, stream);
    case MB(EPI_GELU_BWD) | MB(EPI_ATOMIC): return launch_pair<MB(EPI_GELU_BWD) | MB(EPI_ATOMIC)>(P, stream);
    default: return launch_pair<MODES_ALL>(P, stream);
  }
}

template <int BN, uint32_t MODES>
static cudaError_t launch_bn(const GemmKParams& P, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, MODES>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = P.total_units < num_sms() ? P.total_units : num_sms();
  ProfScope ps(PROF_GEMM, stream, 1);
  {
    const cudaError_t e = launch_pdl(gemm_kernel<BN, MODES>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, stream, P);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <int BN>
static cudaError_t launch_bn_modes(const GemmKParams& P, uint32_t modes, cudaStream_t stream) {
  if (modes & MB(EPI_TAPS)) return launch_bn<BN, MODES_ALL | MB(EPI_TAPS)>(P, stream);  // parity taps
  switch (modes) {
    case MB(EPI_STORE): return launch_bn<BN, MB(EPI_STORE)>(P, stream);
    case MB(EPI_GATE): return launch_bn<BN, MB(EPI_GATE)>(P, stream);
    case MB(EPI_STORE) | MB(EPI_ATOMIC): return launch_bn<BN, MB(EPI_STORE) | MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_GATE_BWD) | MB(EPI_ATOMIC): return launch_bn<BN, MB(EPI_GATE_BWD) | MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_ATOMIC): return launch_bn<BN, MB(EPI_ATOMIC)>(P, stream);
    case MB(EPI_HEAD): return launch_bn<BN, MB(EPI_HEAD)>(P, stream);
    case MB(EPI_GELU): return launch_bn<BN, MB(EPI_GELU)>(P, stream);
    case MB(EPI_GELU_BWD) | MB(EPI_ATOMIC): return launch_bn<BN, MB(EPI_GELU_BWD) | MB(EPI_ATOMIC)>(P, stream);
    default: return launch_bn<BN, MODES_ALL>(P, stream);
  }
}

cudaError_t gemm_launch(const GemmProblem* probs, int nprob, int bn, cudaStream_t stream) {
  if (nprob < 1 || nprob > GEMM_MAX_PROB || (bn != 128 && bn != 256)) return cudaErrorInvalidValue;
  static GemmKParams P;  // large; filled per launch (host-side only)
  memset(&P, 0, sizeof(P));
  P.nprob = nprob;
  // CTA pairs (cta_group::2, 256 x 256 tiles) whenever the N tile is 256 and every M spans a pair tile
  bool pair = bn == 256;
  for (int p = 0; p < nprob; ++p) pair = pair && probs[p].M >= 256 && !probs[p].tf32;
  P.bm = pair ? 256 : BM;
  int total = 0;
  for (int p = 0; p < nprob; ++p) {
    const GemmProblem& g = probs[p];
    KProb& q = P.p[p];
    if (g.M <= 0 || g.N <= 0 || g.N % 32 != 0 || g.nseg < 1 || g.nseg > GEMM_MAX_SEG) return cudaErrorInvalidValue;
    q.M = g.M;
    q.N = g.N;
    q.nseg = g.nseg;
    q.kb_total = 0;
    for (int s = 0; s < g.nseg; ++s) {
      const OperandDesc& A = g.A[s];
      const OperandDesc& B = g.B[s];
      if ((!g.tf32 && (A.cols % 8 || B.cols % 8)) || g.K[s] <= 0) return cudaErrorInvalidValue;
      if (!make_operand_map(&P.mA[p][s], A, BM, g.tf32)) return cudaErrorInvalidValue;
      if (!make_operand_map(&P.mB[p][s], B, pair ? 128 : bn, g.tf32)) return cudaErrorInvalidValue;
      q.a_mn[s] = A.mn_major;
      q.b_mn[s] = B.mn_major;
      const int bke = g.tf32 ? BK / 2 : BK;
      q.kb[s] = (g.K[s] + bke - 1) / bke;
      q.kb_total += q.kb[s];
    }
    q.split_k = g.split_k < 1 ? 1 : (g.split_k > q.kb_total ? q.kb_total : g.split_k);
    q.f16 = g.f16;
    q.tf32 = g.tf32;
    q.m_tiles = (g.M + P.bm - 1) / P.bm;
    q.n_tiles = (g.N + bn - 1) / bn;
    q.unit_begin = total;
    q.epi = g.epi;
    total += q.m_tiles * q.n_tiles * q.split_k;
  }
  P.total_units = total;
  uint32_t modes = 0;
  for (int p = 0; p < nprob; ++p) {
    modes |= MB(probs[p].epi.mode);
    if (probs[p].epi.tap || probs[p].epi.tap2) modes |= MB(EPI_TAPS);
  }
  if (pair) return launch_pair_modes(P, modes, stream);
  return bn == 256 ? launch_bn_modes<256>(P, modes, stream) : launch_bn_modes<128>(P, modes, stream);
}

}  // namespace cadet
