// Shared geometry of the attention kernels (rows A5 / A10).
#pragma once
#include "plan.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace cadet {

// Head-dim tiling: a [128 x HDP] operand tile is held as NB column blocks of CB bf16 columns,
// each block a [128 rows x RB bytes] TMA box with RB-byte swizzle (RB = 128 when hd % 64 == 0,
// else 64).  hd = 88 runs as HDP = 96: TMA zero-fills columns 88..95 of the 3-D [T][H][hd] map.
template <int HD>
struct HeadGeom {
  static constexpr int HDP = (HD + 31) / 32 * 32;
  static constexpr int RB = (HDP % 64 == 0) ? 128 : 64;  // row bytes per block = swizzle width
  static constexpr int CB = RB / 2;                       // bf16 columns per block
  static constexpr int NB = HDP / CB;
  static constexpr int BLK = 128 * RB;                    // bytes per block
  static constexpr int TILE_BYTES = NB * BLK;
  static constexpr uint32_t SWZ = (RB == 128) ? SWZ_128B : SWZ_64B;
};

// K-major operand (rows x HDP) descriptor for k-step kk (16 columns).
template <int HD>
CADET_DEV uint64_t kmajor_desc(uint32_t base, int kk) {
  using G = HeadGeom<HD>;
  const int col = kk * 16;
  const uint32_t addr = base + (col / G::CB) * G::BLK + (col % G::CB) * 2;
  return smem_desc(addr, 16, 8 * G::RB, G::SWZ);
}
// MN-major operand: storage rows = K dimension (16 rows per k-step), columns = N (HDP).
template <int HD>
CADET_DEV uint64_t mnmajor_desc(uint32_t base, int kk) {
  using G = HeadGeom<HD>;
  return smem_desc(base + kk * 16 * G::RB, G::BLK, 8 * G::RB, G::SWZ);
}

// 128 x 128 bf16 tile written by threads (P, P^T, dS^T): 2 blocks of 64 columns, 128B swizzle.
CADET_DEV uint32_t p_off(int row, int col) {  // byte offset of the 8-column chunk holding col
  return (col >> 6) * 16384 + swz_off(row, (col & 63) >> 3, 128);
}
CADET_DEV uint64_t p_kmajor_desc(uint32_t base, int kk) {  // A operand, K = columns
  return smem_desc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, SWZ_128B);
}
CADET_DEV uint64_t p_mnmajor_desc(uint32_t base, int kk) {  // A operand MN-major: M = columns, K = rows
  return smem_desc(base + kk * 16 * 128, 16384, 1024, SWZ_128B);
}

// Visible-key bitmask of query row r over the 32 keys [kc, kc + 32): the prefix [.., e_r), the
// diagonal r and, with the PAIR_PREV bit, r - 1 (SURVEY 8(c) mask structure; Fig. 3).
CADET_DEV uint32_t row_mask32(int e_r, int r, bool pp, int kc) {
  const int lim = e_r - kc;
  uint32_t m = lim >= 32 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
  const int dd = r - kc;
  if (dd >= 0 && dd < 32) m |= 1u << dd;
  if (pp && dd - 1 >= 0 && dd - 1 < 32) m |= 1u << (dd - 1);
  return m;
}

// 2^x for two cells at once on the FMA / ALU pipes (FA4-style MUFU offload): n = rint(x) (1.5 * 2^23
// trick), 2^f on [-1/2, 1/2] by a degree-3 relative-minimax polynomial (max rel err 7.5e-5, far below
// the bf16 rounding of P), n added to the exponent field.  x < -126 (incl. -inf: masked cells) gives
// exactly 0 like ex2.approx.ftz.  Packed f32x2 FADD / FFMA (sm_100) for the float arithmetic.
CADET_DEV float2 exp2_poly3x2(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(xc, magic);
  const float2 f = __fadd2_rn(xc, __fadd2_rn(magic, make_float2(-t.x, -t.y)));
  float2 q = __ffma2_rn(make_float2(0.05516947f, 0.05516947f), f, make_float2(0.24260798f, 0.24260798f));
  q = __ffma2_rn(q, f, make_float2(0.69326111f, 0.69326111f));
  q = __ffma2_rn(q, f, make_float2(0.99992828f, 0.99992828f));
  const float r0 = __int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23));
  const float r1 = __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23));
  return make_float2(x.x < -126.f ? 0.f : r0, x.y < -126.f ? 0.f : r1);
}

struct AttnParams {
  int32_t T, H, hd, d, n;
  float scale_log2;  // log2(e) / sqrt(hd)
  float scale;       // 1 / sqrt(hd)
  int32_t out_f32;
  const int32_t* cu;
  PlanView plan;
  void* O;           // fwd: O out;  bwd: (unused)
  float* lse;        // fwd out / bwd in  [H, T]
  const float* D;    // bwd: rowsum(dO * O) [H, T]
  void* dQ;          // bwd: dQ [T, d], fp32 (core ABI) or bf16 (dq_bf16: the layer path)
  int32_t dq_bf16;
  void* dK;          // bwd out
  void* dV;          // bwd out
  // forward split-KV (small grids, e.g. one serving request): each (q-tile, head) split into
  // fwd_splits CTAs over its visit list, writing unnormalised fp32 partials merged afterwards
  int32_t fwd_splits;
  float* Opart;      // [splits][T][d]
  float* Mpart;      // [splits][H][T] running max (log2 units) of the split
  float* Lpart;      // [splits][H][T] row sum of the split (0 = empty split)
  // two-pass backward (layer path, when the workspace holds the dS region): attn_bwd_dkv_kernel
  // stores every visited dS^T tile (bf16, unscaled) at slot tri_off[seq] + qt (qt + 1) / 2 + kt,
  // rows slot * 128 + key, head h at columns [128 h, 128 h + 128); attn_bwd_dq2_kernel then forms
  // dQ = dS K from those tiles instead of recomputing S and dP
  void* dS;          // nullptr: single-pass dQ kernel (recompute)
  int32_t ds_slots;
};

}  // namespace cadet
