// A5: packed, session-masked attention forward (Eq. 7).
//
// One CTA per (128-row q-tile of one sequence, head), q-tiles taken in descending cost order
// (LPT work list from the plan).  Only the visible k-tiles are visited: the front prefix
// [0, nf) and the diagonal band [kt2, qt] ("skips compute_qk entirely for tiles
// that are fully masked").  Per row, the mask predicate runs only when the row's visible
// prefix does not cover the whole k-tile (PARTIAL rows); FULL rows skip it.
//
//   warp 0     : TMA producer: Q once, then K_j / V_j (single-buffered, 3-D [T][H][hd] maps)
//   warp 1     : TMEM owner + tcgen05.mma issuer: S_j = Q K_j^T into TMEM; O += P_j V_j with
//                P_j read from TMEM (TS form: P overwrites the consumed S columns as packed bf16);
//                by default each K tile runs as two 64-key halves with their own S buffers
//                (PV_a(j), S_a(j+1), PV_b(j), S_b(j+1)), so one half's softmax overlaps the other's MMAs
//   warps 2..5 : softmax, thread = query row: tcgen05.ld S, mask, online softmax with
//                conditional rescaling (threshold 2^8), tcgen05.st P, O rescale, final O / l, LSE.
// ~96 KB of shared memory and 256 TMEM columns per CTA, so two CTAs share an SM and one CTA's
// softmax overlaps the other's MMAs (the role FA4's two softmax warpgroups play).
#include <algorithm>
#include <cstdlib>

#include "attn_common.cuh"
#include "launch.cuh"
#include "prof.cuh"

namespace cadet {

#ifdef CADET_PHASE_TIMING
__device__ unsigned long long g_phase_fwd[8192][16];
#define FT_MARK(slot)                                                              \
  if (lane == 0 && blockIdx.x < 8192) {                                             \
    unsigned long long _n = clock64();                                              \
    atomicAdd(&g_phase_fwd[blockIdx.x][slot], _n - _ft);                            \
    _ft = _n;                                                                       \
  }
#define PP_DECL unsigned long long _pp = clock64(), _pacc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define PP_MARK(slot)                    \
  {                                      \
    unsigned long long _n = clock64();   \
    _pacc[slot] += _n - _pp;             \
    _pp = _n;                            \
  }
#define PP_FLUSH(lo, hi)                                                                  \
  if (blockIdx.x < 8192)                                                                  \
    for (int _i = lo; _i < hi; ++_i) atomicAdd(&g_phase_fwd[blockIdx.x][_i], _pacc[_i]);
#else
#define FT_MARK(slot)
#define PP_DECL
#define PP_MARK(slot)
#define PP_FLUSH(lo, hi)
#endif

// FWD1_NPOLY of every 16 exponentials on the FMA pipe (exp2_poly3x2): 4 helped the single-S kernel
// (~3 %); with the 64-key halves the issue slots, not the MUFU pipe, bind and 0 is fastest
#ifndef FWD1_NPOLY
#define FWD1_NPOLY 0
#endif
// Each 128-key tile as two 64-key halves with their own S buffers and online-softmax steps, so one
// half's softmax overlaps the other half's S / PV MMAs inside the CTA (C4 forward -7..-11 %, same-box
// A/B); FWD_ONE_S builds the single-S variant (S -> softmax -> PV strictly in sequence per CTA).
#ifndef FWD_ONE_S
#define FWD_HALVES 1
#endif
template <int HD>
struct FwdCfg {
  using G = HeadGeom<HD>;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + G::TILE_BYTES;
  static constexpr int V_OFF = K_OFF + G::TILE_BYTES;
  static constexpr int BAR_OFF = V_OFF + G::TILE_BYTES;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int S_COL = 0;    // S (fp32, 128 columns); P (bf16 pairs) reuses columns [0, 64)
  static constexpr int O_COL = 128;  // HDP fp32 columns
  static constexpr uint32_t TMEM_COLS = 256;
};

struct FwdBars {
  uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, p_full, pv_done;
  uint64_t sh_full[2], ph_full[2], pvh_done[2];  // FWD_HALVES: per 64-key half of the tile
  uint32_t tmem_base;
};

__device__ __forceinline__ int visit_tile(const QTileInfo& qi, int j) { return j < qi.nf ? j : qi.kt2 + (j - qi.nf); }

template <int HD>
__global__ void __launch_bounds__(192, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = FwdCfg<HD>;
  pdl_wait();  // not persistent: the whole kernel reads the previous kernels' outputs
  const int nq_total = p.plan.counters[0];
  const int S = p.fwd_splits;
  const int b = blockIdx.x / (p.H * S);
  const int h = (blockIdx.x % (p.H * S)) % p.H;
  const int sp = (blockIdx.x % (p.H * S)) / p.H;  // split index: visit-list slice [j0, j0 + n_kv)
  if (b >= nq_total) return;
  const QTileInfo qi = p.plan.qinfo[p.plan.fwd_order[b]];
  const int sa = p.cu[qi.seq], se = p.cu[qi.seq + 1];
  const int q0 = sa + qi.qt * 128;
  const int rows_valid = min(128, se - q0);
  const int n_all = qi.nf + (qi.qt + 1 - qi.kt2);
  const int chunk = (n_all + S - 1) / S;
  const int j0 = min(n_all, sp * chunk);
  const int n_kv = min(n_all, j0 + chunk) - j0;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + C::BAR_OFF);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->k_full, 1);
    mbar_init(&bars->k_empty, 1);
    mbar_init(&bars->v_full, 1);
    mbar_init(&bars->v_empty, 1);
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->pv_done, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->sh_full[i], 1);
      mbar_init(&bars->ph_full[i], 128);
      mbar_init(&bars->pvh_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first

  if (warp == 0) {
    // ============================ producer
    if (elect_one()) {
      mbar_expect_tx(&bars->q_full, G::TILE_BYTES);
#pragma unroll
      for (int blk = 0; blk < G::NB; ++blk)
        tma_load_3d(smem + C::Q_OFF + blk * G::BLK, &mQ, &bars->q_full, blk * G::CB, h, q0);
      for (int j = 0; j < n_kv; ++j) {
        const int krow = sa + visit_tile(qi, j0 + j) * 128;
        if (j > 0) mbar_wait(&bars->k_empty, (j - 1) & 1);
        mbar_expect_tx(&bars->k_full, G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk)
          tma_load_3d(smem + C::K_OFF + blk * G::BLK, &mK, &bars->k_full, blk * G::CB, h, krow);
        if (j > 0) mbar_wait(&bars->v_empty, (j - 1) & 1);
        mbar_expect_tx(&bars->v_full, G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk)
          tma_load_3d(smem + C::V_OFF + blk * G::BLK, &mV, &bars->v_full, blk * G::CB, h, krow);
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = idesc_bf16(128, G::HDP, 0, 1);
      const uint32_t sQ = smem_u32(smem + C::Q_OFF);
      const uint32_t sK = smem_u32(smem + C::K_OFF);
      const uint32_t sV = smem_u32(smem + C::V_OFF);
#ifdef CADET_PHASE_TIMING
      unsigned long long _ft = clock64();
#endif
      mbar_wait(&bars->q_full, 0);
      FT_MARK(0)
#ifdef FWD_HALVES
      // each K tile as two 64-key halves with their own S buffers (S_a cols [0, 64), S_b [64, 128)), so the
      // softmax of one half overlaps the other half's MMAs: PV_a(j), S_a(j+1), PV_b(j), S_b(j+1), ...
      const uint32_t idesc_h = idesc_bf16(128, 64, 0, 0);
      auto issue_s = [&](int hh) {  // S_hh = Q K[64 hh .. 64 hh + 64)^T
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::S_COL + hh * 64, kmajor_desc<HD>(sQ, kk), kmajor_desc<HD>(sK + hh * 64 * G::RB, kk),
                      idesc_h, kk > 0 ? 1u : 0u);
        mma_commit(&bars->sh_full[hh]);
      };
      if (n_kv > 0) {
        mbar_wait(&bars->k_full, 0);
        tc_fence_after();
        issue_s(0);
        issue_s(1);
        mma_commit(&bars->k_empty);
      }
      for (int j = 0; j < n_kv; ++j) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait(&bars->ph_full[hh], j & 1);
          if (hh == 0) mbar_wait(&bars->v_full, j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 64 / 16; ++kk)  // packed P of the half's keys at its first 32 columns
            mma_bf16_ts(tmem + C::O_COL, tmem + C::S_COL + hh * 64 + kk * 8, mnmajor_desc<HD>(sV, hh * 4 + kk),
                        idesc_o, (j > 0 || hh > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars->pvh_done[hh]);
          if (hh == 1) mma_commit(&bars->v_empty);
          if (j + 1 < n_kv) {
            if (hh == 0) {
              mbar_wait(&bars->k_full, (j + 1) & 1);
              tc_fence_after();
            }
            issue_s(hh);  // over P_hh(j): after PV_hh(j) in issue order
            if (hh == 1) mma_commit(&bars->k_empty);
          }
        }
      }
      if (n_kv > 0) mma_commit(&bars->pv_done);  // once: the epilogue waits parity 0
#else
      for (int j = 0; j < n_kv; ++j) {
        // S_j: the tensor pipe executes in issue order, so S_j overwrites P_{j-1} only after PV_{j-1}
        // has read it; p_full(j-1) (waited below) guarantees the softmax finished with S_{j-1}.
        mbar_wait(&bars->k_full, j & 1);
        FT_MARK(1)
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::S_COL, kmajor_desc<HD>(sQ, kk), kmajor_desc<HD>(sK, kk), idesc_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->k_empty);
        mma_commit(&bars->s_full);
        mbar_wait(&bars->p_full, j & 1);
        FT_MARK(2)
        mbar_wait(&bars->v_full, j & 1);
        FT_MARK(3)
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)  // packed P of keys [32c, 32c + 32) at columns [32c, 32c + 16)
          mma_bf16_ts(tmem + C::O_COL, tmem + C::S_COL + (kk >> 1) * 32 + (kk & 1) * 8, mnmajor_desc<HD>(sV, kk),
                      idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&bars->v_empty);
        mma_commit(&bars->pv_done);
      }
#endif
    }
  } else {
    // ============================ softmax warps 2..5
    const uint32_t quarter = warp & 3;
    const int rt = quarter * 32 + lane;  // row in tile == TMEM lane
    const int r = q0 + rt;
    const bool valid = rt < rows_valid;
    const int e_r = valid ? p.plan.kv_end[r] : 0;
    const bool pp = valid ? (p.plan.row_pp[r] != 0) : false;
    const float sl2 = p.scale_log2;
    float m_used = -INFINITY;  // scaled (log2) running max actually used as the exp base
    float l = 0.f;
#ifdef CADET_PHASE_TIMING
    unsigned long long _ft = clock64();
    const uint32_t lane_save = lane;
#define lane (threadIdx.x == 64 ? 0u : 1u)
#endif
#ifdef FWD_HALVES
    // per tile j, the two 64-key halves as separate online-softmax steps (same running max / sum)
    for (int j = 0; j < n_kv; ++j) {
      const int k0 = sa + visit_tile(qi, j0 + j) * 128;
      const bool partial = !valid || (e_r < k0 + 128);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        mbar_wait(&bars->sh_full[hh], j & 1);
        tc_fence_after();
        uint32_t sv[2][32];
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + hh * 64), sv[0]);
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + hh * 64 + 32), sv[1]);
        tmem_ld_wait();
        if (partial) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t m = valid ? row_mask32(e_r, r, pp, k0 + hh * 64 + c * 32) : 0u;
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (!((m >> q) & 1u)) sv[c][q] = __float_as_uint(-INFINITY);
          }
        }
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          m0 = fmaxf(m0, fmaxf(__uint_as_float(sv[0][q]), __uint_as_float(sv[0][q + 1])));
          m1 = fmaxf(m1, fmaxf(__uint_as_float(sv[1][q]), __uint_as_float(sv[1][q + 1])));
        }
        const float mx_s = fmaxf(m0, m1) * sl2;
        float factor = 1.f;
        bool rescale = false;
        if (mx_s > m_used + 8.f) {  // conditional rescale (also the first finite max)
          factor = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx_s);
          m_used = mx_s;
          rescale = true;
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2v = make_float2(sl2, sl2), nbase = make_float2(-base, -base);
        float2 rs2 = make_float2(0.f, 0.f);
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[c][q]), __uint_as_float(sv[c][q + 1])), sl2v, nbase);
            const float2 pp2 = ((q & 15) + 2 > 16 - FWD1_NPOLY) ? exp2_poly3x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
            rs2 = __fadd2_rn(rs2, pp2);
            w[c * 16 + (q >> 1)] = pack_bf16(pp2.x, pp2.y);
          }
        tmem_st32(tmem_addr(tmem, quarter, C::S_COL + hh * 64), w);
        // O rescale (rare): every earlier PV must be complete -- the other half's latest PV is the only one
        // the S commit does not cover (PV_b(j-1) for half a, PV_a(j) for half b)
        if (__any_sync(0xffffffffu, rescale) && (j > 0 || hh > 0)) {
          if (hh == 0) mbar_wait(&bars->pvh_done[1], (j - 1) & 1);
          else mbar_wait(&bars->pvh_done[0], j & 1);
          tc_fence_after();
          const float f = rescale ? factor : 1.f;
#pragma unroll
          for (int c = 0; c < G::HDP / 32; ++c) {
            uint32_t u[32];
            const uint32_t ta = tmem_addr(tmem, quarter, C::O_COL + c * 32);
            tmem_ld32(ta, u);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q) u[q] = __float_as_uint(__uint_as_float(u[q]) * f);
            tmem_st32(ta, u);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars->ph_full[hh]);
        l = l * factor + (rs2.x + rs2.y);
      }
    }
#else
    for (int j = 0; j < n_kv; ++j) {
      const int k0 = sa + visit_tile(qi, j0 + j) * 128;
      // s_full(j) also implies PV_{j-1} completed (commit tracks all prior tcgen05 ops)
      mbar_wait(&bars->s_full, j & 1);
      FT_MARK(4)
      tc_fence_after();
      const bool partial = !valid || (e_r < k0 + 128);
      auto mask32 = [&](int c, uint32_t (&u)[32]) {
        if (partial) {
          const uint32_t m = valid ? row_mask32(e_r, r, pp, k0 + c * 32) : 0u;
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (!((m >> q) & 1u)) u[q] = __float_as_uint(-INFINITY);
        }
      };
      // pass 1: row max over two batches of two chunks (two loads in flight per wait); chunks 2, 3
      // stay in registers for pass 2
      float mx = -INFINITY;
      uint32_t s2[32], s3[32];
      {
        uint32_t s0[32], s1[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL), s0);
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + 32), s1);
        tmem_ld_wait();
        mask32(0, s0);
        mask32(1, s1);
#pragma unroll
        for (int q = 0; q < 32; ++q) mx = fmaxf(mx, fmaxf(__uint_as_float(s0[q]), __uint_as_float(s1[q])));
      }
      tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + 64), s2);
      tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + 96), s3);
      tmem_ld_wait();
      mask32(2, s2);
      mask32(3, s3);
#pragma unroll
      for (int q = 0; q < 32; ++q) mx = fmaxf(mx, fmaxf(__uint_as_float(s2[q]), __uint_as_float(s3[q])));
      FT_MARK(5)
      const float mx_s = mx * sl2;
      float factor = 1.f;
      bool rescale = false;
      if (mx_s > m_used + 8.f) {  // conditional rescale (also the first finite max)
        factor = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx_s);
        m_used = mx_s;
        rescale = true;
      }
      if (j > 0 && __any_sync(0xffffffffu, rescale)) {
        const float f = rescale ? factor : 1.f;
#pragma unroll
        for (int c = 0; c < G::HDP / 32; ++c) {
          uint32_t u[32];
          const uint32_t ta = tmem_addr(tmem, quarter, C::O_COL + c * 32);
          tmem_ld32(ta, u);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 32; ++q) u[q] = __float_as_uint(__uint_as_float(u[q]) * f);
          tmem_st32(ta, u);
        }
      }
      // pass 2: P = exp2(s * scale_log2 - m) as packed bf16; chunk c's P lands in the first 16 of its
      // own 32 columns (chunks 2, 3 from registers first, then chunks 0, 1 reloaded)
      const float base = (m_used == -INFINITY) ? 0.f : m_used;
      float rs = 0.f;
      // packed f32x2 math; FWD1_NPOLY of every 16 cells' exponentials on the FMA pipe (MUFU offload)
      const float2 sl2v = make_float2(sl2, sl2), nbase = make_float2(-base, -base);
      float2 rs2 = make_float2(0.f, 0.f);
      auto exp_store = [&](int c, const uint32_t (&u)[32]) {
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(u[q]), __uint_as_float(u[q + 1])), sl2v, nbase);
          const float2 pp = ((q & 15) + 2 > 16 - FWD1_NPOLY) ? exp2_poly3x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
          rs2 = __fadd2_rn(rs2, pp);
          w[q >> 1] = pack_bf16(pp.x, pp.y);
        }
        tmem_st16(tmem_addr(tmem, quarter, C::S_COL + c * 32), w);
      };
      exp_store(2, s2);
      exp_store(3, s3);
      {
        uint32_t s0[32], s1[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL), s0);
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + 32), s1);
        tmem_ld_wait();
        mask32(0, s0);
        mask32(1, s1);
        exp_store(0, s0);
        exp_store(1, s1);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      l = l * factor + (rs + rs2.x + rs2.y);
      FT_MARK(6)
    }
#endif
#ifdef CADET_PHASE_TIMING
#undef lane
    (void)lane_save;
#endif
    // ---- epilogue: O / l, LSE
    if (n_kv > 0) {
#ifdef FWD_HALVES
      mbar_wait(&bars->pv_done, 0);
#else
      mbar_wait(&bars->pv_done, (n_kv - 1) & 1);
#endif
      tc_fence_after();
    }
    if (S > 1) {  // split-KV partial: unnormalised O, the split's max (log2 units) and row sum
      if (valid) {
        p.Mpart[((size_t)sp * p.H + h) * p.T + r] = m_used;
        p.Lpart[((size_t)sp * p.H + h) * p.T + r] = l;
      }
#pragma unroll 1
      for (int c = 0; c < G::HDP / 32 && n_kv > 0; ++c) {
        uint32_t u[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::O_COL + c * 32), u);
        tmem_ld_wait();
        if (valid) {
          float* o = p.Opart + ((size_t)sp * p.T + r) * p.d + (size_t)h * p.hd + c * 32;
          const int ncol = min(32, p.hd - c * 32);
          for (int q = 0; q < ncol; q += 4)
            *reinterpret_cast<float4*>(o + q) = make_float4(__uint_as_float(u[q]), __uint_as_float(u[q + 1]),
                                                            __uint_as_float(u[q + 2]), __uint_as_float(u[q + 3]));
        }
      }
    }
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
#pragma unroll
    for (int c = 0; c < G::HDP / 32 && S == 1; ++c) {
      uint32_t u[32];
      tmem_ld32(tmem_addr(tmem, quarter, C::O_COL + c * 32), u);
      tmem_ld_wait();
      if (!p.out_f32) {  // bf16 O through a per-warp transpose in the (now idle) Q tile: coalesced rows
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          w[q] = pack_bf16(__uint_as_float(u[2 * q]) * inv_l, __uint_as_float(u[2 * q + 1]) * inv_l);
        warp_store_rows_bf16(smem_u32(smem + C::Q_OFF) + (warp - 2) * 2048, w,
                             reinterpret_cast<__nv_bfloat16*>(p.O) + (size_t)(q0 + quarter * 32) * p.d +
                                 (size_t)h * p.hd + c * 32,
                             p.d, rows_valid - (int)quarter * 32, min(32, p.hd - c * 32));
      } else if (valid) {
        const size_t off = (size_t)r * p.d + (size_t)h * p.hd + c * 32;
        const int ncol = min(32, p.hd - c * 32);
        if (p.out_f32) {
          float* o = reinterpret_cast<float*>(p.O) + off;
          for (int q = 0; q < ncol; q += 4)
            *reinterpret_cast<float4*>(o + q) =
                make_float4(__uint_as_float(u[q]) * inv_l, __uint_as_float(u[q + 1]) * inv_l,
                            __uint_as_float(u[q + 2]) * inv_l, __uint_as_float(u[q + 3]) * inv_l);
        }
      }
    }
    if (valid && S == 1) p.lse[(size_t)h * p.T + r] = (l > 0.f) ? (m_used + __log2f(l)) * 0.6931471805599453f : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem);
}

// Split-KV merge: per row and head, rescale the splits' partials to the common max and normalise.
// Rows with no visible key in any split (pad rows) get O = 0, LSE = 0 (R17).
__global__ void __launch_bounds__(256) attn_fwd_merge_kernel(const AttnParams p) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int S = p.fwd_splits;
  if (row >= p.cu[p.n]) return;  // pad rows: zeroed by the caller, no partials
  for (int col = threadIdx.x * 4; col < p.d; col += blockDim.x * 4) {
    const int h = col / p.hd;
    float mstar = -INFINITY;
    for (int s = 0; s < S; ++s)
      if (p.Lpart[((size_t)s * p.H + h) * p.T + row] > 0.f) mstar = fmaxf(mstar, p.Mpart[((size_t)s * p.H + h) * p.T + row]);
    float lsum = 0.f, a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int s = 0; s < S; ++s) {
      const float ls = p.Lpart[((size_t)s * p.H + h) * p.T + row];
      if (ls > 0.f) {
        const float w = exp2f(p.Mpart[((size_t)s * p.H + h) * p.T + row] - mstar);
        const float4 o = *reinterpret_cast<const float4*>(p.Opart + ((size_t)s * p.T + row) * p.d + col);
        lsum += w * ls;
        a0 += w * o.x, a1 += w * o.y, a2 += w * o.z, a3 += w * o.w;
      }
    }
    const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
    if (p.out_f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.O) + (size_t)row * p.d + col) =
          make_float4(a0 * inv, a1 * inv, a2 * inv, a3 * inv);
    } else {
      uint2 v;
      v.x = pack_bf16(a0 * inv, a1 * inv);
      v.y = pack_bf16(a2 * inv, a3 * inv);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.O) + (size_t)row * p.d + col) = v;
    }
    if (col % p.hd == 0)
      p.lse[(size_t)h * p.T + row] = lsum > 0.f ? (mstar + __log2f(lsum)) * 0.6931471805599453f : 0.f;
  }
}

// ============================================================================ paired forward
// A5 as one persistent CTA per SM over (q-tile pair, head) items (plan pair_list; dynamic work
// counter, so the jagged items balance like the hardware's own CTA scheduling would).  An item is two
// q-tiles of one sequence (qt, qt - 1) that share one K / V stream: the union of their visit lists,
// each K / V tile loaded once for both.  Two softmax warpgroups, one per q-tile ("slot"), each with
// its own S and O accumulators in TMEM (S0 S1 O0 O1 = 512 columns), so that the tensor core computes
// one slot's S = Q K^T or O += P V while the other slot's softmax runs:
//   warp 0     : producer (work counter, item ring, Q per slot, K / V ring of STAGES)
//   warp 1     : TMEM owner + MMA issuer; per union tile u: PV of each slot's previous tile, then
//                S of the slots that see u (PV_s(prev) precedes S_s(u): P aliases S)
//   warps 4..7 : softmax of slot 0;  warps 8..11 : slot 1 (thread = query row): full S row in
//                registers, mask, conditional rescale (threshold 2^8), exp2 (a fraction on the FMA
//                pipe, exp2_poly3), P as packed bf16 over the row's S columns; item end: O / l, LSE.
template <int HD>
struct PairCfg {
  using G = HeadGeom<HD>;
  static constexpr int STAGES = HD <= 64 ? 3 : 2;
  static constexpr int Q_OFF = 0;                                   // 2 slots
  static constexpr int K_OFF = Q_OFF + 2 * G::TILE_BYTES;           // STAGES
  static constexpr int V_OFF = K_OFF + STAGES * G::TILE_BYTES;      // STAGES
  static constexpr int STG_OFF = V_OFF + STAGES * G::TILE_BYTES;    // [8 softmax warps][2 KB] O store transpose
  static constexpr int BAR_OFF = STG_OFF + 8 * 2048;
  // at least 116 KB: one CTA per SM (the 512 TMEM columns are the whole SM's)
  static constexpr int SMEM = (BAR_OFF + 1024 + 1024) > 118784 ? (BAR_OFF + 1024 + 1024) : 118784;
  static constexpr int THREADS = 384;
  static constexpr int RING = 4;  // item ring entries
};

struct PairItem {  // one decoded work item (the producer writes it into the ring)
  int w, h, sa, se, nslot, pad[3];
  QTileInfo qi[2];
};
struct PairBars {
  uint64_t q_full[2], q_empty[2], s_full[2], p_full[2], o_full[2], o_free[2];
  uint64_t k_full[3], k_empty[3], v_full[3], v_empty[3];
  uint64_t item_full[4], item_empty[4];
  uint32_t tmem_base;
  PairItem item[4];
};
static_assert(sizeof(PairBars) <= 1024, "pair kernel barrier block");
CADET_DEV void pair_item(const AttnParams& p, int w, PairItem& t) {
  t.w = w;
  if (w < 0) return;
  t.h = w % p.H;
  const int g = p.plan.pair_list[w / p.H];
  t.qi[0] = p.plan.qinfo[g];
  t.nslot = t.qi[0].qt >= 1 ? 2 : 1;
  t.qi[1] = t.nslot == 2 ? p.plan.qinfo[g - 1] : t.qi[0];
  t.sa = p.cu[t.qi[0].seq];
  t.se = p.cu[t.qi[0].seq + 1];
}
CADET_DEV bool tile_sees(const QTileInfo& qi, int kt) { return kt < qi.nf || (kt >= qi.kt2 && kt <= qi.qt); }
// next visited k-tile of the slot (or of the union) at or after kt; > qt when none is left
CADET_DEV int next_seen(const QTileInfo& qi, int kt) { return kt < qi.nf ? kt : max(kt, qi.kt2); }

template <int HD, int NPOLY>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                         const __grid_constant__ CUtensorMap mV, const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = PairCfg<HD>;
  constexpr int ST = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  PairBars* bars = reinterpret_cast<PairBars*>(smem + C::BAR_OFF);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_full[s], 128);
      mbar_init(&bars->o_full[s], 1);
      mbar_init(&bars->o_free[s], 128);
    }
    for (int i = 0; i < ST; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
    }
    for (int i = 0; i < C::RING; ++i) {
      mbar_init(&bars->item_full[i], 1);
      mbar_init(&bars->item_empty[i], 2 + 8);  // producer, MMA thread, lane 0 of each softmax warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  pdl_trigger();  // after the TMEM allocation
  pdl_wait();     // every role reads the previous kernels' outputs (plan, Q / K / V)
  const int n_items = p.plan.counters[2] * p.H;

  // registers: warpgroup 0 (producer, MMA, 2 idle warps) gives 112 per thread to the softmax warpgroups
  if (warp == 0) {
    // ============================ producer
    setmaxnreg_dec<56>();
    if (elect_one()) {
      int u = 0, nq[2] = {0, 0};
      for (int it = 0;; ++it) {
        const int r = it % C::RING;
        mbar_wait(&bars->item_full[r], (it / C::RING) & 1);
        const PairItem t = bars->item[r];
        mbar_arrive(&bars->item_empty[r]);
        if (t.w < 0) break;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s >= t.nslot) continue;
          if (nq[s] > 0) mbar_wait(&bars->q_empty[s], (nq[s] - 1) & 1);
          ++nq[s];
          mbar_expect_tx(&bars->q_full[s], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d(smem + C::Q_OFF + s * G::TILE_BYTES + blk * G::BLK, &mQ, &bars->q_full[s], blk * G::CB, t.h,
                        t.sa + t.qi[s].qt * 128);
        }
        const int qtA = t.qi[0].qt;
        for (int kt = 0; kt <= qtA; ++kt) {
          const bool a = tile_sees(t.qi[0], kt), b = t.nslot == 2 && tile_sees(t.qi[1], kt);
          if (!a && !b) continue;
          const int stg = u % ST, use = u / ST;
          const int krow = t.sa + kt * 128;
          if (use > 0) mbar_wait(&bars->k_empty[stg], (use - 1) & 1);
          mbar_expect_tx(&bars->k_full[stg], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d(smem + C::K_OFF + stg * G::TILE_BYTES + blk * G::BLK, &mK, &bars->k_full[stg], blk * G::CB,
                        t.h, krow);
          if (use > 0) mbar_wait(&bars->v_empty[stg], (use - 1) & 1);
          mbar_expect_tx(&bars->v_full[stg], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d(smem + C::V_OFF + stg * G::TILE_BYTES + blk * G::BLK, &mV, &bars->v_full[stg], blk * G::CB,
                        t.h, krow);
          ++u;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    setmaxnreg_dec<56>();
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = idesc_bf16(128, G::HDP, 0, 1);
      int u = 0;
      int nq[2] = {0, 0};     // items per slot (q_full parity, o_free parity)
      int npv[2] = {0, 0};    // PVs issued per slot (p_full parity)
      int pend_u[2] = {-1, -1};   // union tile of the slot's S whose PV is not issued yet
      bool pend_first[2] = {false, false};
      int vleft[3] = {0, 0, 0};  // PVs still to issue per V stage
      PP_DECL
      auto issue_pv = [&](int s) {
        const int pu = pend_u[s];
        const int stg = pu % ST;
        PP_MARK(4)
        mbar_wait(&bars->p_full[s], npv[s] & 1);
        PP_MARK(2)
        if (pend_first[s] && nq[s] > 1) mbar_wait(&bars->o_free[s], (nq[s] - 2) & 1);
        mbar_wait(&bars->v_full[stg], (pu / ST) & 1);
        PP_MARK(3)
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + C::V_OFF + stg * G::TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ts(tmem + 256 + s * 128, tmem + s * 128 + kk * 8, mnmajor_desc<HD>(sV, kk), idesc_o,
                      (!pend_first[s] || kk > 0) ? 1u : 0u);
        ++npv[s];
        pend_u[s] = -1;
        int left = 0;
#pragma unroll
        for (int i = 0; i < ST; ++i)
          if (i == stg) left = --vleft[i];
        if (left == 0) mma_commit(&bars->v_empty[stg]);
      };
      for (int it = 0;; ++it) {
        const int r = it % C::RING;
        PP_MARK(4)
        mbar_wait(&bars->item_full[r], (it / C::RING) & 1);
        PP_MARK(0)
        const PairItem t = bars->item[r];
        mbar_arrive(&bars->item_empty[r]);
        if (t.w < 0) break;
        bool first[2] = {true, true};
        int last[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s < t.nslot) ++nq[s];
          last[s] = t.qi[s].qt;  // the diagonal tile is always the slot's last
        }
        const int qtA = t.qi[0].qt;
        for (int kt = 0; kt <= qtA; ++kt) {
          const bool sees[2] = {tile_sees(t.qi[0], kt), t.nslot == 2 && tile_sees(t.qi[1], kt)};
          if (!sees[0] && !sees[1]) continue;
          const int stg = u % ST;
          PP_MARK(4)
          mbar_wait(&bars->k_full[stg], (u / ST) & 1);
          PP_MARK(1)
#pragma unroll
          for (int i = 0; i < ST; ++i)
            if (i == stg) vleft[i] = (int)sees[0] + (int)sees[1];
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (pend_u[s] >= 0) issue_pv(s);
            if (!sees[s]) continue;
            if (first[s]) {
              PP_MARK(4)
              mbar_wait(&bars->q_full[s], (nq[s] - 1) & 1);
              PP_MARK(1)
            }
            tc_fence_after();
            const uint32_t sQ = smem_u32(smem + C::Q_OFF + s * G::TILE_BYTES);
            const uint32_t sK = smem_u32(smem + C::K_OFF + stg * G::TILE_BYTES);
#pragma unroll
            for (int kk = 0; kk < G::HDP / 16; ++kk)
              mma_bf16_ss(tmem + s * 128, kmajor_desc<HD>(sQ, kk), kmajor_desc<HD>(sK, kk), idesc_s, kk > 0 ? 1u : 0u);
            mma_commit(&bars->s_full[s]);
            if (kt == last[s]) mma_commit(&bars->q_empty[s]);
            pend_u[s] = u;
            pend_first[s] = first[s];
            first[s] = false;
          }
          mma_commit(&bars->k_empty[stg]);
          ++u;
        }
        // the item's last PVs, then its O accumulators are complete
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s >= t.nslot) continue;
          if (pend_u[s] >= 0) issue_pv(s);
          mma_commit(&bars->o_full[s]);
        }
      }
      PP_FLUSH(0, 5)
    }
  } else if (warp == 2) {
    // ============================ scheduler: claims items (dynamic counter) and decodes them into the
    // ring up to RING items ahead, so no role waits on the atomic or the plan loads at an item boundary
    setmaxnreg_dec<56>();
    if (elect_one()) {
      for (int it = 0;; ++it) {
        int w = atomicAdd(&p.plan.counters[4], 1);
        if (w >= n_items) w = -1;
        PairItem t;
        pair_item(p, w, t);
        const int r = it % C::RING;
        if (it >= C::RING) mbar_wait(&bars->item_empty[r], ((it / C::RING) - 1) & 1);
        bars->item[r] = t;
        mbar_arrive(&bars->item_full[r]);
        if (w < 0) break;
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<56>();
  } else {
    // ============================ softmax warpgroups
    setmaxnreg_inc<224>();
    const int s = (warp - 4) >> 2;
    const uint32_t quarter = warp & 3;
    const int rt = quarter * 32 + lane;
    const float sl2 = p.scale_log2;
    const uint32_t tS = tmem_addr(tmem, quarter, s * 128);
    const uint32_t tO = tmem_addr(tmem, quarter, 256 + s * 128);
    const uint32_t stg = smem_u32(smem + C::STG_OFF + (warp - 4) * 2048);
    int nt = 0, ni = 0;  // tiles / items of this slot so far
    PP_DECL
    for (int it = 0;; ++it) {
      const int r = it % C::RING;
      mbar_wait(&bars->item_full[r], (it / C::RING) & 1);
      const PairItem& ti = bars->item[r];
      const int w = ti.w, h = ti.h, sa = ti.sa, se = ti.se, nslot = ti.nslot;
      const QTileInfo qi = ti.qi[s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->item_empty[r]);
      if (w < 0) break;
      if (s >= nslot) continue;
      const int q0 = sa + qi.qt * 128;
      const int rows_valid = min(128, se - q0);
      const int row = q0 + rt;
      const bool valid = rt < rows_valid;
      const int e_r = valid ? p.plan.kv_end[row] : 0;
      const bool pp = valid ? (p.plan.row_pp[row] != 0) : false;
      float m_used = -INFINITY, l = 0.f;
      int j = 0;
      for (int kt = next_seen(qi, 0); kt <= qi.qt; kt = next_seen(qi, kt + 1), ++j, ++nt) {
        const int k0 = sa + kt * 128;
        PP_MARK(7)
        mbar_wait(&bars->s_full[s], nt & 1);
        PP_MARK(5)
        tc_fence_after();
        uint32_t sv[128];
        tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
        tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
        tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[64]));
        tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(&sv[96]));
        tmem_ld_wait();
        PP_MARK(8)
        if (!valid || e_r < k0 + 128) {  // PARTIAL row: mask the cells outside its visible set
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t m = valid ? row_mask32(e_r, row, pp, k0 + c * 32) : 0u;
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (!((m >> q) & 1u)) sv[c * 32 + q] = __float_as_uint(-INFINITY);
          }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int q = 0; q < 128; q += 8) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(sv[q]), __uint_as_float(sv[q + 1])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(sv[q + 2]), __uint_as_float(sv[q + 3])));
          mx2 = fmaxf(mx2, fmaxf(__uint_as_float(sv[q + 4]), __uint_as_float(sv[q + 5])));
          mx3 = fmaxf(mx3, fmaxf(__uint_as_float(sv[q + 6]), __uint_as_float(sv[q + 7])));
        }
        const float mx_s = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        PP_MARK(9)
        float factor = 1.f;
        bool rescale = false;
        if (mx_s > m_used + 8.f) {  // conditional rescale (also the first finite max)
          factor = (m_used == -INFINITY) ? 0.f : fast_exp2(m_used - mx_s);
          m_used = mx_s;
          rescale = true;
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2v = make_float2(sl2, sl2), nbase = make_float2(-base, -base);
        float2 rs0 = make_float2(0.f, 0.f), rs1 = make_float2(0.f, 0.f);
        // P packed in place: word q / 2 of sv takes cells q, q + 1 (both already consumed); each 64-cell
        // half is stored as soon as it is packed, so the first STTM overlaps the second half's math
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int q = hh * 64; q < hh * 64 + 64; q += 4) {
            const float2 x01 = __ffma2_rn(make_float2(__uint_as_float(sv[q]), __uint_as_float(sv[q + 1])), sl2v, nbase);
            const float2 x23 =
                __ffma2_rn(make_float2(__uint_as_float(sv[q + 2]), __uint_as_float(sv[q + 3])), sl2v, nbase);
            // NPOLY of every 16 cells on the FMA pipe (MUFU offload), in pairs
            float2 p01, p23;
            if ((q & 15) + 2 > 16 - NPOLY) p01 = exp2_poly3x2(x01);
            else p01 = make_float2(fast_exp2(x01.x), fast_exp2(x01.y));
            if ((q & 15) + 4 > 16 - NPOLY) p23 = exp2_poly3x2(x23);
            else p23 = make_float2(fast_exp2(x23.x), fast_exp2(x23.y));
            rs0 = __fadd2_rn(rs0, p01);
            rs1 = __fadd2_rn(rs1, p23);
            sv[q >> 1] = pack_bf16(p01.x, p01.y);  // F2FP: not on the MUFU pipe (scripts/pipe_bench.cu)
            sv[(q >> 1) + 1] = pack_bf16(p23.x, p23.y);
          }
          tmem_st32(tS + hh * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[hh * 32]));
        }
        PP_MARK(10)
        // O rescale after the S row is dead (registers); s_full(j) was committed after PV(j - 1), so O
        // holds every earlier tile's product, and PV(j) waits for p_full(j) below
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
          const float f = rescale ? factor : 1.f;
#pragma unroll
          for (int c = 0; c < G::HDP / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * f);
            tmem_st32(tO + c * 32, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars->p_full[s]);
        PP_MARK(11)
        l = l * factor + ((rs0.x + rs1.x) + (rs0.y + rs1.y));
      }
      // ---- item end: O / l (bf16 rows through the warp's staging transpose, or fp32), LSE
      PP_MARK(7)
      mbar_wait(&bars->o_full[s], ni & 1);
      PP_MARK(12)
      tc_fence_after();
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      {
        uint32_t o[G::HDP];  // the whole O row in registers, then the accumulator is released at once
#pragma unroll
        for (int c = 0; c < G::HDP / 32; ++c) tmem_ld32(tO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars->o_free[s]);
#pragma unroll
        for (int c = 0; c < G::HDP / 32; ++c) {
          const int ncol = min(32, p.hd - c * 32);
          if (!p.out_f32) {
            uint32_t wv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              wv[q] = pack_bf16(__uint_as_float(o[c * 32 + 2 * q]) * inv_l, __uint_as_float(o[c * 32 + 2 * q + 1]) * inv_l);
            warp_store_rows_bf16(stg, wv,
                                 reinterpret_cast<__nv_bfloat16*>(p.O) + (size_t)(q0 + quarter * 32) * p.d +
                                     (size_t)h * p.hd + c * 32,
                                 p.d, rows_valid - (int)quarter * 32, ncol);
          } else if (valid) {
            float* dst = reinterpret_cast<float*>(p.O) + (size_t)row * p.d + (size_t)h * p.hd + c * 32;
            for (int q = 0; q < ncol; q += 4)
              *reinterpret_cast<float4*>(dst + q) =
                  make_float4(__uint_as_float(o[c * 32 + q]) * inv_l, __uint_as_float(o[c * 32 + q + 1]) * inv_l,
                              __uint_as_float(o[c * 32 + q + 2]) * inv_l, __uint_as_float(o[c * 32 + q + 3]) * inv_l);
          }
        }
      }
      if (valid) p.lse[(size_t)h * p.T + row] = (l > 0.f) ? (m_used + __log2f(l)) * 0.6931471805599453f : 0.f;
      PP_MARK(13)
      ++ni;
    }
    if (threadIdx.x == 128) { PP_FLUSH(5, 16) }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {  // the last CTA out resets the work counters for the next launch on this plan
    __threadfence();
    if (atomicAdd(&p.plan.counters[5], 1) == (int)gridDim.x - 1) {
      p.plan.counters[4] = 0;
      p.plan.counters[5] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- host
bool make_head_map(CUtensorMap* m, const void* ptr, int T, int H, int hd);  // attn_host (below)

bool make_head_map(CUtensorMap* m, const void* ptr, int T, int H, int hd) {
  const int HDP = (hd + 31) / 32 * 32;
  const int RB = (HDP % 64 == 0) ? 128 : 64;
  uint64_t dims[3] = {(uint64_t)hd, (uint64_t)H, (uint64_t)T};
  uint64_t strides[2] = {(uint64_t)hd * 2, (uint64_t)H * hd * 2};
  uint32_t box[3] = {(uint32_t)(RB / 2), 1, 128};
  return encode_bf16_map(m, ptr, 3, dims, strides, box,
                         RB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

#ifndef FWD_NPOLY
#define FWD_NPOLY 5
#endif
// The paired persistent kernel is opt-in (CADET_FWD_PAIRED=1): same-box A/B on C4 measured it slower
// than the one-q-tile-per-CTA kernel (0.321 vs 0.305 ms, round 2).
static bool pair_disabled() {
  const char* e = getenv("CADET_FWD_PAIRED");
  return !(e && e[0] == '1');
}

template <int HD>
static cudaError_t fwd_hd(const CUtensorMap& mQ, const CUtensorMap& mK, const CUtensorMap& mV, const AttnParams& p,
                          cudaStream_t st) {
  using C = FwdCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = p.plan.nq_cap * p.H * p.fwd_splits;
  if (grid == 0) return cudaSuccess;
  if (p.fwd_splits == 1 && !pair_disabled()) {  // persistent paired kernel, one CTA per SM
    using PC = PairCfg<HD>;
    constexpr int NPOLY = FWD_NPOLY;
    static bool pattr = false;
    if (!pattr) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd_pair_kernel<HD, NPOLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           PC::SMEM);
      if (e != cudaSuccess) return e;
      pattr = true;
    }
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // pairs <= (nq_cap + n) / 2 + n; the kernel reads the exact count from the plan
    const int items_cap = ((p.plan.nq_cap + 1) / 2 + p.n) * p.H;
    ProfScope ps(PROF_ATTN_FWD, st, 1);
    cudaError_t e = launch_pdl(attn_fwd_pair_kernel<HD, NPOLY>, dim3(std::min(sms, std::max(items_cap, 1))),
                               dim3(PC::THREADS), PC::SMEM, st, mQ, mK, mV, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  ProfScope ps(PROF_ATTN_FWD, st, p.fwd_splits > 1 ? 2 : 1);
  cudaError_t e = launch_pdl(attn_fwd_kernel<HD>, grid, 192, C::SMEM, st, mQ, mK, mV, p);
  if (e != cudaSuccess) return e;
  if (p.fwd_splits > 1) launch_pdl(attn_fwd_merge_kernel, dim3(p.T), dim3(256), 0, st, p);
  return cudaGetLastError();
}

cudaError_t attn_fwd_launch(const void* Qr, const void* Kr, const void* V, const AttnParams& p, cudaStream_t st) {
  CUtensorMap mQ, mK, mV;
  if (!make_head_map(&mQ, Qr, p.T, p.H, p.hd) || !make_head_map(&mK, Kr, p.T, p.H, p.hd) ||
      !make_head_map(&mV, V, p.T, p.H, p.hd))
    return cudaErrorInvalidValue;
  switch ((p.hd + 31) / 32 * 32) {
    case 32: return fwd_hd<32>(mQ, mK, mV, p, st);
    case 64: return fwd_hd<64>(mQ, mK, mV, p, st);
    case 96: return fwd_hd<96>(mQ, mK, mV, p, st);
    case 128: return fwd_hd<128>(mQ, mK, mV, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cadet

#ifdef CADET_PHASE_TIMING
extern "C" int cadet_debug_phase_read_fwd(unsigned long long* out, int n) {
  cudaMemcpyFromSymbol(out, cadet::g_phase_fwd, sizeof(unsigned long long) * n);
  return n;
}
extern "C" int cadet_debug_phase_reset_fwd() {
  static unsigned long long z[8192 * 16];
  cudaMemcpyToSymbol(cadet::g_phase_fwd, z, sizeof(z));
  return 0;
}
#endif
