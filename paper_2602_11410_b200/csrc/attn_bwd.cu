// A10: attention backward (adjoint of PAPER.md Eq. 7) for the packed, session-masked layout,
// as two atomic-free kernels (deterministic; no fp32 reductions through L2):
//
// attn_bwd_dq_kernel  — one CTA per (q-tile, head), k-tiles visited exactly as in the forward:
//   S_j = Q K_j^T (TMEM, double-buffered), dP_j = dO V_j^T (TMEM);  thread = query row:
//   P = exp2(S log2e/sqrt(hd) - LSE log2e) on visible cells, dS = P (dP - D) / sqrt(hd) written
//   as packed bf16 over the consumed dP columns;  dQ += dS K_j as a TMEM-A (TS) MMA; dQ leaves
//   TMEM once, at the end.
// attn_bwd_dkv_kernel — one CTA per (k-tile, head), walking the q-tiles that see it (transpose of
//   the visit rule, list built once in smem):  S^T = K Q_i^T, dP^T = V dO_i^T;  thread = key row
//   (two warps per TMEM lane quarter, 64 q columns each): P^T, dS^T as packed bf16 over the
//   consumed columns;  dV += P^T dO_i, dK += dS^T Q_i as TS MMAs; Q_i / dO_i double-buffered.
// The extra S/dP recompute (7 MMAs per tile pair instead of 5) buys the removal of 1.1 GB of dQ
// atomics per C4 step and of the drain -> dP dependency.
#include <algorithm>
#include <cstring>

#include "attn_common.cuh"
#include "launch.cuh"
#include "prof.cuh"

namespace cadet {

#ifdef CADET_PHASE_TIMING
// Phase timers (profiling builds only): per CTA, summed clock64 deltas, [blockIdx][8].
__device__ unsigned long long g_phase[8192][16];
// CTA timeline: [blockIdx][kernel 0=dq 1=dkv] {entry, first MMA result, all MMAs done, exit, smid, n}
__device__ unsigned long long g_trace[8192][2][6];
CADET_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
CADET_DEV uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TR(k, slot, v) \
  if (blockIdx.x < 8192) g_trace[blockIdx.x][k][slot] = (v);
#define PT_DECL unsigned long long _pt = clock64();
#define PT_MARK(slot)                                          \
  {                                                            \
    unsigned long long _n = clock64();                         \
    if (blockIdx.x < 8192) atomicAdd(&g_phase[blockIdx.x][slot], _n - _pt); \
    _pt = _n;                                                  \
  }
#else
#define PT_DECL
#define PT_MARK(slot)
#define TR(k, slot, v)
#endif
#ifdef CADET_PHASE_TIMING
// per-thread event timelines of CTA 7 (no atomics: each traced thread owns a row, its counter in a register)
__device__ unsigned long long g_tl[4][4096];
#define TLX(code, idx)                                                                  \
  if (blockIdx.x == 7 && _tln < 4096) {                                                 \
    g_tl[_tlr][_tln++] = (clock64() << 16) | ((unsigned long long)(code) << 10) | ((idx) & 1023); \
  }
#define TL_DECL(row) int _tln = 0; const int _tlr = (row);
#else
#define TLX(code, idx)
#define TL_DECL(row)
#endif
#define PTM(cond, slot) \
  if (cond) { PT_MARK(slot) }

__device__ __forceinline__ int visit_tile_b(const QTileInfo& qi, int j) { return j < qi.nf ? j : qi.kt2 + (j - qi.nf); }
__device__ __forceinline__ bool q_sees_k(const QTileInfo& qi, int kt) {
  return kt < qi.nf || (kt >= qi.kt2 && kt <= qi.qt);
}

// ============================================================================ dQ kernel
// Persistent: CTA c takes work items w = c, c + gridDim.x, ... of the (q-tile in fwd_order, head)
// list (LPT order preserved per stride).  Barrier phases count globally across items; Q/dO are
// released (qd_empty) once the item's last S / dP MMA is issued and the dQ accumulator once the
// compute warps have drained it (dq_free), so the next item's loads and first MMAs overlap the
// current item's tail and dQ store.
template <int HD>
struct DqCfg {
  using G = HeadGeom<HD>;
  static constexpr int Q_OFF = 0;
  static constexpr int DO_OFF = Q_OFF + G::TILE_BYTES;
  static constexpr int K_OFF = DO_OFF + G::TILE_BYTES;        // two stages
  static constexpr int V_OFF = K_OFF + 2 * G::TILE_BYTES;     // two stages
  static constexpr int STG_OFF = V_OFF + 2 * G::TILE_BYTES;   // [8 compute warps][4 KB] store transpose
  static constexpr int BAR_OFF = STG_OFF + 8 * 4096;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int S_COL = 0, DP_COL = 256, DQ_COL = 384;  // S double-buffered
  static constexpr int THREADS = 320;  // producer, MMA, 2 compute warpgroups (64 S/dP columns each)
};

struct DqBars {
  uint64_t qd_full, qd_empty, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], s_free[2], dp_full, ds_ready,
      dq_done, dq_free;
  uint32_t tmem_base;
};

struct DqWork {
  QTileInfo qi;
  int h, sa, se, q0, rows_valid, n_kv;
};
CADET_DEV DqWork dq_work(const AttnParams& p, int w) {
  DqWork t;
  t.h = w % p.H;
  t.qi = p.plan.qinfo[p.plan.fwd_order[w / p.H]];
  t.sa = p.cu[t.qi.seq];
  t.se = p.cu[t.qi.seq + 1];
  t.q0 = t.sa + t.qi.qt * 128;
  t.rows_valid = min(128, t.se - t.q0);
  t.n_kv = t.qi.nf + (t.qi.qt + 1 - t.qi.kt2);
  return t;
}

template <int HD>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                       const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                       const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = DqCfg<HD>;
  if (threadIdx.x == 0) { TR(0, 0, gtime()); TR(0, 4, smid()); }

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  DqBars* bars = reinterpret_cast<DqBars*>(smem + C::BAR_OFF);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bars->qd_full, 1);
    mbar_init(&bars->qd_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], 256);
    }
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->ds_ready, 256);
    mbar_init(&bars->dq_done, 1);
    mbar_init(&bars->dq_free, 256);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first
  pdl_wait();  // everything below reads the previous kernels' outputs
  const int n_work = p.plan.counters[0] * p.H;

  if (warp == 0) {
    if (elect_one()) {
      int gk = 0;  // global k-tile counter: stage gk & 1, use gk >> 1
      for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
        const DqWork t = dq_work(p, w);
        if (wi > 0) mbar_wait(&bars->qd_empty, (wi - 1) & 1);
        mbar_expect_tx(&bars->qd_full, 2 * G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk) {
          tma_load_3d(smem + C::Q_OFF + blk * G::BLK, &mQ, &bars->qd_full, blk * G::CB, t.h, t.q0);
          tma_load_3d(smem + C::DO_OFF + blk * G::BLK, &mdO, &bars->qd_full, blk * G::CB, t.h, t.q0);
        }
        for (int j = 0; j < t.n_kv; ++j, ++gk) {
          const int st = gk & 1, use = gk >> 1;
          const int krow = t.sa + visit_tile_b(t.qi, j) * 128;
          if (use > 0) mbar_wait(&bars->k_empty[st], (use - 1) & 1);
          mbar_expect_tx(&bars->k_full[st], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d(smem + C::K_OFF + st * G::TILE_BYTES + blk * G::BLK, &mK, &bars->k_full[st], blk * G::CB, t.h,
                        krow);
          if (use > 0) mbar_wait(&bars->v_empty[st], (use - 1) & 1);
          mbar_expect_tx(&bars->v_full[st], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d(smem + C::V_OFF + st * G::TILE_BYTES + blk * G::BLK, &mV, &bars->v_full[st], blk * G::CB, t.h,
                        krow);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t id_q = idesc_bf16(128, G::HDP, 0, 1);
      const uint32_t sQ = smem_u32(smem + C::Q_OFF), sdO = smem_u32(smem + C::DO_OFF);
      int gs = 0;  // global k-tile counter (S buffer, K/V stage)
      for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
        const int n_kv = dq_work(p, w).n_kv;
        mbar_wait(&bars->qd_full, wi & 1);
        tc_fence_after();
        auto issue_s = [&](int j) {
          const int g = gs + j, st = g & 1, use = g >> 1;
          if (use > 0) mbar_wait(&bars->s_free[st], (use - 1) & 1);
          mbar_wait(&bars->k_full[st], use & 1);
          tc_fence_after();
          const uint32_t sK = smem_u32(smem + C::K_OFF + st * G::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < G::HDP / 16; ++kk)
            mma_bf16_ss(tmem + C::S_COL + st * 128, kmajor_desc<HD>(sQ, kk), kmajor_desc<HD>(sK, kk), id_s,
                        kk > 0 ? 1u : 0u);
          mma_commit(&bars->s_full[st]);
        };
        if (n_kv > 0) issue_s(0);
        for (int j = 0; j < n_kv; ++j) {
          const int g = gs + j, st = g & 1, use = g >> 1;
          // dP_j over dS_{j-1}: in-order after dQ_{j-1}, which read it
          mbar_wait(&bars->v_full[st], use & 1);
          tc_fence_after();
          const uint32_t sV = smem_u32(smem + C::V_OFF + st * G::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < G::HDP / 16; ++kk)
            mma_bf16_ss(tmem + C::DP_COL, kmajor_desc<HD>(sdO, kk), kmajor_desc<HD>(sV, kk), id_s, kk > 0 ? 1u : 0u);
          mma_commit(&bars->dp_full);
          mma_commit(&bars->v_empty[st]);
          if (j + 1 < n_kv)
            issue_s(j + 1);
          else
            mma_commit(&bars->qd_empty);  // the item's last reads of Q (S) and dO (dP) are issued
          mbar_wait(&bars->ds_ready, g & 1);
          tc_fence_after();
          if (j == 0 && wi > 0) {
            mbar_wait(&bars->dq_free, (wi - 1) & 1);
            tc_fence_after();
          }
          const uint32_t sK = smem_u32(smem + C::K_OFF + st * G::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)
            mma_bf16_ts(tmem + C::DQ_COL, tmem + C::DP_COL + (kk >> 1) * 32 + (kk & 1) * 8, mnmajor_desc<HD>(sK, kk),
                        id_q, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars->k_empty[st]);
        }
        if (n_kv == 0) {
          mma_commit(&bars->qd_empty);
          if (wi > 0) mbar_wait(&bars->dq_free, (wi - 1) & 1);
        }
        mma_commit(&bars->dq_done);
        gs += n_kv;
      }
    }
  } else {
    // thread = query row; warpgroup grp (warps 2..5 -> 0, 6..9 -> 1) owns S/dP columns [64 grp, +64)
    const uint32_t quarter = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int rt = quarter * 32 + lane;
    const float sl2 = p.scale_log2;
    int gs = 0;
    // items decoded one ahead: the row loads below depend on no global-load chain
    DqWork t = dq_work(p, blockIdx.x < n_work ? blockIdx.x : 0);
    DqWork tn = dq_work(p, blockIdx.x + gridDim.x < n_work ? blockIdx.x + gridDim.x : 0);
    for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
      const int r = t.q0 + rt;
      const bool valid = rt < t.rows_valid;
      const int e_r = valid ? p.plan.kv_end[r] : 0;
      const bool pp = valid ? (p.plan.row_pp[r] != 0) : false;
      const float lse2 = valid ? p.lse[(size_t)t.h * p.T + r] * 1.4426950408889634f : 0.f;
      const float Dr = valid ? p.D[(size_t)t.h * p.T + r] : 0.f;
      for (int j = 0; j < t.n_kv; ++j) {
        const int g = gs + j, st = g & 1, use = g >> 1;
        const int k0 = t.sa + visit_tile_b(t.qi, j) * 128;
        const bool partial = !valid || (e_r < k0 + 128);
        mbar_wait(&bars->s_full[st], use & 1);
        mbar_wait(&bars->dp_full, g & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * grp + cc;
          uint32_t us[32], ud[32];
          tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + st * 128 + c * 32), us);
          tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + c * 32), ud);
          tmem_ld_wait();
          uint32_t wv[16];
          const uint32_t m = !partial ? 0xFFFFFFFFu : (valid ? row_mask32(e_r, r, pp, k0 + c * 32) : 0u);
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            float ds[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float xe = fmaf(__uint_as_float(us[q + e]), sl2, -lse2);
              xe = ((m >> (q + e)) & 1u) ? xe : -INFINITY;
              const float pr = fast_exp2(xe);
              ds[e] = pr * (__uint_as_float(ud[q + e]) - Dr);  // 1/sqrt(hd) applied in the dQ epilogue
            }
            wv[q >> 1] = pack_bf16(ds[0], ds[1]);
          }
          // packed dS of keys [32c, 32c + 32) -> dP columns [32c, 32c + 16): this thread's own, loaded chunk
          tmem_st16(tmem_addr(tmem, quarter, C::DP_COL + c * 32), wv);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars->s_free[st]);
        mbar_arrive(&bars->ds_ready);
      }
      mbar_wait(&bars->dq_done, wi & 1);
      tc_fence_after();
      const uint32_t stg = smem_u32(smem + C::STG_OFF + (warp - 2) * 4096);
#pragma unroll 1
      for (int c = grp; c < G::HDP / 32; c += 2) {
        uint32_t u[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::DQ_COL + c * 32), u);
        tmem_ld_wait();
        const float f = t.n_kv > 0 ? p.scale : 0.f;
        const size_t off = (size_t)(t.q0 + quarter * 32) * p.d + (size_t)t.h * p.hd + c * 32;
        if (p.dq_bf16) {
          uint32_t wv[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) wv[jj] = pack_bf16(f * __uint_as_float(u[2 * jj]), f * __uint_as_float(u[2 * jj + 1]));
          warp_store_rows_bf16(stg, wv, reinterpret_cast<__nv_bfloat16*>(p.dQ) + off, p.d, t.rows_valid - (int)quarter * 32,
                               min(32, p.hd - c * 32));
        } else {
          warp_store_rows_f32(stg, u, f, reinterpret_cast<float*>(p.dQ) + off, p.d, t.rows_valid - (int)quarter * 32,
                              min(32, p.hd - c * 32));
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
      gs += t.n_kv;
      t = tn;
      if (w + 2 * gridDim.x < n_work) tn = dq_work(p, w + 2 * gridDim.x);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) { TR(0, 3, gtime()); }
}

// ============================================================================ dK / dV kernel
// Persistent like the dQ kernel, over (k-tile in bwd_order, head) items; each item walks the
// q-tiles of its plan visit list (bwd_list).  Each visited q-tile is processed as two 64-column
// halves: the MMA warp issues S^T_h = K Q_h^T and dP^T_h = V dO_h^T into TMEM half-buffer
// (h & 1) BEFORE waiting for half h-1's P^T/dS^T, so the tensor core works while a compute
// warpgroup (one per half-buffer, thread = key row, 64 q columns) turns the previous half into
// P^T / dS^T.  K/V are released (kv_empty) after the item's last S^T/dP^T, the dK/dV
// accumulators after the compute warps drained them (acc_free).
// One 32-column chunk of P^T / dS^T for key row `key` (thread): straight-line, with the
// per-column vectors (LSE*log2e, D, visible-prefix end) read from shared memory at vaddr,
// vaddr + 256 and vaddr + 512.  MASKED: column i is visible iff key < e_i or bit i of extra.
// dS^T is left unscaled (the dK epilogue applies 1/sqrt(hd)).
#ifndef BWD_NPOLY
#define BWD_NPOLY 0
#endif
// Visible-prefix bits of a 32-column chunk for key row `key`: column i is visible iff key < e_i (the
// column's prefix end, staged at vaddr + 1024); the caller ORs in the diagonal / transposed-pair bits and
// masks columns past the sequence end.
CADET_DEV uint32_t dkv_prefix_mask(uint32_t vaddr, int key) {
  uint32_t vis = 0;
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const int4 e4 = lds_i4(vaddr + 1024 + i * 4);
    vis |= (key < e4.x ? 1u : 0u) << i;
    vis |= (key < e4.y ? 1u : 0u) << (i + 1);
    vis |= (key < e4.z ? 1u : 0u) << (i + 2);
    vis |= (key < e4.w ? 1u : 0u) << (i + 3);
  }
  return vis;
}
// Softmax phase of one 32-column chunk: P = exp2(S^T log2e / sqrt(hd) - LSE log2e) (-LSE log2e at vaddr), packed
// bf16 into wp; MASKED: invisible columns (vis bit clear) give exactly 0.
template <bool MASKED>
CADET_DEV void dkv_p_chunk(const uint32_t (&us)[32], uint32_t vaddr, uint32_t vis, float sl2, uint32_t (&wp)[16]) {
  const float2 sl2v = make_float2(sl2, sl2);
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const float4 l4 = lds_f4(vaddr + i * 4);  // -LSE log2e, premultiplied by the vector loader
    const float2 nl01 = make_float2(l4.x, l4.y), nl23 = make_float2(l4.z, l4.w);
    float2 x01 = __ffma2_rn(make_float2(__uint_as_float(us[i]), __uint_as_float(us[i + 1])), sl2v, nl01);
    float2 x23 = __ffma2_rn(make_float2(__uint_as_float(us[i + 2]), __uint_as_float(us[i + 3])), sl2v, nl23);
    if (MASKED) {
      if (!((vis >> i) & 1u)) x01.x = -INFINITY;
      if (!((vis >> (i + 1)) & 1u)) x01.y = -INFINITY;
      if (!((vis >> (i + 2)) & 1u)) x23.x = -INFINITY;
      if (!((vis >> (i + 3)) & 1u)) x23.y = -INFINITY;
    }
    const float2 p01 = ((i & 15) + 2 > 16 - BWD_NPOLY) ? exp2_poly3x2(x01) : make_float2(fast_exp2(x01.x), fast_exp2(x01.y));
    const float2 p23 = ((i & 15) + 4 > 16 - BWD_NPOLY) ? exp2_poly3x2(x23) : make_float2(fast_exp2(x23.x), fast_exp2(x23.y));
    wp[i >> 1] = pack_bf16(p01.x, p01.y);
    wp[(i >> 1) + 1] = pack_bf16(p23.x, p23.y);
  }
}
// dS phase of one chunk from the packed bf16 P^T (the values the dV MMA used): dS^T = P^T (dP^T - D)
CADET_DEV void dkv_ds_chunk_pk(const uint32_t (&ud)[32], const uint32_t* pk, uint32_t vaddr, uint32_t (&wd)[16]) {
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const float4 d4 = lds_f4(vaddr + 512 + i * 4);
    const float2 dd01 = __fadd2_rn(make_float2(__uint_as_float(ud[i]), __uint_as_float(ud[i + 1])), make_float2(-d4.x, -d4.y));
    const float2 dd23 =
        __fadd2_rn(make_float2(__uint_as_float(ud[i + 2]), __uint_as_float(ud[i + 3])), make_float2(-d4.z, -d4.w));
    const uint32_t w0 = pk[i >> 1], w1 = pk[(i >> 1) + 1];
    const float2 p01 = make_float2(__uint_as_float(w0 << 16), __uint_as_float(w0 & 0xFFFF0000u));
    const float2 p23 = make_float2(__uint_as_float(w1 << 16), __uint_as_float(w1 & 0xFFFF0000u));
    const float2 s01 = __fmul2_rn(p01, dd01), s23 = __fmul2_rn(p23, dd23);
    wd[i >> 1] = pack_bf16(s01.x, s01.y);
    wd[(i >> 1) + 1] = pack_bf16(s23.x, s23.y);
  }
}

template <int HD>
struct DkvCfg {
  using G = HeadGeom<HD>;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + G::TILE_BYTES;
  static constexpr int Q_OFF = V_OFF + G::TILE_BYTES;          // two stages
  static constexpr int DO_OFF = Q_OFF + 2 * G::TILE_BYTES;     // two stages
  // VSTAGES stages of one q-tile's column vectors, written by the vector-loader warp: -LSE log2e [128] f32 at +0,
  // D [128] f32 at +512, kv_end [128] i32 at +1024, the visit-list entry at +1536
  static constexpr int VSTAGES = 4;
  static constexpr int VEC_OFF = DO_OFF + 2 * G::TILE_BYTES;
  static constexpr int VEC_BYTES = 2048;
  static constexpr int STG_OFF = VEC_OFF + VSTAGES * VEC_BYTES;  // [8 compute warps][2 KB] store transpose
  // dS^T chunks by TMA bulk tensor stores from the stage (hd 128: -4..-7 % on C4) or by the warp's own
  // LDS + STG (hd <= 96: the TMA variant measured +5 % on C3's attention backward)
  static constexpr bool TMA_DS = HD == 128;
  static constexpr bool TMA_DRAIN = HD == 128;  // dK / dV drain likewise (hd 96: +6 % on C3 with it)
  static constexpr int BAR_OFF = STG_OFF + 8 * 2048;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  // S^T/P^T half-buffers at [0,64) and [64,128); dP^T/dS^T at [128,192) and [192,256)
  static constexpr int S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 384;
  static constexpr int THREADS = 352;  // producer, MMA, 2 compute warpgroups (one per half-buffer), vector loader
};

struct DkvBars {
  uint64_t kv_full, kv_empty, q_full[2], q_empty[2], do_full[2], do_empty[2], s_full, dp_full, p_ready[2], ds_ready[2],
      mma_done, acc_free, vec_full[4], vec_empty[4];
  uint32_t tmem_base;
};

struct DkvWork {
  int h, seq, kt, sa, se, k0, keys_valid, off, n_it;
};
CADET_DEV DkvWork dkv_work(const AttnParams& p, int w) {
  DkvWork t;
  t.h = w % p.H;
  const int g = p.plan.bwd_order[w / p.H];
  const QTileInfo ki = p.plan.qinfo[g];
  t.seq = ki.seq;
  t.kt = ki.qt;
  t.sa = p.cu[ki.seq];
  t.se = p.cu[ki.seq + 1];
  t.k0 = t.sa + t.kt * 128;
  t.keys_valid = min(128, t.se - t.k0);
  t.off = p.plan.bwd_off[g];
  t.n_it = p.plan.bwd_cnt[g];
  return t;
}

template <int HD>
__global__ void __launch_bounds__(352, 1)
    attn_bwd_dkv_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                        const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                        const __grid_constant__ CUtensorMap mDSs, const __grid_constant__ CUtensorMap mDK,
                        const __grid_constant__ CUtensorMap mDV, const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = DkvCfg<HD>;
  if (threadIdx.x == 0) { TR(1, 0, gtime()); TR(1, 4, smid()); }

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  DkvBars* bars = reinterpret_cast<DkvBars*>(smem + C::BAR_OFF);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
      mbar_init(&bars->do_full[i], 1);
      mbar_init(&bars->do_empty[i], 1);
      mbar_init(&bars->p_ready[i], 128);
      mbar_init(&bars->ds_ready[i], 128);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->mma_done, 1);
    mbar_init(&bars->acc_free, 256);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bars->vec_full[i], 32);
      mbar_init(&bars->vec_empty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first
  pdl_wait();  // everything below reads the previous kernels' outputs
  const int n_work = p.plan.counters[0] * p.H;
  const int32_t* list = p.plan.bwd_list;

  if (warp == 0) {
    if (elect_one()) {
      int gq = 0;  // global q-tile counter: stage gq & 1, use gq >> 1
      // Q_i / dO_i are re-read by every k-tile that sees q-tile i: keep them in L2 (evict_last)
      const uint64_t pol_qd = l2_policy_evict_last();
      for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
        const DkvWork t = dkv_work(p, w);
        if (wi > 0) mbar_wait(&bars->kv_empty, (wi - 1) & 1);
        mbar_expect_tx(&bars->kv_full, 2 * G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk) {
          tma_load_3d(smem + C::K_OFF + blk * G::BLK, &mK, &bars->kv_full, blk * G::CB, t.h, t.k0);
          tma_load_3d(smem + C::V_OFF + blk * G::BLK, &mV, &bars->kv_full, blk * G::CB, t.h, t.k0);
        }
        for (int it = 0; it < t.n_it; ++it, ++gq) {  // list entry: qt | full << 30
          const int st = gq & 1, use = gq >> 1;
          const int q0 = t.sa + (list[t.off + it] & 0xFFFF) * 128;
          if (use > 0) mbar_wait(&bars->q_empty[st], (use - 1) & 1);
          mbar_expect_tx(&bars->q_full[st], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d_hint(smem + C::Q_OFF + st * G::TILE_BYTES + blk * G::BLK, &mQ, &bars->q_full[st], blk * G::CB,
                             t.h, q0, pol_qd);
          if (use > 0) mbar_wait(&bars->do_empty[st], (use - 1) & 1);
          mbar_expect_tx(&bars->do_full[st], G::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d_hint(smem + C::DO_OFF + st * G::TILE_BYTES + blk * G::BLK, &mdO, &bars->do_full[st],
                             blk * G::CB, t.h, q0, pol_qd);
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer.  Per q-tile g (full 128-column S^T / dP^T, N = 128 MMAs at
    // their floor): S^T(g) -> [softmax phase] -> dV(g), then S^T(g + 1) over the consumed P^T(g);
    // dP^T(g) -> [dS phase] -> dK(g), then dP^T(g + 1) over the consumed dS^T(g).  The tensor core runs
    // dP^T(g) during the softmax phase and dV(g) + S^T(g + 1) during the dS phase.
    if (elect_one()) {
      const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t id_kv = idesc_bf16(128, G::HDP, 0, 1);
      const uint32_t sK = smem_u32(smem + C::K_OFF), sV = smem_u32(smem + C::V_OFF);
      int gq = 0;  // global q-tile counter
      PT_DECL
      TL_DECL(0)
      auto issue_s = [&](int g) {  // S^T = K Q_g^T into S_COL
        const int st = g & 1;
        const uint32_t sQ = smem_u32(smem + C::Q_OFF + st * G::TILE_BYTES);
        mbar_wait(&bars->q_full[st], (g >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::S_COL, kmajor_desc<HD>(sK, kk), kmajor_desc<HD>(sQ, kk), id_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->s_full);
      };
      auto issue_dp = [&](int g) {  // dP^T = V dO_g^T into DP_COL
        const int st = g & 1;
        const uint32_t sdO = smem_u32(smem + C::DO_OFF + st * G::TILE_BYTES);
        mbar_wait(&bars->do_full[st], (g >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::DP_COL, kmajor_desc<HD>(sV, kk), kmajor_desc<HD>(sdO, kk), id_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->dp_full);
      };
      for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
        const int n_it = dkv_work(p, w).n_it;
        PT_MARK(3)
        mbar_wait(&bars->kv_full, wi & 1);
        tc_fence_after();
        PT_MARK(0)
        if (n_it == 0) {
          mma_commit(&bars->kv_empty);
          if (wi > 0) mbar_wait(&bars->acc_free, (wi - 1) & 1);
          mma_commit(&bars->mma_done);
          continue;
        }
        issue_s(gq);
        issue_dp(gq);
        if (n_it == 1) mma_commit(&bars->kv_empty);  // the item's last reads of K / V are issued
        for (int it = 0; it < n_it; ++it) {
          const int g = gq + it, st = g & 1;
          const uint32_t sQ = smem_u32(smem + C::Q_OFF + st * G::TILE_BYTES);
          const uint32_t sdO = smem_u32(smem + C::DO_OFF + st * G::TILE_BYTES);
          PT_MARK(3)
          mbar_wait(&bars->p_ready[0], g & 1);
          mbar_wait(&bars->p_ready[1], g & 1);
          tc_fence_after();
          TLX(3, 2 * it)
          PT_MARK(2)
          if (it == 0 && wi > 0) {
            mbar_wait(&bars->acc_free, (wi - 1) & 1);
            tc_fence_after();
          }
          PT_MARK(1)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int kk = 0; kk < 64 / 16; ++kk)
              mma_bf16_ts(tmem + C::DV_COL, tmem + C::S_COL + hf * 64 + kk * 8, mnmajor_desc<HD>(sdO, hf * 4 + kk),
                          id_kv, (it > 0 || hf > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars->do_empty[st]);  // dO(g): dP^T(g) and dV(g) issued
          if (it + 1 < n_it) issue_s(g + 1);  // over P^T(g): after dV(g) in issue order
          TLX(4, 2 * it)
          PT_MARK(3)
          mbar_wait(&bars->ds_ready[0], g & 1);
          mbar_wait(&bars->ds_ready[1], g & 1);
          tc_fence_after();
          TLX(3, 2 * it + 1)
          PT_MARK(2)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int kk = 0; kk < 64 / 16; ++kk)
              mma_bf16_ts(tmem + C::DK_COL, tmem + C::DP_COL + hf * 64 + kk * 8, mnmajor_desc<HD>(sQ, hf * 4 + kk),
                          id_kv, (it > 0 || hf > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars->q_empty[st]);  // Q(g): S^T(g) and dK(g) issued
          if (it + 1 < n_it) {
            issue_dp(g + 1);  // over dS^T(g): after dK(g) in issue order
            if (it + 1 == n_it - 1) mma_commit(&bars->kv_empty);
          }
          TLX(4, 2 * it + 1)
        }
        mma_commit(&bars->mma_done);
        gq += n_it;
      }
    }
  } else if (warp == 10) {
    // ============================ vector loader: per visited q-tile, LSE, D and kv_end of its 128 columns
    // (coalesced, +inf / 0 / -1 past the sequence end) and the visit-list entry, VSTAGES q-tiles ahead
    int g = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const DkvWork t = dkv_work(p, w);
      for (int it = 0; it < t.n_it; ++it, ++g) {
        const int vs = g % C::VSTAGES, use = g / C::VSTAGES;
        const int entry = list[t.off + it];
        const int q0 = t.sa + (entry & 0xFFFF) * 128;
        float lv[4], dv[4];
        int ev[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = q0 + j * 32 + lane;
          const bool v = q < t.se;
          lv[j] = v ? -1.4426950408889634f * p.lse[(size_t)t.h * p.T + q] : -INFINITY;  // -LSE log2e
          dv[j] = v ? p.D[(size_t)t.h * p.T + q] : 0.f;
          ev[j] = v ? p.plan.kv_end[q] : -1;
        }
        if (use > 0) mbar_wait(&bars->vec_empty[vs], (use - 1) & 1);
        float* vb = reinterpret_cast<float*>(smem + C::VEC_OFF + vs * C::VEC_BYTES);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          vb[j * 32 + lane] = lv[j];
          vb[128 + j * 32 + lane] = dv[j];
          reinterpret_cast<int*>(vb)[256 + j * 32 + lane] = ev[j];
        }
        if (lane == 0) reinterpret_cast<int*>(vb)[384] = entry;
        mbar_arrive(&bars->vec_full[vs]);
      }
    }
  } else {
    // warpgroup grp (warps 2..5 -> 0, 6..9 -> 1) owns TMEM half-buffer grp = q columns [64 grp, +64)
    const uint32_t quarter = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int tr = quarter * 32 + lane;
    const int gt = (threadIdx.x - 64) & 127;  // 0..127 inside the warpgroup
    const float sl2 = p.scale_log2;
    const bool tracer = gt == 0;
    // items are decoded one ahead, so no dependent global-load chain sits at an item boundary
    DkvWork t = dkv_work(p, blockIdx.x < n_work ? blockIdx.x : 0);
    DkvWork tn = dkv_work(p, blockIdx.x + gridDim.x < n_work ? blockIdx.x + gridDim.x : 0);
    int gq = 0;
    PT_DECL
    TL_DECL(1 + grp)
    for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
      const bool has_next = w + gridDim.x < n_work;
      const int key = t.k0 + tr;
      const bool key_valid = tr < t.keys_valid;
      // two-pass backward: dS^T tiles of this k-tile go to slots tri_off[seq] + qt (qt + 1) / 2 + kt
      const int ds_base = p.dS ? p.plan.tri_off[t.seq] + t.kt : 0;
      // query row key+1 carries the PAIR_PREV bit: then it sees this key (the transposed pair cell)
      const bool ppn = key_valid && key + 1 < t.se && p.plan.row_pp[key + 1] != 0;
      for (int it = 0; it < t.n_it; ++it) {
        const int g = gq + it, vs = g % C::VSTAGES;
        const uint32_t vst = smem_u32(smem + C::VEC_OFF + vs * C::VEC_BYTES);
        PTM(tracer, 7)
        mbar_wait(&bars->vec_full[vs], (g / C::VSTAGES) & 1);  // this q-tile's column vectors
        mbar_wait(&bars->s_full, g & 1);
        tc_fence_after();
        if (tracer) { TLX(10 + grp, g) }
        PTM(tracer, 6)
        const int entry = *reinterpret_cast<const int*>(smem + C::VEC_OFF + vs * C::VEC_BYTES + 1536);
        const bool full = (entry >> 30) & 1;
        const int qbase = t.sa + (entry & 0xFFFF) * 128 + grp * 64;
        // ---- softmax phase: P^T of this warpgroup's 64 columns (kept in fp32 for the dS phase)
        // P^T kept packed (bf16, the values the dV MMA multiplies) for the dS phase; both chunks' TMEM
        // loads in flight before one wait in each phase (TMEM load latency is long while the tensor
        // core is busy)
        uint32_t pk[32];
        {
          PTM(tracer, 8)
          uint32_t us0[32], us1[32];
          tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + grp * 64), us0);
          tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + grp * 64 + 32), us1);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t va = vst + (grp * 64 + c * 32) * 4;
            uint32_t wp[16];
            if (full) {
              dkv_p_chunk<false>(c == 0 ? us0 : us1, va, 0u, sl2, wp);
            } else {
              const int q0c = qbase + c * 32;
              const int dd = key - q0c;
              uint32_t extra = 0;
              if (key_valid && dd >= 0 && dd < 32) extra |= 1u << dd;
              if (ppn && dd + 1 >= 0 && dd + 1 < 32) extra |= 1u << (dd + 1);
              const int nv = t.se - q0c;
              const uint32_t colmask = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
              const uint32_t vis = (dkv_prefix_mask(va, key) | extra) & colmask & (key_valid ? 0xFFFFFFFFu : 0u);
              dkv_p_chunk<true>(c == 0 ? us0 : us1, va, vis, sl2, wp);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[c * 16 + j] = wp[j];
            tmem_st16(tmem_addr(tmem, quarter, C::S_COL + grp * 64 + c * 16), wp);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bars->p_ready[grp]);
          PTM(tracer, 9)
        }
        uint32_t wkeep[16];
        mbar_wait(&bars->dp_full, g & 1);
        tc_fence_after();
        {
          uint32_t ud0[32], ud1[32];
          tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + grp * 64), ud0);
          tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + grp * 64 + 32), ud1);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t va = vst + (grp * 64 + c * 32) * 4;
            uint32_t wd[16];
            dkv_ds_chunk_pk(c == 0 ? ud0 : ud1, &pk[c * 16], va, wd);
            if (p.dS) {  // chunk 0 -> the warp's stage now (after the previous TMA store read it), chunk 1 kept
              if (c == 0) {
                if (C::TMA_DS || C::TMA_DRAIN) {
                  if (lane == 0) bulk_wait_read0();
                  __syncwarp();
                }
                warp_stage_rows_bf16(smem_u32(smem + C::STG_OFF + (warp - 2) * 2048), wd);
              }
              else
#pragma unroll
                for (int j = 0; j < 16; ++j) wkeep[j] = wd[j];
            }
            tmem_st16(tmem_addr(tmem, quarter, C::DP_COL + grp * 64 + c * 16), wd);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bars->ds_ready[grp]);
        }
        if (tracer) { TLX(12 + grp, g) }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->vec_empty[vs]);  // the warp's vector reads are done
        PTM(tracer, 10)
        if (p.dS) {  // two-pass backward: this warp's 32 keys x 64 q columns of dS^T, off the MMA's path
          const int qt = entry & 0xFFFF;
          const int slot = ds_base + qt * (qt + 1) / 2;
          if (slot < p.ds_slots) {  // (a batch violating max_seqlen latches E_TOO_LONG; stay in bounds)
            // the warp's 32 keys x 32 q chunks leave through TMA bulk tensor stores straight from the
            // (64B-swizzled) stage: no LDS / STG by the warp, which moves on to the next q-tile
            const uint32_t stg = smem_u32(smem + C::STG_OFF + (warp - 2) * 2048);
            if (C::TMA_DS) {
              const int row = slot * 128 + quarter * 32;
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&mDSs, stg, grp * 64, t.h, row);
                bulk_commit();
                bulk_wait_read0();
              }
              __syncwarp();
              warp_stage_rows_bf16(stg, wkeep);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&mDSs, stg, grp * 64 + 32, t.h, row);
                bulk_commit();
              }
            } else {
              __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.dS) +
                                   (((size_t)slot * 128 + quarter * 32) * p.H + t.h) * 128 + grp * 64;
              // streaming (evict-first) stores: the dS^T tiles are read once, by the next kernel
              warp_flush_rows_bf16<true>(stg, dst, (size_t)p.H * 128, 32, 32);
              warp_stage_rows_bf16(stg, wkeep);
              warp_flush_rows_bf16<true>(stg, dst + 32, (size_t)p.H * 128, 32, 32);
            }
          } else {
            __syncwarp();
          }
        }
        if (tracer) { TLX(14 + grp, g) }
      }
      // dK, dV (thread = key row; each warpgroup writes half of the hd columns)
      if (lane == 0) bulk_wait_read0();  // the stage is free of the last dS^T store
      __syncwarp();
      PTM(tracer, 7)
      mbar_wait(&bars->mma_done, wi & 1);
      tc_fence_after();
      PTM(tracer, 4)
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        void* out = which == 0 ? p.dK : p.dV;
        const int col0 = which == 0 ? C::DK_COL : C::DV_COL;
        const float f = t.n_it == 0 ? 0.f : (which == 0 ? p.scale : 1.f);  // dS^T was accumulated without 1/sqrt(hd)
#pragma unroll 1
        for (int c = grp; c < G::HDP / 32; c += 2) {
          uint32_t u[32];
          tmem_ld32(tmem_addr(tmem, quarter, col0 + c * 32), u);
          tmem_ld_wait();
          if (which == 1 && c + 2 >= G::HDP / 32) {  // this warp's last accumulator read: hand the
            tc_fence_before();                        // accumulators to the next item's MMAs before
            mbar_arrive(&bars->acc_free);             // the last stores
          }
          const int ncol = min(32, p.hd - c * 32);
          if (!p.out_f32) {
            uint32_t wv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) wv[j] = pack_bf16(f * __uint_as_float(u[2 * j]), f * __uint_as_float(u[2 * j + 1]));
            const uint32_t stg = smem_u32(smem + C::STG_OFF + (warp - 2) * 2048);
            if (C::TMA_DRAIN && t.keys_valid == 128 && p.dS) {  // full k-tile: TMA bulk store from the stage
              if (lane == 0) bulk_wait_read0();
              __syncwarp();
              warp_stage_rows_bf16(stg, wv);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(which == 0 ? &mDK : &mDV, stg, c * 32, t.h, t.k0 + quarter * 32);
                bulk_commit();
              }
            } else {
              if (C::TMA_DS || C::TMA_DRAIN) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              warp_store_rows_bf16(stg, wv,
                                   reinterpret_cast<__nv_bfloat16*>(out) + (size_t)(t.k0 + quarter * 32) * p.d +
                                       (size_t)t.h * p.hd + c * 32,
                                   p.d, t.keys_valid - (int)quarter * 32, ncol);
            }
          } else if (key_valid) {  // fp32 outputs (exactness mode): direct row stores
            float* o = reinterpret_cast<float*>(out) + (size_t)key * p.d + (size_t)t.h * p.hd + c * 32;
            for (int j = 0; j < ncol; j += 4)
              *reinterpret_cast<float4*>(o + j) = make_float4(f * __uint_as_float(u[j]), f * __uint_as_float(u[j + 1]),
                                                              f * __uint_as_float(u[j + 2]), f * __uint_as_float(u[j + 3]));
          }
        }
      }
      if (grp >= G::HDP / 32) {  // (hd = 32: the second warpgroup holds no accumulator chunk)
        tc_fence_before();
        mbar_arrive(&bars->acc_free);
      }
      PTM(tracer, 5)
      gq += t.n_it;
      t = tn;
      const int w2 = w + 2 * gridDim.x;
      if (w2 < n_work) tn = dkv_work(p, w2);
    }
  }
  if (warp >= 2 && warp < 10 && lane == 0) bulk_wait0();  // this warp's dS^T stores complete
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) { TR(1, 3, gtime()); }
}

// ============================================================================ dQ from stored dS
// Two-pass backward (p.dS set): attn_bwd_dkv_kernel has stored every visited dS^T tile, so
// dQ_i = sum_j dS_ij K_j needs no recompute of S and dP (7 -> 5 MMAs per tile pair; the dS
// round trip is 32 KB of HBM per tile pair each way).  Persistent CTA over the (q-tile, head)
// list: warp 0 streams (dS^T_j, K_j) through STAGES TMA stages, warp 1 issues one SS MMA chain per
// tile (A = dS^T as an MN-major operand, B = K_j MN-major) into a double-buffered TMEM
// accumulator, warps 2..5 drain dQ (x 1/sqrt(hd)) while the next item accumulates.
template <int HD>
struct Dq2Cfg {
  using G = HeadGeom<HD>;
  static constexpr int THREADS = 192;
  static constexpr int STAGES = 3;
  static constexpr int DS_BYTES = 2 * 16384;  // [128 keys][128 q] bf16: 2 blocks of 64 columns
  static constexpr int STAGE_BYTES = DS_BYTES + G::TILE_BYTES;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = STG_OFF + 4 * 4096;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};
struct Dq2Bars {
  uint64_t full[4], empty[4], acc_full[2], acc_free[2];
  uint32_t tmem_base;
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_bwd_dq2_kernel(const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mDS,
                        const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = Dq2Cfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Dq2Bars* bars = reinterpret_cast<Dq2Bars*>(smem + C::BAR_OFF);
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->acc_full[b], 1);
      mbar_init(&bars->acc_free[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  pdl_trigger();  // after the TMEM allocation: a dependent CTA never takes this CTA's columns first
  pdl_wait();  // everything below reads the previous kernels' outputs
  const int n_work = p.plan.counters[0] * p.H;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_ds = l2_policy_evict_first(), pol_k = l2_policy_evict_last();
      int g = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const DqWork t = dq_work(p, w);
        const int base = p.plan.tri_off[t.qi.seq] + t.qi.qt * (t.qi.qt + 1) / 2;
        for (int j = 0; j < t.n_kv; ++j, ++g) {
          const int st = g % C::STAGES, use = g / C::STAGES;
          const int kt = visit_tile_b(t.qi, j);
          if (use > 0) mbar_wait(&bars->empty[st], (use - 1) & 1);
          mbar_expect_tx(&bars->full[st], C::STAGE_BYTES);
          uint8_t* sbuf = smem + st * C::STAGE_BYTES;
#pragma unroll
          for (int blk = 0; blk < 2; ++blk)
            tma_load_3d_hint(sbuf + blk * 16384, &mDS, &bars->full[st], blk * 64, t.h, (base + kt) * 128, pol_ds);
#pragma unroll
          for (int blk = 0; blk < G::NB; ++blk)
            tma_load_3d_hint(sbuf + C::DS_BYTES + blk * G::BLK, &mK, &bars->full[st], blk * G::CB, t.h,
                             t.sa + kt * 128, pol_k);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t id = idesc_bf16(128, G::HDP, 1, 1);
      int g = 0;
      for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
        const int n_kv = dq_work(p, w).n_kv;
        const int buf = wi & 1, ause = wi >> 1;
        if (ause > 0) mbar_wait(&bars->acc_free[buf], (ause - 1) & 1);
        tc_fence_after();
        for (int j = 0; j < n_kv; ++j, ++g) {
          const int st = g % C::STAGES, use = g / C::STAGES;
          mbar_wait(&bars->full[st], use & 1);
          tc_fence_after();
          const uint32_t sD = smem_u32(smem + st * C::STAGE_BYTES), sK = sD + C::DS_BYTES;
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)
            mma_bf16_ss(tmem + buf * 128, p_mnmajor_desc(sD, kk), mnmajor_desc<HD>(sK, kk), id,
                        (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars->empty[st]);
        }
        mma_commit(&bars->acc_full[buf]);
      }
    }
  } else {
    const uint32_t quarter = warp & 3;
    const uint32_t stg = smem_u32(smem + C::STG_OFF + (warp - 2) * 4096);
    for (int w = blockIdx.x, wi = 0; w < n_work; w += gridDim.x, ++wi) {
      const DqWork t = dq_work(p, w);
      const int buf = wi & 1;
      mbar_wait(&bars->acc_full[buf], (wi >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < G::HDP / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tmem_addr(tmem, quarter, buf * 128 + c * 32), u);
        tmem_ld_wait();
        if (t.n_kv == 0) {  // no MMA ran: the accumulator holds stale data
#pragma unroll
          for (int j = 0; j < 32; ++j) u[j] = 0u;
        }
        const float f = p.scale;
        const size_t off = (size_t)(t.q0 + quarter * 32) * p.d + (size_t)t.h * p.hd + c * 32;
        if (p.dq_bf16) {
          uint32_t wv[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            wv[jj] = pack_bf16(f * __uint_as_float(u[2 * jj]), f * __uint_as_float(u[2 * jj + 1]));
          warp_store_rows_bf16(stg, wv, reinterpret_cast<__nv_bfloat16*>(p.dQ) + off, p.d,
                               t.rows_valid - (int)quarter * 32, min(32, p.hd - c * 32));
        } else {
          warp_store_rows_f32(stg, u, f, reinterpret_cast<float*>(p.dQ) + off, p.d, t.rows_valid - (int)quarter * 32,
                              min(32, p.hd - c * 32));
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->acc_free[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

// D_i = rowsum(dO_i * O_i) per head (FlashAttention preprocess), bf16 inputs, fp32 out [H, T].
// One warp per row, 16-byte loads (8 columns per lane per 256-column pass); per-head sums by
// segmented shuffles when hd / 8 lanes is a power of two dividing the pass, else shared atomics.
__global__ void __launch_bounds__(256) attn_bwd_pre_kernel(const __nv_bfloat16* O, const __nv_bfloat16* dO, float* D,
                                                            int T, int H, int hd) {
  pdl_trigger();
  pdl_wait();
  __shared__ float acc[8][128];
  __shared__ float part[8][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + w;
  const int d = H * hd, lpg = hd / 8;  // lanes per head
  const bool seg = (lpg & (lpg - 1)) == 0 && lpg <= 32;
  for (int h = lane; h < H; h += 32) acc[w][h] = 0.f;
  __syncwarp();
  if (row < T) {  // warp-uniform: every lane runs every pass (shuffles), lanes past d contribute 0
    for (int c0 = 0; c0 < d; c0 += 256) {
      const int c = c0 + lane * 8;
      const bool valid = c < d;
      float p = 0.f;
      if (valid) {
        const uint4 o = *reinterpret_cast<const uint4*>(O + (size_t)row * d + c);
        const uint4 g = *reinterpret_cast<const uint4*>(dO + (size_t)row * d + c);
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = __bfloat1622float2(o2[e]), b = __bfloat1622float2(g2[e]);
          p = fmaf(a.x, b.x, fmaf(a.y, b.y, p));
        }
      }
      if (seg) {
        for (int off = lpg >> 1; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        if (valid && (lane & (lpg - 1)) == 0) acc[w][c / hd] += p;  // one lane per head segment
      } else {  // head segments not aligned to lane groups (hd = 88): the lanes' partials summed in lane
                // order by the first lane of each head (fixed order: deterministic)
        __syncwarp();
        part[w][lane] = valid ? p : 0.f;
        __syncwarp();
        const int h0 = c0 / hd, h1 = min((c0 + 255) / hd, H - 1);
        for (int h = h0 + lane; h <= h1; h += 32) {
          float sum = 0.f;
          for (int l = 0; l < 32; ++l) {
            const int cl = c0 + l * 8;
            if (cl < d && cl / hd == h) sum += part[w][l];
          }
          acc[w][h] += sum;
        }
      }
    }
  }
  __syncwarp();
  if (row < T)
    for (int h = lane; h < H; h += 32) D[(size_t)h * T + row] = acc[w][h];
}

bool make_head_map(CUtensorMap* m, const void* ptr, int T, int H, int hd);

static int num_sms_attn() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int HD>
static cudaError_t bwd_hd(const CUtensorMap& mQ, const CUtensorMap& mK, const CUtensorMap& mV, const CUtensorMap& mdO,
                          const CUtensorMap& mDS, const CUtensorMap& mDSs, const CUtensorMap& mDK, const CUtensorMap& mDV,
                          const AttnParams& p, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DqCfg<HD>::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dkv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               DkvCfg<HD>::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Dq2Cfg<HD>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // persistent: one CTA per SM (smem-limited), never more CTAs than work items
  const int grid = std::min(p.plan.nq_cap * p.H, num_sms_attn());
  if (grid == 0) return cudaSuccess;
  {
    ProfScope ps(PROF_ATTN_BWD, st, 2);
    if (p.dS) {  // two-pass: dK, dV and the dS^T tiles, then dQ from the tiles
      cudaError_t e = launch_pdl(attn_bwd_dkv_kernel<HD>, grid, DkvCfg<HD>::THREADS, DkvCfg<HD>::SMEM, st, mQ, mK, mV,
                                 mdO, mDSs, mDK, mDV, p);
      if (e == cudaSuccess) e = launch_pdl(attn_bwd_dq2_kernel<HD>, grid, Dq2Cfg<HD>::THREADS, Dq2Cfg<HD>::SMEM, st, mK, mDS, p);
      if (e != cudaSuccess) return e;
    } else {
      cudaError_t e = launch_pdl(attn_bwd_dq_kernel<HD>, grid, DqCfg<HD>::THREADS, DqCfg<HD>::SMEM, st, mQ, mK, mV, mdO, p);
      if (e == cudaSuccess)
        e = launch_pdl(attn_bwd_dkv_kernel<HD>, grid, DkvCfg<HD>::THREADS, DkvCfg<HD>::SMEM, st, mQ, mK, mV, mdO, mDSs,
                       mDK, mDV, p);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t attn_bwd_pre_launch(const void* O, const void* dO, float* D, float* dQacc, int T, int H, int hd,
                                cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (T > 0)
    launch_pdl(attn_bwd_pre_kernel, dim3((T + 7) / 8), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(O),
                                                      reinterpret_cast<const __nv_bfloat16*>(dO), D, T, H, hd);
  (void)dQacc;  // dQ is written exactly once per row by attn_bwd_dq_kernel (pad rows zeroed by the caller)
  return cudaGetLastError();
}

cudaError_t attn_bwd_launch(const void* Qr, const void* Kr, const void* V, const void* dO, const AttnParams& p,
                            cudaStream_t st) {
  CUtensorMap mQ, mK, mV, mdO, mDS, mDSs, mDK, mDV;
  memset(&mDS, 0, sizeof(mDS));
  memset(&mDSs, 0, sizeof(mDSs));
  memset(&mDK, 0, sizeof(mDK));
  memset(&mDV, 0, sizeof(mDV));
  if (p.dS && p.hd == 128 && !p.out_f32) {  // dK / dV drains of full k-tiles by TMA stores: [T][H][128], 64B swizzle
    uint64_t dims[3] = {(uint64_t)p.hd, (uint64_t)p.H, (uint64_t)p.T};
    uint64_t strides[2] = {(uint64_t)p.hd * 2, (uint64_t)p.H * p.hd * 2};
    uint32_t box[3] = {32, 1, 32};
    if (!encode_bf16_map(&mDK, p.dK, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !encode_bf16_map(&mDV, p.dV, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  }
  if (p.dS) {  // dS^T stores from the dK/dV kernel's 32 x 32 warp stages: [rows][H][128] bf16, 64B swizzle
    uint64_t dims[3] = {128, (uint64_t)p.H, (uint64_t)p.ds_slots * 128};
    uint64_t strides[2] = {128 * 2, (uint64_t)p.H * 128 * 2};
    uint32_t box[3] = {32, 1, 32};
    if (!encode_bf16_map(&mDSs, p.dS, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
  }
  if (!make_head_map(&mQ, Qr, p.T, p.H, p.hd) || !make_head_map(&mK, Kr, p.T, p.H, p.hd) ||
      !make_head_map(&mV, V, p.T, p.H, p.hd) || !make_head_map(&mdO, dO, p.T, p.H, p.hd) ||
      (p.dS && !make_head_map(&mDS, p.dS, p.ds_slots * 128, p.H, 128)))
    return cudaErrorInvalidValue;
  switch ((p.hd + 31) / 32 * 32) {
    case 32: return bwd_hd<32>(mQ, mK, mV, mdO, mDS, mDSs, mDK, mDV, p, st);
    case 64: return bwd_hd<64>(mQ, mK, mV, mdO, mDS, mDSs, mDK, mDV, p, st);
    case 96: return bwd_hd<96>(mQ, mK, mV, mdO, mDS, mDSs, mDK, mDV, p, st);
    case 128: return bwd_hd<128>(mQ, mK, mV, mdO, mDS, mDSs, mDK, mDV, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cadet

#ifdef CADET_PHASE_TIMING
extern "C" int cadet_debug_phase_read(unsigned long long* out, int n) {
  if (n > 8192 * 16) n = 8192 * 16;
  cudaMemcpyFromSymbol(out, cadet::g_phase, sizeof(unsigned long long) * n);
  return n;
}
extern "C" int cadet_debug_trace_read(unsigned long long* out, int n) {
  if (n > 8192 * 12) n = 8192 * 12;
  cudaMemcpyFromSymbol(out, cadet::g_trace, sizeof(unsigned long long) * n);
  return n;
}
extern "C" int cadet_debug_tl_read(unsigned long long* out, int n) {
  if (n > 4 * 4096) n = 4 * 4096;
  cudaMemcpyFromSymbol(out, cadet::g_tl, sizeof(unsigned long long) * n);
  return n;
}
extern "C" int cadet_debug_tl_reset() {
  static unsigned long long z[4 * 4096];
  cudaMemcpyToSymbol(cadet::g_tl, z, sizeof(z));
  return 0;
}
extern "C" int cadet_debug_phase_reset() {
  static unsigned long long z[8192 * 16];
  cudaMemcpyToSymbol(cadet::g_phase, z, sizeof(z));
  return 0;
}
#endif
