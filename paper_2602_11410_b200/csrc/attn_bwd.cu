// A10: attention backward (adjoint of PAPER.md Eq. 7) for the packed, session-masked layout.
//
// One CTA per (128-key tile of one sequence, head), k-tiles in descending cost order.  K_j, V_j
// stay in shared memory; the CTA walks the q-tiles that see k-tile j (transpose of the forward
// visit rule: q-tile i visits j iff j < nf_i or kt2_i <= j <= i; list built once in smem), and per
// q-tile i:
//   S^T  = K_j Q_i^T           -> TMEM [0,128)        dP^T = V_j dO_i^T -> TMEM [128,256)
//   P^T  = exp2(S^T scale log2e - LSE_i log2e) on visible cells (predicate only on non-FULL pairs)
//   dS^T = P^T (dP^T - D_i) scale
//   P^T, dS^T are written back as packed bf16 over the consumed S^T / dP^T columns and feed
//   dV += P^T dO_i and dK += dS^T Q_i as TMEM-A (TS) MMAs into TMEM [256,384) / [384,512);
//   dS^T also goes to shared memory for dQ_i = dS K_j (MN-major A), written over [128,256) and
//   drained by four dedicated warps with fp32 vector atomics while the next S^T is computed.
//
//   warp 0      : TMA producer (K_j, V_j once; Q_i, dO_i per q-tile)
//   warp 1      : TMEM owner + MMA issuer
//   warps 2..5  : thread = key row (TMEM lane): P^T, dS^T
//   warps 6..9  : thread = query row: dQ drain; final dK, dV epilogue
#include "attn_common.cuh"
#include "prof.cuh"

namespace cadet {

template <int HD>
struct BwdCfg {
  using G = HeadGeom<HD>;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + G::TILE_BYTES;
  static constexpr int Q_OFF = V_OFF + G::TILE_BYTES;
  static constexpr int DO_OFF = Q_OFF + G::TILE_BYTES;
  static constexpr int DS_OFF = DO_OFF + G::TILE_BYTES;  // dS^T bf16 [128 keys x 128 q], 128B swizzle
  static constexpr int VEC_OFF = DS_OFF + 32768;          // [2][4][128] x 4 B: lse2, D, e, q|pp
  static constexpr int LIST_OFF = VEC_OFF + 2 * 4 * 128 * 4;
  static constexpr int MAX_LIST = 512;                    // visited q-tiles per k-tile (T/128 bound)
  static constexpr int BAR_OFF = LIST_OFF + MAX_LIST * 4;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 384;
  static constexpr int THREADS = 320;
};

struct BwdBars {
  uint64_t kv_full, qd_full, qd_empty, s_full, dp_full, pds_ready, dq_full, dq_free;
  uint32_t tmem_base;
  int32_t n_it;
};

__device__ __forceinline__ bool q_sees_k(const QTileInfo& qi, int kt) {
  return kt < qi.nf || (kt >= qi.kt2 && kt <= qi.qt);
}

template <int HD>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                    const AttnParams p) {
  using G = HeadGeom<HD>;
  using C = BwdCfg<HD>;
  const int nq_total = p.plan.counters[0];
  const int b = blockIdx.x / p.H;
  const int h = blockIdx.x % p.H;
  if (b >= nq_total) return;
  const int g = p.plan.bwd_order[b];
  const QTileInfo ki = p.plan.qinfo[g];
  const int kt = ki.qt;
  const int sa = p.cu[ki.seq], se = p.cu[ki.seq + 1];
  const int tile0 = g - kt;  // tile index of q-tile 0 of this sequence
  const int nq_s = (se - sa + 127) / 128;
  const int k0 = sa + kt * 128;
  const int keys_valid = min(128, se - k0);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + C::BAR_OFF);
  float* vec = reinterpret_cast<float*>(smem + C::VEC_OFF);
  int* list = reinterpret_cast<int*>(smem + C::LIST_OFF);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0) {
    // visited q-tiles (and whether the (q-tile, k-tile) pair is FULL) -> smem list
    int n = 0;
    for (int base = kt; base < nq_s; base += 32) {
      const int qt = base + (int)lane;
      int entry = -1;
      if (qt < nq_s) {
        const QTileInfo qi = p.plan.qinfo[tile0 + qt];
        if (q_sees_k(qi, kt)) {
          const bool full = qi.rows == 128 && qi.emin >= (kt + 1) * 128;
          entry = qt | (full ? (1 << 30) : 0);
        }
      }
      const uint32_t m = __ballot_sync(0xffffffffu, entry >= 0);
      const int pos = n + __popc(m & ((1u << lane) - 1u));
      if (entry >= 0 && pos < C::MAX_LIST) list[pos] = entry;
      n += __popc(m);
    }
    if (lane == 0) {
      bars->n_it = min(n, C::MAX_LIST);
      mbar_init(&bars->kv_full, 1);
      mbar_init(&bars->qd_full, 1);
      mbar_init(&bars->qd_empty, 1);
      mbar_init(&bars->s_full, 1);
      mbar_init(&bars->dp_full, 1);
      mbar_init(&bars->pds_ready, 128);
      mbar_init(&bars->dq_full, 1);
      mbar_init(&bars->dq_free, 128);
      fence_mbar_init();
    }
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int n_it = bars->n_it;

  if (warp == 0) {
    // ============================ producer
    if (elect_one()) {
      mbar_expect_tx(&bars->kv_full, 2 * G::TILE_BYTES);
#pragma unroll
      for (int blk = 0; blk < G::NB; ++blk) {
        tma_load_3d(smem + C::K_OFF + blk * G::BLK, &mK, &bars->kv_full, blk * G::CB, h, k0);
        tma_load_3d(smem + C::V_OFF + blk * G::BLK, &mV, &bars->kv_full, blk * G::CB, h, k0);
      }
      for (int it = 0; it < n_it; ++it) {
        const int q0 = sa + (list[it] & 0xFFFF) * 128;
        if (it > 0) mbar_wait(&bars->qd_empty, (it - 1) & 1);
        mbar_expect_tx(&bars->qd_full, 2 * G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk) {
          tma_load_3d(smem + C::Q_OFF + blk * G::BLK, &mQ, &bars->qd_full, blk * G::CB, h, q0);
          tma_load_3d(smem + C::DO_OFF + blk * G::BLK, &mdO, &bars->qd_full, blk * G::CB, h, q0);
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    if (elect_one()) {
      const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t id_kv = idesc_bf16(128, G::HDP, 0, 1);
      const uint32_t id_q = idesc_bf16(128, G::HDP, 1, 1);
      const uint32_t sK = smem_u32(smem + C::K_OFF), sV = smem_u32(smem + C::V_OFF);
      const uint32_t sQ = smem_u32(smem + C::Q_OFF), sdO = smem_u32(smem + C::DO_OFF);
      const uint32_t sDS = smem_u32(smem + C::DS_OFF);
      mbar_wait(&bars->kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(&bars->qd_full, it & 1);
        tc_fence_after();
        // S^T_i over the P^T_{i-1} columns: in-order after dV_{i-1}, which read them.
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::S_COL, kmajor_desc<HD>(sK, kk), kmajor_desc<HD>(sQ, kk), id_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->s_full);
        if (it > 0) {
          mbar_wait(&bars->dq_free, (it - 1) & 1);  // dQ_{i-1} drained from [128, 256)
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::DP_COL, kmajor_desc<HD>(sV, kk), kmajor_desc<HD>(sdO, kk), id_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->dp_full);
        mbar_wait(&bars->pds_ready, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ts(tmem + C::DV_COL, tmem + C::S_COL + kk * 8, mnmajor_desc<HD>(sdO, kk), id_kv,
                      (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ts(tmem + C::DK_COL, tmem + C::DP_COL + kk * 8, mnmajor_desc<HD>(sQ, kk), id_kv,
                      (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&bars->qd_empty);
        // dQ_i = dS K_j over the dS^T columns: in-order after dK_i, which read them.
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ss(tmem + C::DP_COL, p_mnmajor_desc(sDS, kk), mnmajor_desc<HD>(sK, kk), id_q, kk > 0 ? 1u : 0u);
        mma_commit(&bars->dq_full);
      }
    }
  } else if (warp < 6) {
    // ============================ P^T / dS^T warps (thread = key row)
    const uint32_t quarter = warp & 3;
    const int tr = quarter * 32 + lane;
    const int ct = threadIdx.x - 64;  // 0..127 vector-loader index
    const int key = k0 + tr;
    const bool key_valid = tr < keys_valid;
    const float sl2 = p.scale_log2;
    const float LOG2E = 1.4426950408889634f;
    uint8_t* sDS = smem + C::DS_OFF;
    for (int it = 0; it < n_it; ++it) {
      const int ent = list[it];
      const bool full = (ent >> 30) & 1;
      const int q0 = sa + (ent & 0xFFFF) * 128;
      const int qvalid = min(128, se - q0);
      float* vb = vec + (it & 1) * 512;
      int* vbi = reinterpret_cast<int*>(vb);
      {
        const int q = q0 + ct;
        const bool v = ct < qvalid;
        vb[ct] = v ? p.lse[(size_t)h * p.T + q] * LOG2E : INFINITY;
        vb[128 + ct] = v ? p.D[(size_t)h * p.T + q] : 0.f;
        vbi[256 + ct] = v ? p.plan.kv_end[q] : -1;
        vbi[384 + ct] = v ? (q | (p.plan.row_pp[q] ? (1 << 30) : 0)) : -2;
      }
      named_bar_sync(1, 128);
      mbar_wait(&bars->s_full, it & 1);
      tc_fence_after();
      float pr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t us[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + c * 32), us);
        tmem_ld_wait();
#pragma unroll
        for (int q4 = 0; q4 < 32; q4 += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(vb + c * 32 + q4);  // broadcast LDS.128
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) pr[c * 32 + q4 + e] = fast_exp2(fmaf(__uint_as_float(us[q4 + e]), sl2, -lv[e]));
        }
        if (!full) {
#pragma unroll
          for (int q4 = 0; q4 < 32; q4 += 4) {
            const int4 e4 = *reinterpret_cast<const int4*>(vbi + 256 + c * 32 + q4);
            const int4 w4 = *reinterpret_cast<const int4*>(vbi + 384 + c * 32 + q4);
            const int ev[4] = {e4.x, e4.y, e4.z, e4.w}, wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int qw = wv[e];
              const int qq = qw & ~(1 << 30);
              const bool ppq = (qw >= 0) && (qw & (1 << 30));
              const bool ok = key_valid && qw >= 0 && ((key < ev[e]) || (key == qq) || (ppq && key == qq - 1));
              if (!ok) pr[c * 32 + q4 + e] = 0.f;
            }
          }
        }
      }
      // P^T (bf16) over the consumed S^T columns [0, 64)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 32; q += 2) w[q >> 1] = pack_bf16(pr[c * 32 + q], pr[c * 32 + q + 1]);
        tmem_st16(tmem_addr(tmem, quarter, C::S_COL + c * 16), w);
      }
      mbar_wait(&bars->dp_full, it & 1);
      tc_fence_after();
      if (it > 0) mbar_wait(&bars->dq_full, (it - 1) & 1);  // dQ_{i-1} MMA has finished reading dS smem
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t ud[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + c * 32), ud);
        tmem_ld_wait();
        uint32_t w[16];
#pragma unroll
        for (int q4 = 0; q4 < 32; q4 += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(vb + 128 + c * 32 + q4);
          const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
          float ds[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) ds[e] = pr[c * 32 + q4 + e] * (__uint_as_float(ud[q4 + e]) - dv[e]) * p.scale;
          w[q4 >> 1] = pack_bf16(ds[0], ds[1]);
          w[(q4 >> 1) + 1] = pack_bf16(ds[2], ds[3]);
        }
        tmem_st16(tmem_addr(tmem, quarter, C::DP_COL + c * 16), w);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          *reinterpret_cast<uint4*>(sDS + p_off(tr, c * 32 + ch * 8)) =
              make_uint4(w[ch * 4], w[ch * 4 + 1], w[ch * 4 + 2], w[ch * 4 + 3]);
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->pds_ready);
    }
  } else {
    // ============================ dQ drain warps (thread = query row), then dK / dV epilogue
    const uint32_t quarter = warp & 3;
    const int tr = quarter * 32 + lane;
    for (int it = 0; it < n_it; ++it) {
      const int q0 = sa + (list[it] & 0xFFFF) * 128;
      const int q = q0 + tr;
      const bool qv = q < se;
      mbar_wait(&bars->dq_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < G::HDP / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + c * 32), u);
        tmem_ld_wait();
        if (qv) {
          float* dst = p.dQ + (size_t)q * p.d + (size_t)h * p.hd + c * 32;
          const int ncol = min(32, p.hd - c * 32);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (j < ncol)
              atomicAdd(reinterpret_cast<float4*>(dst + j),
                        make_float4(__uint_as_float(u[j]), __uint_as_float(u[j + 1]), __uint_as_float(u[j + 2]),
                                    __uint_as_float(u[j + 3])));
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
    }
    // dK, dV (thread = key row): all MMAs completed (the last dq_full tracks every prior MMA)
    const int key = k0 + tr;
    const bool key_valid = tr < keys_valid;
    if (n_it > 0) {
      tc_fence_after();
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        void* out = which == 0 ? p.dK : p.dV;
        const int col0 = which == 0 ? C::DK_COL : C::DV_COL;
#pragma unroll 1
        for (int c = 0; c < G::HDP / 32; ++c) {
          uint32_t u[32];
          tmem_ld32(tmem_addr(tmem, quarter, col0 + c * 32), u);
          tmem_ld_wait();
          if (key_valid) {
            const size_t off = (size_t)key * p.d + (size_t)h * p.hd + c * 32;
            const int ncol = min(32, p.hd - c * 32);
            if (p.out_f32) {
              float* o = reinterpret_cast<float*>(out) + off;
              for (int j = 0; j < ncol; j += 4)
                *reinterpret_cast<float4*>(o + j) = make_float4(__uint_as_float(u[j]), __uint_as_float(u[j + 1]),
                                                                __uint_as_float(u[j + 2]), __uint_as_float(u[j + 3]));
            } else {
              __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + off;
              for (int j = 0; j < ncol; j += 8)
                *reinterpret_cast<uint4*>(o + j) =
                    make_uint4(pack_bf16(__uint_as_float(u[j]), __uint_as_float(u[j + 1])),
                               pack_bf16(__uint_as_float(u[j + 2]), __uint_as_float(u[j + 3])),
                               pack_bf16(__uint_as_float(u[j + 4]), __uint_as_float(u[j + 5])),
                               pack_bf16(__uint_as_float(u[j + 6]), __uint_as_float(u[j + 7])));
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// D_i = rowsum(dO_i * O_i) per head (FlashAttention preprocess), bf16 inputs, fp32 out [H, T].
__global__ void __launch_bounds__(256) attn_bwd_pre_kernel(const __nv_bfloat16* O, const __nv_bfloat16* dO, float* D,
                                                            int T, int H, int hd) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int d = H * hd;
  for (int h = 0; h < H; ++h) {
    float acc = 0.f;
    for (int c = lane * 2; c < hd; c += 64) {
      const float2 o = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(O + (size_t)row * d + h * hd + c));
      const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dO + (size_t)row * d + h * hd + c));
      acc = fmaf(o.x, g.x, fmaf(o.y, g.y, acc));
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) D[(size_t)h * T + row] = acc;
  }
}

bool make_head_map(CUtensorMap* m, const void* ptr, int T, int H, int hd);

template <int HD>
static cudaError_t bwd_hd(const CUtensorMap& mQ, const CUtensorMap& mK, const CUtensorMap& mV, const CUtensorMap& mdO,
                          const AttnParams& p, cudaStream_t st) {
  using C = BwdCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = p.plan.nq_cap * p.H;
  if (grid == 0) return cudaSuccess;
  ProfScope ps(PROF_ATTN_BWD, st, 1);
  attn_bwd_kernel<HD><<<grid, C::THREADS, C::SMEM, st>>>(mQ, mK, mV, mdO, p);
  return cudaGetLastError();
}

cudaError_t attn_bwd_pre_launch(const void* O, const void* dO, float* D, float* dQacc, int T, int H, int hd,
                                cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  if (T > 0)
    attn_bwd_pre_kernel<<<(T + 7) / 8, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(O),
                                                      reinterpret_cast<const __nv_bfloat16*>(dO), D, T, H, hd);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && dQacc) e = cudaMemsetAsync(dQacc, 0, sizeof(float) * (size_t)T * H * hd, st);
  return e;
}

cudaError_t attn_bwd_launch(const void* Qr, const void* Kr, const void* V, const void* dO, const AttnParams& p,
                            cudaStream_t st) {
  CUtensorMap mQ, mK, mV, mdO;
  if (!make_head_map(&mQ, Qr, p.T, p.H, p.hd) || !make_head_map(&mK, Kr, p.T, p.H, p.hd) ||
      !make_head_map(&mV, V, p.T, p.H, p.hd) || !make_head_map(&mdO, dO, p.T, p.H, p.hd))
    return cudaErrorInvalidValue;
  switch ((p.hd + 31) / 32 * 32) {
    case 32: return bwd_hd<32>(mQ, mK, mV, mdO, p, st);
    case 64: return bwd_hd<64>(mQ, mK, mV, mdO, p, st);
    case 96: return bwd_hd<96>(mQ, mK, mV, mdO, p, st);
    case 128: return bwd_hd<128>(mQ, mK, mV, mdO, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cadet
