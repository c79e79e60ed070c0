// A10: attention backward (adjoint of PAPER.md Eq. 7) for the packed, session-masked layout.
//
// One CTA per (128-key tile of one sequence, head), k-tiles in descending cost order.  K_j, V_j
// stay in shared memory; the CTA walks the q-tiles that see k-tile j (the transpose of the
// forward visit rule: q-tile i visits j iff j < nf_i or kt2_i <= j <= i), and per q-tile:
//   S^T  = K_j Q_i^T,  dP^T = V_j dO_i^T            (tcgen05, TMEM cols [0,128) and [128,256))
//   P^T  = exp2(S^T scale log2e - LSE_i log2e) on visible cells, dS^T = P^T (dP^T - D_i) * scale
//   dV  += P^T dO_i,  dK += dS^T Q_i                   (TMEM accumulators [256,384), [384,512))
//   dQ_i = dS K_j  (TMEM [128, 128+HDP), reusing dP^T) -> fp32 atomics into the dQ accumulator
//
//   warp 0     : TMA producer (K_j, V_j once; Q_i, dO_i per q-tile)
//   warp 1     : TMEM owner + MMA issuer
//   warps 2..5 : thread = key row for P^T / dS^T (TMEM lane), = query row for the dQ drain
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
  static constexpr int PT_OFF = DO_OFF + G::TILE_BYTES;
  static constexpr int DS_OFF = PT_OFF + 32768;
  static constexpr int VEC_OFF = DS_OFF + 32768;      // [2][4][128] x 4 B
  static constexpr int BAR_OFF = VEC_OFF + 2 * 4 * 128 * 4;
  static constexpr int USED = BAR_OFF + 256;
  static constexpr int SMEM = (USED + 1024 > 118784 ? USED + 1024 : 118784);
  static constexpr int S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 384;
};

struct BwdBars {
  uint64_t kv_full, qd_full, qd_empty, sdp_full, pds_full, mma2_done, dq_free;
  uint32_t tmem_base;
};

__device__ __forceinline__ bool q_sees_k(const QTileInfo& qi, int kt) {
  return kt < qi.nf || (kt >= qi.kt2 && kt <= qi.qt);
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
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
  float* vec = reinterpret_cast<float*>(smem + C::VEC_OFF);  // [2][4][128]: lse2, D, e (int), q|pp (int)
  const uint32_t warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->qd_full, 1);
    mbar_init(&bars->qd_empty, 1);
    mbar_init(&bars->sdp_full, 1);
    mbar_init(&bars->pds_full, 128);
    mbar_init(&bars->mma2_done, 1);
    mbar_init(&bars->dq_free, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============================ producer
    if (elect_one()) {
      tma_prefetch(&mQ);
      tma_prefetch(&mK);
      tma_prefetch(&mV);
      tma_prefetch(&mdO);
      mbar_expect_tx(&bars->kv_full, 2 * G::TILE_BYTES);
#pragma unroll
      for (int blk = 0; blk < G::NB; ++blk) {
        tma_load_3d(smem + C::K_OFF + blk * G::BLK, &mK, &bars->kv_full, blk * G::CB, h, k0);
        tma_load_3d(smem + C::V_OFF + blk * G::BLK, &mV, &bars->kv_full, blk * G::CB, h, k0);
      }
      int it = 0;
      for (int qt = kt; qt < nq_s; ++qt) {
        const QTileInfo qi = p.plan.qinfo[tile0 + qt];
        if (!q_sees_k(qi, kt)) continue;
        if (it > 0) mbar_wait(&bars->qd_empty, (it - 1) & 1);
        const int q0 = sa + qt * 128;
        mbar_expect_tx(&bars->qd_full, 2 * G::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < G::NB; ++blk) {
          tma_load_3d(smem + C::Q_OFF + blk * G::BLK, &mQ, &bars->qd_full, blk * G::CB, h, q0);
          tma_load_3d(smem + C::DO_OFF + blk * G::BLK, &mdO, &bars->qd_full, blk * G::CB, h, q0);
        }
        ++it;
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
      const uint32_t sPT = smem_u32(smem + C::PT_OFF), sDS = smem_u32(smem + C::DS_OFF);
      mbar_wait(&bars->kv_full, 0);
      int it = 0;
      for (int qt = kt; qt < nq_s; ++qt) {
        const QTileInfo qi = p.plan.qinfo[tile0 + qt];
        if (!q_sees_k(qi, kt)) continue;
        mbar_wait(&bars->qd_full, it & 1);
        if (it > 0) mbar_wait(&bars->dq_free, (it - 1) & 1);  // dQ_{i-1} drained from the dP region
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::S_COL, kmajor_desc<HD>(sK, kk), kmajor_desc<HD>(sQ, kk), id_s, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < G::HDP / 16; ++kk)
          mma_bf16_ss(tmem + C::DP_COL, kmajor_desc<HD>(sV, kk), kmajor_desc<HD>(sdO, kk), id_s, kk > 0 ? 1u : 0u);
        mma_commit(&bars->sdp_full);
        mbar_wait(&bars->pds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ss(tmem + C::DV_COL, p_kmajor_desc(sPT, kk), mnmajor_desc<HD>(sdO, kk), id_kv,
                      (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ss(tmem + C::DK_COL, p_kmajor_desc(sDS, kk), mnmajor_desc<HD>(sQ, kk), id_kv,
                      (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          mma_bf16_ss(tmem + C::DP_COL, p_mnmajor_desc(sDS, kk), mnmajor_desc<HD>(sK, kk), id_q, kk > 0 ? 1u : 0u);
        mma_commit(&bars->qd_empty);
        mma_commit(&bars->mma2_done);
        ++it;
      }
    }
  } else {
    // ============================ compute warps 2..5
    const uint32_t quarter = warp & 3;
    const int tr = quarter * 32 + lane;      // TMEM lane = key row (P^T) = query row (dQ drain)
    const int ct = threadIdx.x - 64;         // 0..127 loader index
    const int key = k0 + tr;
    const bool key_valid = tr < keys_valid;
    const float sl2 = p.scale_log2;
    const float LOG2E = 1.4426950408889634f;
    uint8_t* sPT = smem + C::PT_OFF;
    uint8_t* sDS = smem + C::DS_OFF;
    int it = 0;
    for (int qt = kt; qt < nq_s; ++qt) {
      const QTileInfo qi = p.plan.qinfo[tile0 + qt];
      if (!q_sees_k(qi, kt)) continue;
      const int q0 = sa + qt * 128;
      const int qvalid = min(128, se - q0);
      float* vb = vec + (it & 1) * 512;
      int* vbi = reinterpret_cast<int*>(vb);
      {  // per-query vectors of this q-tile
        const int q = q0 + ct;
        const bool v = ct < qvalid;
        vb[ct] = v ? p.lse[(size_t)h * p.T + q] * LOG2E : INFINITY;
        vb[128 + ct] = v ? p.D[(size_t)h * p.T + q] : 0.f;
        vbi[256 + ct] = v ? p.plan.kv_end[q] : -1;
        vbi[384 + ct] = v ? (q | (p.plan.row_pp[q] ? (1 << 30) : 0)) : -2;
      }
      named_bar_sync(1, 128);
      mbar_wait(&bars->sdp_full, it & 1);
      tc_fence_after();
      if (it > 0) {  // PT / DST shared buffers are free once the previous MMAs completed
        mbar_wait(&bars->mma2_done, (it - 1) & 1);
      }
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t us[32], ud[32];
        tmem_ld32(tmem_addr(tmem, quarter, C::S_COL + c * 32), us);
        tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + c * 32), ud);
        tmem_ld_wait();
        uint32_t wp[16], wd[16];
#pragma unroll
        for (int q2 = 0; q2 < 32; q2 += 2) {
          float pv[2], dv[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = c * 32 + q2 + e;
            const int qe = vbi[256 + col];
            const int qw = vbi[384 + col];
            const int qq = qw & ~(1 << 30);
            const bool ppq = (qw >= 0) && (qw & (1 << 30));
            const bool ok = key_valid && qw >= 0 && ((key < qe) || (key == qq) || (ppq && key == qq - 1));
            const float s = __uint_as_float(us[q2 + e]);
            const float pr = ok ? fast_exp2(fmaf(s, sl2, -vb[col])) : 0.f;
            pv[e] = pr;
            dv[e] = pr * (__uint_as_float(ud[q2 + e]) - vb[128 + col]) * p.scale;
          }
          wp[q2 >> 1] = pack_bf16(pv[0], pv[1]);
          wd[q2 >> 1] = pack_bf16(dv[0], dv[1]);
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          *reinterpret_cast<uint4*>(sPT + p_off(tr, c * 32 + ch * 8)) =
              make_uint4(wp[ch * 4], wp[ch * 4 + 1], wp[ch * 4 + 2], wp[ch * 4 + 3]);
          *reinterpret_cast<uint4*>(sDS + p_off(tr, c * 32 + ch * 8)) =
              make_uint4(wd[ch * 4], wd[ch * 4 + 1], wd[ch * 4 + 2], wd[ch * 4 + 3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->pds_full);
      // ---- dQ_i drain: thread = query row
      mbar_wait(&bars->mma2_done, it & 1);
      tc_fence_after();
      {
        const int q = q0 + tr;
        const bool qv = tr < qvalid;
#pragma unroll 1
        for (int c = 0; c < G::HDP / 32; ++c) {
          uint32_t u[32];
          tmem_ld32(tmem_addr(tmem, quarter, C::DP_COL + c * 32), u);
          tmem_ld_wait();
          if (qv) {
            float* dst = p.dQ + (size_t)q * p.d + (size_t)h * p.hd + c * 32;
            const int ncol = min(32, p.hd - c * 32);
            for (int j = 0; j < ncol; j += 4)
              atomicAdd(reinterpret_cast<float4*>(dst + j),
                        make_float4(__uint_as_float(u[j]), __uint_as_float(u[j + 1]), __uint_as_float(u[j + 2]),
                                    __uint_as_float(u[j + 3])));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
      ++it;
    }
    // ---- dK, dV epilogue (thread = key row)
    if (it > 0) {
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
  attn_bwd_kernel<HD><<<grid, 192, C::SMEM, st>>>(mQ, mK, mV, mdO, p);
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
