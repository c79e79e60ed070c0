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
//                P_j read from TMEM (TS form: P overwrites the consumed S columns as packed bf16)
//   warps 2..5 : softmax, thread = query row: tcgen05.ld S, mask, online softmax with
//                conditional rescaling (threshold 2^8), tcgen05.st P, O rescale, final O / l, LSE.
// ~96 KB of shared memory and 256 TMEM columns per CTA, so two CTAs share an SM and one CTA's
// softmax overlaps the other's MMAs (the role FA4's two softmax warpgroups play).
#include "attn_common.cuh"
#include "launch.cuh"
#include "prof.cuh"

namespace cadet {

#ifdef CADET_PHASE_TIMING
__device__ unsigned long long g_phase_fwd[8192][8];
#define FT_MARK(slot)                                                              \
  if (lane == 0 && blockIdx.x < 8192) {                                             \
    unsigned long long _n = clock64();                                              \
    atomicAdd(&g_phase_fwd[blockIdx.x][slot], _n - _ft);                            \
    _ft = _n;                                                                       \
  }
#else
#define FT_MARK(slot)
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
      auto exp_store = [&](int c, const uint32_t (&u)[32]) {
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          const float p0 = fast_exp2(fmaf(__uint_as_float(u[q]), sl2, -base));
          const float p1 = fast_exp2(fmaf(__uint_as_float(u[q + 1]), sl2, -base));
          rs += p0 + p1;
          w[q >> 1] = pack_bf16(p0, p1);
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
      l = l * factor + rs;
      FT_MARK(6)
    }
#ifdef CADET_PHASE_TIMING
#undef lane
    (void)lane_save;
#endif
    // ---- epilogue: O / l, LSE
    if (n_kv > 0) {
      mbar_wait(&bars->pv_done, (n_kv - 1) & 1);
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
  static unsigned long long z[8192 * 8];
  cudaMemcpyToSymbol(cadet::g_phase_fwd, z, sizeof(z));
  return 0;
}
#endif
