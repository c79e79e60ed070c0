// A0 chunk, A1 mask plan, A13 pack: the integer part of the hot path (bit-exact).
//   plan_seq_kernel   : validate offsets, tile offsets (scan of ceil(len/128)), export offsets
//   plan_row_kernel   : per row kv_end (binary search over int64 timestamps / session ids), pairs
//   plan_tile_kernel  : per 128-row tile the visit bounds + LPT cost histograms
//   plan_order_kernel : descending-cost bucket offsets;  plan_scatter_kernel : work lists
// The mask itself is never materialised: attention kernels evaluate
//   allowed(i, j) = j < kv_end[i]  ||  j == i  ||  (pp_i && j == i - 1)
// on PARTIAL rows only.  This is exactly the structure of the mask of PAPER.md Eq. 6 / Fig. 3 /
// P:540-546 when timestamps (and session ids) are non-decreasing inside a sequence.
#include "plan.cuh"
#include "launch.cuh"
#include "prof.cuh"
#include "ptx.cuh"

namespace cadet {

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static int32_t nq_cap_of(int32_t n, int32_t T) { return (T + TILE - 1) / TILE + n; }
static int32_t hmax_of(int32_t max_seqlen) { return (max_seqlen + TILE - 1) / TILE + 3; }
// sum_s nq_s (nq_s + 1) / 2 with sum_s nq_s <= nq_cap and nq_s <= hmax
static size_t list_cap_of(size_t nq, size_t hm) { return nq * (hm + 1) / 2 + hm; }

size_t plan_bytes(int32_t n, int32_t T, int32_t max_seqlen) {
  const size_t nq = nq_cap_of(n, T), hm = hmax_of(max_seqlen);
  size_t b = 0;
  b += align256(16);                        // err
  b += align256(4 * sizeof(int32_t));       // counters
  b += align256(sizeof(unsigned long long));
  b += align256((size_t)T * 4) * 2;         // kv_end, row_seq
  b += align256((size_t)T);                 // row_pp
  b += align256((size_t)(n + 1) * 4);
  b += align256((size_t)(n + 1) * 8);
  b += align256(nq * sizeof(QTileInfo));
  b += align256(nq * 4) * 2;
  b += align256(hm * 3 * 4);
  b += align256((size_t)(n + 1) * 4);
  b += align256(nq * 4) * 2;
  b += align256(list_cap_of(nq, hm) * 4);
  b += align256((size_t)(n + 1) * 4);       // seq_rank
  b += align256(nq * 4);                    // pair_list
  b += align256(64 * sizeof(float2));       // RoPE theta (hi, lo)
  b += align256((size_t)T * sizeof(float2));  // per-row rebased time (hi, lo)
  return b;
}

PlanView plan_carve(void* ws, int32_t n, int32_t T, int32_t max_seqlen) {
  PlanView v;
  v.nq_cap = nq_cap_of(n, T);
  v.hmax = hmax_of(max_seqlen);
  v.list_cap = (int32_t)list_cap_of(v.nq_cap, v.hmax);
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += align256(bytes);
    return r;
  };
  v.err = reinterpret_cast<uint32_t*>(take(16));
  v.counters = reinterpret_cast<int32_t*>(take(16));
  v.pairs = reinterpret_cast<unsigned long long*>(take(8));
  v.kv_end = reinterpret_cast<int32_t*>(take((size_t)T * 4));
  v.row_seq = reinterpret_cast<int32_t*>(take((size_t)T * 4));
  v.row_pp = reinterpret_cast<uint8_t*>(take((size_t)T));
  v.tile_off = reinterpret_cast<int32_t*>(take((size_t)(n + 1) * 4));
  v.tc_off = reinterpret_cast<int64_t*>(take((size_t)(n + 1) * 8));
  v.qinfo = reinterpret_cast<QTileInfo*>(take((size_t)v.nq_cap * sizeof(QTileInfo)));
  v.fwd_order = reinterpret_cast<int32_t*>(take((size_t)v.nq_cap * 4));
  v.bwd_order = reinterpret_cast<int32_t*>(take((size_t)v.nq_cap * 4));
  v.hist = reinterpret_cast<int32_t*>(take((size_t)v.hmax * 3 * 4));
  v.tri_off = reinterpret_cast<int32_t*>(take((size_t)(n + 1) * 4));
  v.bwd_off = reinterpret_cast<int32_t*>(take((size_t)v.nq_cap * 4));
  v.bwd_cnt = reinterpret_cast<int32_t*>(take((size_t)v.nq_cap * 4));
  v.bwd_list = reinterpret_cast<int32_t*>(take(list_cap_of(v.nq_cap, v.hmax) * 4));
  v.seq_rank = reinterpret_cast<int32_t*>(take((size_t)(n + 1) * 4));
  v.pair_list = reinterpret_cast<int32_t*>(take((size_t)v.nq_cap * 4));
  v.theta = reinterpret_cast<float2*>(take(64 * sizeof(float2)));
  v.rope_dt = reinterpret_cast<float2*>(take((size_t)T * sizeof(float2)));
  return v;
}

// ---------------------------------------------------------------- block scan helper (1024 threads)
template <typename T>
__device__ T block_exclusive_scan(T x, T* sh, T& total) {
  const int tid = threadIdx.x;
  sh[tid] = x;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    T y = (tid >= off) ? sh[tid - off] : T(0);
    __syncthreads();
    sh[tid] += y;
    __syncthreads();
  }
  total = sh[blockDim.x - 1];
  T incl = sh[tid];
  __syncthreads();
  return incl - x;
}

__device__ __forceinline__ int32_t seq_len_safe(const int32_t* cu, int s, int T) {
  int a = cu[s], e = cu[s + 1];
  a = min(max(a, 0), T);
  e = min(max(e, a), T);
  return e - a;
}

// ---------------------------------------------------------------- K1
__global__ void __launch_bounds__(1024) plan_seq_kernel(PlanArgs a, PlanView v) {
  pdl_trigger();
  pdl_wait();
  __shared__ long long sh[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (a.n + nt - 1) / nt;
  const int s0 = min(tid * per, a.n), s1 = min(s0 + per, a.n);
  uint32_t err = 0;
  if (tid < 64) {  // RoPE theta_i in fp64, stored as a float hi + lo pair (exact to ~2^-48 relative)
    float2 th = make_float2(0.f, 0.f);
    if (tid < a.head_dim / 2 && a.rope_dt_max > 0.0) {
      const double x = (a.rope_phi_min / a.rope_dt_max) * pow(a.rope_base, 2.0 * tid / (double)a.head_dim);
      th.x = (float)x;
      th.y = (float)(x - (double)th.x);
    }
    v.theta[tid] = th;
  }
  if (tid == 0) {
    if (a.n > 0 && a.cu[0] != 0) err |= ERRBIT_OFFSETS;
    if (a.n > 0 && a.cu[a.n] > a.T) err |= ERRBIT_OFFSETS;
  }
  long long nq_sum = 0, tc_sum = 0, tri_sum = 0;
  for (int s = s0; s < s1; ++s) {
    const int ra = a.cu[s], re = a.cu[s + 1];
    if (re <= ra) err |= ERRBIT_OFFSETS;
    const int len = seq_len_safe(a.cu, s, a.T);
    if (len > a.max_seqlen) err |= ERRBIT_TOO_LONG;
    if (a.ncand && (a.ncand[s] < 0 || a.ncand[s] > len)) err |= ERRBIT_CAND;
    const long long nq = (min(len, a.max_seqlen) + TILE - 1) / TILE;
    nq_sum += nq;
    tc_sum += nq * nq;
    tri_sum += nq * (nq + 1) / 2;
  }
  long long tot_nq, tot_tc, tot_tri;
  long long pre_nq = block_exclusive_scan<long long>(nq_sum, sh, tot_nq);
  long long pre_tc = block_exclusive_scan<long long>(tc_sum, sh, tot_tc);
  long long pre_tri = block_exclusive_scan<long long>(tri_sum, sh, tot_tri);
  for (int s = s0; s < s1; ++s) {
    v.tile_off[s] = (int32_t)pre_nq;
    v.tc_off[s] = pre_tc;
    v.tri_off[s] = (int32_t)pre_tri;
    const int len = min(seq_len_safe(a.cu, s, a.T), a.max_seqlen);
    const long long nq = (len + TILE - 1) / TILE;
    pre_nq += nq;
    pre_tc += nq * nq;
    pre_tri += nq * (nq + 1) / 2;
  }
  if (tid == 0) {
    v.tile_off[a.n] = (int32_t)min(tot_nq, (long long)v.nq_cap);
    v.tc_off[a.n] = tot_tc;
    v.counters[0] = (int32_t)min(tot_nq, (long long)v.nq_cap);
    v.counters[1] = a.n;
    v.counters[2] = 0;
    v.counters[4] = 0;  // pair-forward work counter / done counter
    v.counters[5] = 0;
    *v.pairs = 0ull;
  }
  for (int i = tid; i < 3 * v.hmax; i += nt) v.hist[i] = 0;
  if (err) atomicOr(v.err, err);
}

// ---------------------------------------------------------------- K2
// #{j in [lo, hi) : x[j] <= key} + lo for non-decreasing x (upper bound).
__device__ __forceinline__ int upper_bound_i64(const int64_t* x, int lo, int hi, int64_t key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (x[mid] <= key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int lower_bound_i32(const int32_t* x, int lo, int hi, int32_t key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (x[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) plan_row_kernel(PlanArgs a, PlanView v) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cnt = 0;
  uint32_t err = 0;
  if (i < a.T) {
    const int nreal = (a.n > 0) ? min(max(a.cu[a.n], 0), a.T) : 0;
    if (i >= nreal) {
      v.kv_end[i] = i;
      v.row_seq[i] = -1;
      v.row_pp[i] = 0;
      v.rope_dt[i] = make_float2(0.f, 0.f);
    } else {
      // sequence of row i: largest s with cu[s] <= i
      int lo = 0, hi = a.n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.cu[mid] <= i)
          lo = mid;
        else
          hi = mid - 1;
      }
      const int s = lo;
      const int sa = min(max(a.cu[s], 0), i);
      const int se = min(max(a.cu[s + 1], i + 1), a.T);
      const int m = se - sa;
      int nc = a.ncand ? a.ncand[s] : 0;
      nc = min(max(nc, 0), m);
      const int L = m - nc;
      const int li = i - sa;
      const int64_t ti = a.t[i];
      {  // the row's time rebased to its sequence start, split exactly into two floats (RoPE; R21)
        const long long dt = (long long)(ti - a.t[sa]);
        const float hi = (float)dt;
        v.rope_dt[i] = make_float2(hi, (float)(dt - (long long)hi));
      }
      if (li > 0 && a.t[i - 1] > ti) err |= ERRBIT_ORDER;
      if (a.sess && li > 0 && a.sess[i - 1] > a.sess[i]) err |= ERRBIT_ORDER;
      int e;
      uint8_t pp = 0;
      if (li < L) {  // context query (Eq. 6)
        e = li;
        if (a.mask_flags & 1) e = min(e, upper_bound_i64(a.t, sa, i, ti - a.delta_ctx) - sa);
        if ((a.mask_flags & 2) && a.sess) e = min(e, lower_bound_i32(a.sess, sa, i, a.sess[i]) - sa);
        if (a.nstatic) e = max(e, min(li, max(a.nstatic[s], 0)));
        if ((a.mask_flags & 4) && a.flags && li >= 1 && (a.flags[i] & 1)) pp = 1;
      } else {  // candidate query: context keys with t_j <= t_i - Delta_cand, plus itself
        e = min(L, upper_bound_i64(a.t, sa, sa + L, ti - a.delta_cand) - sa);
      }
      e = max(e, 0);
      v.kv_end[i] = sa + e;
      v.row_seq[i] = s;
      v.row_pp[i] = pp;
      cnt = (unsigned long long)e + 1ull + ((pp && (li - 1) >= e) ? 1ull : 0ull);
    }
  }
  // warp reduce the pair count, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(v.pairs, cnt);
  if (err) atomicOr(v.err, err);
}

// ---------------------------------------------------------------- K3
__device__ __forceinline__ int tile_seq(const PlanView& v, int n, int g) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (v.tile_off[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// one warp per tile: the 128 rows' visible-prefix ends are reduced across the lanes
__global__ void __launch_bounds__(128) plan_tile_kernel(PlanArgs a, PlanView v) {
  pdl_trigger();
  pdl_wait();
  const int g = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int nq_total = v.counters[0];
  if (g >= nq_total) return;
  const int s = tile_seq(v, a.n, g);
  const int qt = g - v.tile_off[s];
  const int sa = a.cu[s];
  const int len = min(seq_len_safe(a.cu, s, a.T), a.max_seqlen);
  const int nq_s = (len + TILE - 1) / TILE;
  const int r0 = sa + qt * TILE, r1 = min(sa + len, r0 + TILE);
  int emax = 0, emin = 1 << 30;
  for (int r = r0 + lane; r < r1; r += 32) {
    const int e = v.kv_end[r] - sa;
    emax = max(emax, e);
    emin = min(emin, e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
  }
  if (lane != 0) return;
  const int nf = min((emax + TILE - 1) / TILE, qt + 1);
  const int kt_pp = (qt > 0 && v.row_pp[r0]) ? qt - 1 : qt;
  const int kt2 = max(nf, kt_pp);
  QTileInfo info;
  info.seq = s;
  info.qt = qt;
  info.nf = nf;
  info.kt2 = kt2;
  info.emin = (r1 > r0) ? emin : 0;
  info.rows = r1 - r0;
  info.pad0 = info.pad1 = 0;
  v.qinfo[g] = info;
  const int cost_f = min(nf + (qt + 1 - kt2), v.hmax - 1);
  const int lb = min(nq_s, v.hmax - 1);
  atomicAdd(&v.hist[cost_f], 1);
  atomicAdd(&v.hist[v.hmax + lb], 1);                        // tiles per sequence-length bucket
  if (qt == 0) v.seq_rank[s] = atomicAdd(&v.hist[2 * v.hmax + lb], 1);  // the sequence's rank in it
}

// ---------------------------------------------------------------- K4 / K5
// Exclusive scan of the cost histograms in DESCENDING cost order (LPT: most expensive first).
__global__ void __launch_bounds__(1024) plan_order_kernel(PlanView v) {
  pdl_trigger();
  pdl_wait();
  __shared__ long long sh[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  // which = 2: the per-bucket sequence counts (rank counters, no longer needed after plan_tile) become
  // the bucket's first forward pair: sequences of b tiles contribute ceil(b / 2) pairs each
  for (int which = 0; which < 3; ++which) {
    int* h = v.hist + which * v.hmax;
    const int per = (v.hmax + nt - 1) / nt;
    auto wgt = [&](int b) { return which == 2 ? (b + 1) / 2 : 1; };
    // thread t owns reversed positions [t*per, (t+1)*per): cost c = hmax-1-pos
    long long local = 0;
    for (int q = tid * per; q < min((tid + 1) * per, v.hmax); ++q)
      local += (long long)h[v.hmax - 1 - q] * wgt(v.hmax - 1 - q);
    long long total;
    long long pre = block_exclusive_scan<long long>(local, sh, total);
    if (which == 2 && tid == 0) v.counters[2] = (int)total;
    int vals[64];
    const int cnt = max(0, min((tid + 1) * per, v.hmax) - tid * per);
    for (int q = 0; q < cnt && q < 64; ++q) vals[q] = h[v.hmax - 1 - (tid * per + q)] * wgt(v.hmax - 1 - (tid * per + q));
    __syncthreads();
    for (int q = 0; q < cnt && q < 64; ++q) {
      h[v.hmax - 1 - (tid * per + q)] = (int)pre;
      pre += vals[q];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) plan_scatter_kernel(PlanArgs a, PlanView v) {
  pdl_trigger();
  pdl_wait();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq_total = v.counters[0];
  if (g >= nq_total) return;
  const QTileInfo info = v.qinfo[g];
  const int len = min(seq_len_safe(a.cu, info.seq, a.T), a.max_seqlen);
  const int nq_s = (len + TILE - 1) / TILE;
  const int cost_f = min(info.nf + (info.qt + 1 - info.kt2), v.hmax - 1);
  const int lb = min(nq_s, v.hmax - 1);
  (void)cost_f;
  // sequence-major orders: bucket start (longest sequences first) + rank * tiles + tile, q-tiles
  // in descending order (the last q-tile sees the most keys), k-tiles ascending (k-tile 0 is seen
  // by every q-tile): the CTAs running together work on one sequence, whose K / V (forward) or
  // Q / dO (backward) tiles then come from L2
  const int seq0 = v.hist[v.hmax + lb] + v.seq_rank[info.seq] * lb;
  if (seq0 + lb <= v.nq_cap) {
    v.fwd_order[seq0 + (lb - 1 - info.qt)] = g;
    v.bwd_order[seq0 + info.qt] = g;
  }
  // forward pairs: the sequence's q-tiles from the last down, two at a time (a lone tile 0 at the end)
  const int rel = lb - 1 - info.qt;
  if (rel >= 0 && (rel & 1) == 0) {
    const int pi = v.hist[2 * v.hmax + lb] + v.seq_rank[info.seq] * ((lb + 1) / 2) + rel / 2;
    if (pi < v.nq_cap) v.pair_list[pi] = g;
  }
  // visit list of g as a k-tile (transpose of the forward visit rule): q-tiles qt >= kt of the
  // sequence with kt < nf(qt) or kt2(qt) <= kt <= qt; slots [base, base + nq_s - kt) of the
  // sequence's triangle
  const int kt = info.qt, tile0 = g - kt;
  const int base = v.tri_off[info.seq] + kt * nq_s - kt * (kt - 1) / 2;
  int n = 0;
  for (int qt = kt; qt < nq_s && tile0 + qt < nq_total; ++qt) {
    const QTileInfo qi = v.qinfo[tile0 + qt];
    if (kt < qi.nf || (kt >= qi.kt2 && kt <= qi.qt)) {
      const bool full = qi.rows == TILE && qi.emin >= (kt + 1) * TILE;
      if (base + n < v.list_cap) v.bwd_list[base + n] = qt | (full ? (1 << 30) : 0);  // (invalid offsets latch E_OFFSETS)
      ++n;
    }
  }
  v.bwd_off[g] = base;
  v.bwd_cnt[g] = base + n <= v.list_cap ? n : 0;
}

cudaError_t plan_launch(const PlanArgs& a, const PlanView& v, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 5);
  launch_pdl(plan_seq_kernel, dim3(1), dim3(1024), 0, st, a, v);
  if (a.T > 0) launch_pdl(plan_row_kernel, dim3((a.T + 255) / 256), dim3(256), 0, st, a, v);
  const int nb = (v.nq_cap + 127) / 128;
  if (nb > 0) {
    launch_pdl(plan_tile_kernel, dim3((v.nq_cap + 3) / 4), dim3(128), 0, st, a, v);
    launch_pdl(plan_order_kernel, dim3(1), dim3(1024), 0, st, v);
    launch_pdl(plan_scatter_kernel, dim3(nb), dim3(128), 0, st, a, v);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- export (test hook)
__global__ void __launch_bounds__(128) plan_export_kernel(PlanArgs a, PlanView v, int8_t* tc_out, int64_t tc_cap) {
  pdl_trigger();
  pdl_wait();
  const int g = blockIdx.x;
  const int nq_total = v.counters[0];
  if (g >= nq_total) return;
  const QTileInfo info = v.qinfo[g];
  const int s = info.seq, qt = info.qt;
  const int sa = a.cu[s];
  const int len = min(seq_len_safe(a.cu, s, a.T), a.max_seqlen);
  const int nq_s = (len + TILE - 1) / TILE;
  const int r0 = sa + qt * TILE, r1 = min(sa + len, r0 + TILE);
  for (int kt = threadIdx.x; kt < nq_s; kt += blockDim.x) {
    const int k0 = sa + kt * TILE, k1 = min(sa + len, k0 + TILE);
    long long allowed = 0;
    for (int r = r0; r < r1; ++r) {
      const int e = v.kv_end[r];
      long long c = max(0, min(k1, e) - k0);          // prefix part inside [k0, k1)
      if (r >= k0 && r < k1 && r >= e) c += 1;         // diagonal
      if (v.row_pp[r] && (r - 1) >= k0 && (r - 1) < k1 && (r - 1) >= e) c += 1;
      allowed += c;
    }
    const long long cells = (long long)(r1 - r0) * (k1 - k0);
    const int8_t cls = allowed == 0 ? 0 : (allowed == cells ? 2 : 1);
    const long long idx = v.tc_off[s] + (long long)qt * nq_s + kt;
    if (idx < tc_cap) tc_out[idx] = cls;
  }
}

__global__ void copy_kv_end_kernel(const int32_t* src, int32_t* dst, int T, const unsigned long long* pairs,
                                   int64_t* pairs_out) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < T) dst[i] = src[i];
  if (i == 0 && pairs_out) *pairs_out = (int64_t)*pairs;
}

cudaError_t plan_export_launch(const PlanArgs& a, const PlanView& v, int32_t* kv_end_out, int8_t* tc_out,
                               int64_t tc_cap, int64_t* pairs_out, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 2);
  if (kv_end_out || pairs_out)
    launch_pdl(copy_kv_end_kernel, dim3((a.T + 255) / 256 + 1), dim3(256), 0, st, v.kv_end, kv_end_out ? kv_end_out : v.kv_end,
                                                              kv_end_out ? a.T : 0, v.pairs, pairs_out);
  if (tc_out && v.nq_cap > 0) launch_pdl(plan_export_kernel, dim3(v.nq_cap), dim3(128), 0, st, a, v, tc_out, tc_cap);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- A0 chunk
__global__ void __launch_bounds__(1024) chunk_kernel(const int32_t* cu_in, int n, int L, int32_t* cu_out, int cap,
                                                      int32_t* n_out, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  __shared__ long long sh[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int s0 = min(tid * per, n), s1 = min(s0 + per, n);
  long long local = 0;
  uint32_t e = 0;
  for (int s = s0; s < s1; ++s) {
    const int len = cu_in[s + 1] - cu_in[s];
    if (len <= 0) e |= ERRBIT_OFFSETS;
    local += len > 0 ? (len + L - 1) / L : 0;
  }
  long long total;
  long long pre = block_exclusive_scan<long long>(local, sh, total);
  if (total + 1 > cap) e |= ERRBIT_CAPACITY;
  for (int s = s0; s < s1; ++s) {
    const int a = cu_in[s], b = cu_in[s + 1];
    const int len = b - a;
    if (len <= 0) continue;
    const int nch = (len + L - 1) / L;
    for (int c = 0; c < nch; ++c) {
      // chunk c in buffer order: c = 0 is the oldest (possibly short) chunk; the newest
      // chunk [b - L, b) is full.
      const long long pos = pre + c;
      const int start = (c == 0) ? a : b - (nch - c) * L;
      if (pos < cap) cu_out[pos] = start;
    }
    pre += nch;
  }
  if (tid == 0) {
    if (total < cap) cu_out[total] = (n > 0) ? cu_in[n] : 0;
    *n_out = (int32_t)total;
  }
  if (e) atomicOr(err, e);
}

cudaError_t chunk_launch(const int32_t* cu_in, int32_t n_in, int32_t L, int32_t* cu_out, int32_t cap, int32_t* n_out,
                         uint32_t* err, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 1);
  launch_pdl(chunk_kernel, dim3(1), dim3(1024), 0, st, cu_in, n_in, L, cu_out, cap, n_out, err);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- A13 pack
__global__ void __launch_bounds__(1024) pack_offsets_kernel(const int32_t* lens, int B, int budget, int32_t* cu_out,
                                                             int32_t* n_packed, uint32_t* err) {
  pdl_trigger();
  pdl_wait();
  __shared__ long long sh[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (B + nt - 1) / nt;
  const int s0 = min(tid * per, B), s1 = min(s0 + per, B);
  long long local = 0;
  uint32_t e = 0;
  for (int s = s0; s < s1; ++s) {
    if (lens[s] <= 0) e |= ERRBIT_OFFSETS;
    local += max(lens[s], 0);
  }
  long long total;
  long long pre = block_exclusive_scan<long long>(local, sh, total);
  // greedy arrival order: sequences are taken while the running total fits the budget
  __shared__ int first_over;
  if (tid == 0) first_over = B;
  __syncthreads();
  for (int s = s0; s < s1; ++s) {
    pre += max(lens[s], 0);
    if (pre > budget) atomicMin(&first_over, s);
  }
  __syncthreads();
  const int k = first_over;
  pre = block_exclusive_scan<long long>(local, sh, total);
  for (int s = s0; s < s1; ++s) {
    cu_out[s] = (int32_t)min(pre, (long long)budget);
    pre += max(lens[s], 0);
  }
  __syncthreads();
  // entries past n_packed repeat the packed total
  if (tid == 0) {
    long long tot = 0;
    n_packed[0] = k;
    (void)tot;
  }
  __syncthreads();
  const int packed_total = (k > 0) ? cu_out[k - 1] + lens[k - 1] : 0;
  for (int s = tid; s <= B; s += nt)
    if (s >= k) cu_out[s] = packed_total;
  if (B > 0 && k == 0 && tid == 0) e |= ERRBIT_TOO_LONG;
  if (e) atomicOr(err, e);
}

__global__ void __launch_bounds__(256) pack_rows_kernel(const uint8_t* src, const int64_t* src_row, const int32_t* cu,
                                                         const int32_t* n_packed, int row_bytes, int budget, const int64_t* tp,
                                                         const int32_t* sp, uint8_t* packed, int64_t* t_out,
                                                         int32_t* s_out) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x / 32;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= budget) return;
  const int k = *n_packed;
  const int total = cu[k];
  uint4* dst = reinterpret_cast<uint4*>(packed + (size_t)r * row_bytes);
  const int nvec = row_bytes / 16;
  if (r < total) {
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cu[mid] <= r)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int s = lo, j = r - cu[s];
    const size_t sr = src_row ? (size_t)src_row[s] + j : (size_t)r;  // contiguous: packed row == source row
    const uint4* sv = reinterpret_cast<const uint4*>(src + sr * row_bytes);
    for (int c = lane; c < nvec; c += 32) dst[c] = sv[c];
    if (lane == 0) {
      if (t_out) t_out[r] = tp ? tp[sr] : 0;
      if (s_out) s_out[r] = sp ? sp[sr] : 0;
    }
  } else {
    for (int c = lane; c < nvec; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
    if (lane == 0) {
      if (t_out) t_out[r] = 0;
      if (s_out) s_out[r] = 0;
    }
  }
}

// Metadata-only pack (src == packed == null): the per-row timestamps / session ids, one thread per
// row, so the row data can be moved by a second call on another stream.
__global__ void __launch_bounds__(256) pack_meta_kernel(const int64_t* src_row, const int32_t* cu,
                                                         const int32_t* n_packed, int budget, const int64_t* tp,
                                                         const int32_t* sp, int64_t* t_out, int32_t* s_out) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= budget) return;
  const int k = *n_packed;
  if (r < cu[k]) {
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cu[mid] <= r)
        lo = mid;
      else
        hi = mid - 1;
    }
    const size_t sr = src_row ? (size_t)src_row[lo] + (r - cu[lo]) : (size_t)r;
    if (t_out) t_out[r] = tp ? tp[sr] : 0;
    if (s_out) s_out[r] = sp ? sp[sr] : 0;
  } else {
    if (t_out) t_out[r] = 0;
    if (s_out) s_out[r] = 0;
  }
}

cudaError_t pack_launch(const void* src, const int64_t* src_row, const int32_t* lens, int32_t B, int32_t d,
                        int32_t budget, const int64_t* tp, const int32_t* sp, void* packed, int64_t* t_out,
                        int32_t* s_out, int32_t* cu_out, int32_t* n_packed, uint32_t* err, cudaStream_t st) {
  ProfScope ps(PROF_OTHER, st, 2);
  launch_pdl(pack_offsets_kernel, dim3(1), dim3(1024), 0, st, lens, B, budget, cu_out, n_packed, err);
  if (!packed) {
    launch_pdl(pack_meta_kernel, dim3((budget + 255) / 256), dim3(256), 0, st, src_row, cu_out, n_packed, budget, tp,
               sp, t_out, s_out);
    return cudaGetLastError();
  }
  const int rows_per_block = 8;
  launch_pdl(pack_rows_kernel, dim3((budget + rows_per_block - 1) / rows_per_block), dim3(256), 0, st, reinterpret_cast<const uint8_t*>(src), src_row, cu_out, n_packed, d * 2, budget, tp, sp,
      reinterpret_cast<uint8_t*>(packed), t_out, s_out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- zero pad rows [cu[n], T)
struct PadBufs {
  uint8_t* buf[4];
};
// blockIdx.y selects the buffer: up to 4 [T, row_bytes] buffers in one launch
__global__ void zero_pad_rows_kernel(PadBufs b, int row_bytes, int T, const int32_t* cu, int n) {
  pdl_trigger();
  pdl_wait();
  uint8_t* buf = b.buf[blockIdx.y];
  const int nreal = n > 0 ? min(max(cu[n], 0), T) : 0;
  const size_t begin = (size_t)nreal * row_bytes, end = (size_t)T * row_bytes;
  for (size_t i = begin + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < end;
       i += (size_t)gridDim.x * blockDim.x * 16)
    *reinterpret_cast<uint4*>(buf + i) = make_uint4(0, 0, 0, 0);
}

cudaError_t zero_pad_rows_launch(void* buf, int32_t row_bytes, int32_t T, const int32_t* cu, int32_t n,
                                 cudaStream_t st) {
  void* one[1] = {buf};
  return zero_pad_rows_multi_launch(one, 1, row_bytes, T, cu, n, st);
}
cudaError_t zero_pad_rows_multi_launch(void* const* bufs, int nbuf, int32_t row_bytes, int32_t T, const int32_t* cu,
                                       int32_t n, cudaStream_t st) {
  if (nbuf < 1 || nbuf > 4) return cudaErrorInvalidValue;
  PadBufs b;
  for (int i = 0; i < 4; ++i) b.buf[i] = reinterpret_cast<uint8_t*>(bufs[i < nbuf ? i : 0]);
  ProfScope ps(PROF_OTHER, st, 1);
  launch_pdl(zero_pad_rows_kernel, dim3(148, nbuf), dim3(256), 0, st, b, row_bytes, T, cu, n);
  return cudaGetLastError();
}

}  // namespace cadet
