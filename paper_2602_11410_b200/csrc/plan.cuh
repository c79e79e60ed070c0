// Plan data carved from the workspace.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace cadet {

constexpr int TILE = 128;

struct QTileInfo {  // one per (sequence, 128-row tile), anchored at the sequence start
  int32_t seq;      // sequence index
  int32_t qt;       // tile index inside the sequence
  int32_t nf;       // front k-tiles [0, nf) are visited (prefix region, max_i kv_end)
  int32_t kt2;      // then tiles [kt2, qt] (diagonal, and qt-1 for a PAIR_PREV first row); kt2 >= nf
  int32_t emin;     // min over the tile's rows of the local visible-prefix end (k-tiles below emin/128 are FULL)
  int32_t rows;     // rows of this tile inside the sequence (<= 128)
  int32_t pad0, pad1;
};

struct PlanView {   // device pointers into the workspace
  uint32_t* err;      // [1] latched error bits
  int32_t* counters;  // [0] = nq_total, [1] = n (for checking)
  unsigned long long* pairs;  // [1]
  int32_t* kv_end;    // [T]
  int32_t* row_seq;   // [T] (-1 for pad rows)
  uint8_t* row_pp;    // [T] PAIR_PREV bit resolved for the row
  int32_t* tile_off;  // [n+1] prefix sum of nq_s
  int64_t* tc_off;    // [n+1] prefix sum of nq_s^2 (export)
  QTileInfo* qinfo;   // [nq_cap]
  int32_t* fwd_order; // [nq_cap] q-tiles, sequence-major (see bwd_order), each sequence's q-tiles descending
  int32_t* bwd_order; // [nq_cap] k-tiles, sequence-major: sequences by descending length, each sequence's
                      // k-tiles in ascending order (heaviest first), so the CTAs running together share
                      // one sequence's Q / dO tiles in L2
  int32_t* hist;      // [3 * hmax] histograms / cursors (fwd cost, bwd sequence length, rank counters)
  int32_t* tri_off;   // [n+1] prefix sum of nq_s (nq_s + 1) / 2 (visit-list slots per sequence)
  int32_t* bwd_off;   // [nq_cap] start of k-tile g's visit list in bwd_list
  int32_t* bwd_cnt;   // [nq_cap] its length
  int32_t* bwd_list;  // [list_cap] q-tiles visiting k-tile g: qt | FULL << 30 (all cells visible)
  int32_t* seq_rank;  // [n] rank of a sequence among those with the same tile count (bwd order)
  int32_t* pair_list; // [nq_cap] forward work items: q-tile g (descending inside its sequence) paired with
                      // tile g - 1 of the same sequence when qt(g) >= 1; sequence-major like fwd_order.
                      // counters[2] = number of pairs; counters[4..5] = the pair kernel's dynamic work
                      // counter and done counter (zeroed by the plan, reset by the kernel's last CTA)
  float2* theta;      // [64] RoPE theta_i as (hi, lo) floats, i < head_dim / 2
  float2* rope_dt;    // [T] t_row - t_(sequence start) as exact (hi, lo) floats (0 for pad rows)
  int32_t nq_cap, hmax, list_cap;
};

struct PlanArgs {
  int32_t n, T, max_seqlen, mask_flags;
  int64_t delta_ctx, delta_cand;
  const int32_t* cu;
  const int64_t* t;
  const int32_t* sess;
  const int32_t* ncand;
  const int32_t* nstatic;
  const uint8_t* flags;
  // timestamp RoPE frequencies theta_i = (phi_min / dt_max) base^(2i / hd), written by the
  // plan as float hi + lo pairs for the kernels that rotate (angles evaluated on the fly)
  double rope_phi_min, rope_dt_max, rope_base;
  int32_t head_dim;
};

size_t plan_bytes(int32_t n, int32_t T, int32_t max_seqlen);
PlanView plan_carve(void* ws, int32_t n, int32_t T, int32_t max_seqlen);
cudaError_t plan_launch(const PlanArgs& a, const PlanView& v, cudaStream_t st);
cudaError_t plan_export_launch(const PlanArgs& a, const PlanView& v, int32_t* kv_end_out, int8_t* tc_out,
                               int64_t tc_cap, int64_t* pairs_out, cudaStream_t st);
cudaError_t chunk_launch(const int32_t* cu_in, int32_t n_in, int32_t L, int32_t* cu_out, int32_t cap,
                         int32_t* n_out, uint32_t* err, cudaStream_t st);
cudaError_t pack_launch(const void* src, const int64_t* src_row, const int32_t* lens, int32_t B, int32_t d,
                        int32_t budget, const int64_t* tp, const int32_t* sp, void* packed, int64_t* t_out,
                        int32_t* s_out, int32_t* cu_out, int32_t* n_packed, uint32_t* err, cudaStream_t st);
cudaError_t zero_pad_rows_launch(void* buf, int32_t row_bytes, int32_t T, const int32_t* cu, int32_t n,
                                 cudaStream_t st);
// the same for up to 4 buffers of equal row size in one launch
cudaError_t zero_pad_rows_multi_launch(void* const* bufs, int nbuf, int32_t row_bytes, int32_t T, const int32_t* cu,
                                       int32_t n, cudaStream_t st);

}  // namespace cadet
