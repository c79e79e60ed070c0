// Launchers of the elementwise / reduction kernels (misc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include "../../include/cadet.h"

namespace cadet {
// Timestamp RoPE evaluated on the fly (no (cos, sin) table in HBM): alpha_i = (t_row -
// t_(sequence start)) theta_i, theta_i = (phi_min / dt_max) base^(2i / hd).  theta_i is
// evaluated once per plan in fp64 and kept as a float pair (hi + lo, PlanView::theta); the product with
// the int64 rebased time (also split hi + lo) and the mod-2 pi reduction run in compensated fp32 (an FMA
// two-product and a two-constant 2 pi), ~3e-7 rad absolute for |alpha| <= 1e4 rad, then MUFU sincos.
// on = 0: no RoPE (ablation).
struct RopeOTF {
  const float2* dt;        // [T] the plan's rebased row times (hi, lo): t_row - t_(sequence start)
  const float2* theta;     // [hd / 2] (hi, lo)
  int32_t on;
};
cudaError_t rope_apply_launch(const void* in, void* out, int T, int d, int hd, const RopeOTF& rp, cudaStream_t st);
// A4 elementwise half: Qr = RoPE(Q * sigma(Z_q)), Kr = RoPE(K * sigma(Z_k)) (Z stored by the gate GEMMs)
cudaError_t gate_rope_fwd_launch(const void* Q, const void* K, const void* Gq, const void* Gk, const RopeOTF& rp,
                                 void* Qr, void* Kr, int T, int d, int hd, cudaStream_t st, float* tapQ = nullptr,
                                 float* tapK = nullptr);
// both sides (Q and K) in one launch: arrays of nsides (<= 2) pointers
cudaError_t rope_gate_bwd_launch2(const void* const* dr, const void* const* Xq, const void* const* Z,
                                  void* const* out_u, void* const* out_r, int nsides, int dr_f32, int r_bf16, int T,
                                  int d, int hd, const RopeOTF& rp, cudaStream_t st, float* const* tap_u = nullptr,
                                  float* const* tap_r = nullptr);
cudaError_t rope_gate_bwd_launch(const void* dr, int dr_f32, const void* Xq, const void* Z, void* out_u, void* out_r,
                                 int r_bf16, int T, int d, int hd, const RopeOTF& rp, cudaStream_t st);
// to_f16: the gathered rows are written as fp16 (the towers' GEMM operand)
cudaError_t gather_rows_launch(const void* H, const int32_t* rows, int n, int T, int d, void* out, uint32_t* err,
                               cudaStream_t st, int to_f16 = 0);
cudaError_t bf16_to_f16_launch(const void* src, void* dst, size_t n, cudaStream_t st);
cudaError_t head_init_launch(float* logits, const float* b2, int n, int K, cudaStream_t st);
cudaError_t head_dz_launch(const float* logits, const int32_t* bucket, const float* label, int n, int K, float* dz,
                           float* loss_sum, float* db2, uint32_t* err, cudaStream_t st);
cudaError_t head_dhid_launch(const void* pre, const float* dz, const int32_t* bucket, const float* w2, int n, int K,
                             int dh, void* dhid, void* dhid_lo, float* db1, float* dw2, cudaStream_t st);
// NEXT-2 (loss.cu): tower backward from a full dz [n, K] (dhid hi + lo, db1, dw2, db2)
cudaError_t head_dhid_full_launch(const void* pre, const float* dz, const float* w2, int n, int K, int dh, void* dhid,
                                  void* dhid_lo, float* db1, float* dw2, float* db2, cudaStream_t st);
cudaError_t add_bf16_launch(const void* a, const void* b, void* out, size_t n, cudaStream_t st);
// Zero up to 8 buffers in ONE launch (instead of one memset node each): spans of `bytes` at `ptr`
// (null entries skipped; 16-byte stores when ptr is 16-byte aligned, bytewise otherwise).
struct ZeroSpan {
  void* ptr;
  size_t bytes;
};
cudaError_t zero_many_launch(const ZeroSpan* spans, int n, cudaStream_t st);
// NEXT-3 embeddings (embed.cu)
size_t embed_ws_bytes(const cadet_embed_config* c);
cudaError_t embed_forward_launch(const cadet_embed_config* c, const void* const* tables, const int32_t* ids, int T,
                                 const int32_t* n_valid, void* X, void* ws, cudaStream_t st);
cudaError_t embed_backward_launch(const cadet_embed_config* c, const int32_t* ids, int T, const int32_t* n_valid,
                                  const void* dX, float* const* dtables, void* ws, cudaStream_t st);
struct Bounds {  // context-bucket boundaries (cadet_bucketize), strictly increasing
  int32_t b[32];
  int32_t nb;
};
cudaError_t bucketize_launch(const int32_t* pos, int n, const Bounds& bd, int32_t* out, uint32_t* err,
                             cudaStream_t st);
// out[i] = sum_{s = 0..nsplit-1} slabs[s n + i], in that order (deterministic split-K reduction)
cudaError_t slab_reduce_launch(const float* slabs, int nsplit, size_t n, float* out, cudaStream_t st);
}  // namespace cadet
