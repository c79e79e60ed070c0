/* cadet.h — C ABI of libcadet: the CADET (arXiv 2602.11410) data-parallel hot path on B200.
 *
 * The hot path is the packed (jagged) self-attention layer over user interaction
 * sequences with timestamp RoPE, the session/delay + candidate mask, the
 * representation- and interaction-level sigmoid self-gates, and the
 * context-conditioned multi-tower heads.
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * CONVENTIONS (apply to every call)
 *  - Every pointer is a DEVICE pointer unless its name ends in _h (host).
 *  - Every call enqueues work on `stream` and returns without synchronising; no call
 *    allocates device memory.  The caller owns all buffers; scratch is passed as
 *    `ws` (workspace) sized by the *_bytes queries, 256-byte aligned.
 *  - Matrices are row-major.  Projections are row-vector: y = x . W with
 *    W[d_in][d_out].  bf16 tensors are passed as void* (uint16 storage).
 *  - Packed batch (Fig. 4): tokens of n sequences back to back in a buffer of
 *    exactly T rows; sequence s owns rows [cu_seqlens[s], cu_seqlens[s+1]); rows
 *    [cu_seqlens[n], T) are padding.  Pad rows produce 0 outputs and 0 gradients and
 *    never attend or get attended.
 *  - Return codes only; no exceptions cross the ABI.  cadet_last_error() returns a
 *    thread-local message for the last non-OK status.  Host-detected errors (null
 *    pointers, unsupported shapes, small workspace) return synchronously.
 *    Device-detected input errors (offsets, ordering, n_candidates, bucket range,
 *    NaN/Inf) are latched into the workspace error word and returned by the next
 *    cadet_poll(ws); kernels stay memory-safe on invalid input (indices clamped,
 *    invalid sequences skipped) and results are unspecified until cadet_poll
 *    returns CADET_OK.
 *  - Stateless and reentrant: concurrent calls on different streams with different
 *    workspaces are allowed.
 */
#ifndef CADET_H
#define CADET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CADET_ABI_VERSION 1

typedef struct CUstream_st* cadet_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  CADET_OK = 0,
  CADET_E_ARG = 1,         /* null pointer / bad shape: d % H, head_dim not in {32,64,88,96,128}, H > 128, d % 32 ("dimension error") */
  CADET_E_OFFSETS = 2,     /* cu_seqlens[0] != 0, empty or decreasing sequence, cu[n] > T          (device) */
  CADET_E_ORDER = 3,       /* timestamps or session ids decrease inside a sequence ("ordering error") (device) */
  CADET_E_TOO_LONG = 4,    /* a sequence longer than max_seqlen or the budget: chunk first          (device) */
  CADET_E_CAND = 5,        /* n_candidates[s] > length of s                                                (device) */
  CADET_E_BUCKET = 6,      /* bucket outside [0, K) ("routing error")                                (device) */
  CADET_E_NONFINITE = 7,   /* NaN/Inf in a loss (fail-fast numerics)                                  (device) */
  CADET_E_WORKSPACE = 8,   /* workspace / capacity too small                                                         */
  CADET_E_UNSUPPORTED = 9, /* valid but not implemented in this build                                                  */
  CADET_E_CUDA = 10        /* a CUDA runtime error; see cadet_last_error()                                          */
} cadet_status;

enum { CADET_BF16 = 0, CADET_FP32 = 1 };

/* Mask rule bits (Fig. 3). */
enum {
  CADET_MASK_TIME = 1,     /* context query i sees j < i only if t_j <= t_i - delta_delay_ms (Eq. 6; tie allowed) */
  CADET_MASK_SESSION = 2,  /* context query i sees j < i only if session_id_j < session_id_i (opt-in reading R10)  */
  CADET_MASK_PAIR_PREV = 4 /* context query i also sees i-1 when token_flags[i] & 1 (SPEC S:310 exception, R12)     */
};
/* Always: the diagonal is visible (Fig. 3 "preserved diagonal", R8); candidate queries (the last
 * n_candidates[s] rows of s) see context keys j with t_j <= t_i - delta_cand_ms and themselves only
 * (P:285); j < n_static[s] is visible to every context query (R13). */

typedef struct {
  int32_t d_model;   /* d, multiple of 32 */
  int32_t n_heads;   /* H <= 128; head_dim = d / H must be one of {32, 64, 88, 96, 128} (else CADET_E_ARG) */
  int32_t head_dim;  /* must equal d_model / n_heads */
  int32_t dtype;     /* CADET_BF16: bf16 tensors and weights, fp32 accumulation (the product path).
                        CADET_FP32: the parity mode (SURVEY 8(c) ii, north star "1e-4 for an fp32 mode"): every
                        tensor / weight argument of the layer and core calls is fp32 (saved and workspace sizes
                        follow), GEMMs are 3xTF32 on the tensor cores, gates / RoPE / attention run in fp32
                        arithmetic; out_f32 and the two-pass dS workspace do not apply. */
  int32_t mask_flags;
  int32_t out_f32;   /* core calls: 1 = write O / dQr / dKr / dV as fp32 (parity protocol, SURVEY 8(c) iii).
                        layer calls: 1 = ALSO write every stage's fp32 value before its bf16 rounding into the
                        tap region of ws (cadet_attn_workspace_bytes grows by CADET_N_TAPS * T * d * 4 B;
                        pointers from cadet_attn_stage_views); the bf16 results are unchanged.  The attention
                        taps (O, dQr, dKr, dV) come from a second run of the same deterministic kernels with
                        fp32 stores.  Parity / debugging only (about 2x the layer's time). */
  int32_t use_rope, use_rep_gate, use_int_gate, use_out_proj; /* ablation switches (Table 1) */
  int32_t deterministic; /* 0: split-K weight gradients and D = rowsum(dO * O) accumulate with fp32 atomics (order
                            not fixed).  1 (bf16 only): bit-reproducible layer backward -- each split-K partial
                            of a weight gradient goes to its own fp32 slab in ws (cadet_attn_workspace_bytes
                            grows by 3 * splits * d^2 * 4 B) and a reduction sums the slabs in split order; D
                            comes from the fixed-order preprocess kernel.  The attention kernels, the mask plan
                            and every forward kernel are atomic-free in both modes (P:569 reproducibility). */
  int32_t plan_ready;    /* 0 = plan inside the call; 1 (or 2, kept for compatibility) = ws already holds
                            cadet_mask_plan's plan for this batch (same ws, same batch): the layer/core calls skip
                            re-planning (one plan per step for all layers).  RoPE angles are evaluated on the fly
                            from the int64 timestamps by the kernels that rotate: no (cos, sin) table in HBM. */
  int64_t delta_delay_ms;       /* Delta for context queries, Eq. 6; default 3,600,000 */
  int64_t delta_cand_ms;        /* Delta for candidate queries; default 0 (R11) */
  int64_t rope_delta_t_max_ms;  /* Delta t_max; default 31,536,000,000 = 1 year (R6) */
  double rope_phi_min;          /* default 1e-4 */
  double rope_base;             /* default 600000 */
} cadet_attn_config;

typedef struct {
  int32_t n_seqs;       /* n (host scalar) */
  int32_t total_tokens; /* T = budget rows of every [T, ...] buffer (host scalar) */
  int32_t max_seqlen;   /* upper bound on any sequence length (host scalar) */
  int32_t reserved0;
  const int32_t* cu_seqlens;    /* [n+1] */
  const int64_t* timestamps_ms; /* [T] Unix ms; non-decreasing within a sequence */
  const int32_t* session_ids;   /* [T] or NULL (required with CADET_MASK_SESSION); non-decreasing within a sequence */
  const int32_t* n_candidates;  /* [n] or NULL: the last n_candidates[s] tokens of s are candidates */
  const int32_t* n_static;      /* [n] or NULL: always-visible static prefix length (R13) */
  const uint8_t* token_flags;   /* [T] or NULL: bit0 = may see token i-1 under CADET_MASK_PAIR_PREV */
} cadet_batch;

/* Seven [d, d] bf16 matrices (Eqs. 3-5): rep gate, Q, K, V, Q gate, K gate, output. */
typedef struct {
  const void *W_xg, *W_q, *W_k, *W_v, *W_qg, *W_kg, *W_o;
} cadet_attn_weights;
/* fp32 [d, d] gradients, OVERWRITTEN (not accumulated) by cadet_attn_backward. */
typedef struct {
  float *dW_xg, *dW_q, *dW_k, *dW_v, *dW_qg, *dW_kg, *dW_o;
} cadet_attn_grads;

/* Context-conditioned towers (Eq. 8; R14): z_k = w2_k . ReLU(h W1_k + b1_k) + b2_k.
 * W1 is stored as ONE [d, K*dh] bf16 matrix whose columns [k*dh, (k+1)*dh) are tower k. */
typedef struct {
  int32_t K;        /* towers (K = 2 at P:624) */
  int32_t d_model;
  int32_t d_hidden; /* dh >= 32, multiple of 8, K*dh multiple of 32 (default d/2) */
  int32_t dtype;    /* CADET_BF16 (W1, Hs, dHs, pre bf16) or CADET_FP32 (all fp32, 3xTF32 GEMMs: parity mode) */
  int32_t rows_in_ws; /* backward calls: 1 = ws still holds H[rows] gathered by cadet_heads_forward (same Hs, rows,
                         n, ws), so the gather is skipped; the rows are still bounds-checked by the scatter */
} cadet_head_config;
typedef struct {
  const void* W1;   /* bf16 [d, K*dh] */
  const float* b1;  /* [K*dh] */
  const float* w2;  /* [K*dh] */
  const float* b2;  /* [K] */
} cadet_head_weights;
typedef struct {
  float *dW1 /*[d, K*dh]*/, *db1 /*[K*dh]*/, *dw2 /*[K*dh]*/, *db2 /*[K]*/; /* overwritten */
} cadet_head_grads;

/* ------------------------------------------------------------------ queries */
int32_t cadet_abi_version(void);
const char* cadet_last_error(void);
const char* cadet_status_string(cadet_status s);
void cadet_default_attn_config(cadet_attn_config* cfg_h, int32_t d_model, int32_t n_heads);
void cadet_tile_shape(int32_t* bm_h, int32_t* bn_h); /* 128, 128: the tile of cadet_mask_export's tile classes */

/* Workspace for cadet_mask_plan / the core calls (plan + error word), and for the full layer
 * (plan + backward temporaries).  `saved` holds the forward activations needed by the backward:
 * Zx, X~, Q, K, Zq, Zk, Qr, Kr, V, O (bf16 [T, d] each) and LSE (fp32 [H, T]). */
size_t cadet_plan_workspace_bytes(int32_t n_seqs, int32_t total_tokens);
size_t cadet_attn_workspace_bytes(const cadet_attn_config* cfg_h, int32_t n_seqs, int32_t total_tokens);
size_t cadet_attn_saved_bytes(const cadet_attn_config* cfg_h, int32_t total_tokens);
/* Optional extra layer workspace enabling the two-pass attention backward (A10): with
 * ws_bytes >= cadet_attn_workspace_bytes + cadet_attn_bwd_ds_bytes(max_seqlen = the batch's
 * max_seqlen), cadet_attn_backward stores every visited dS^T tile (bf16, [128 x 128] per tile
 * pair and head) from the dK/dV kernel and forms dQ = dS K from them, instead of a dQ kernel that
 * recomputes S and dP (5 instead of 7 MMAs per tile pair).  Same results up to MMA accumulation
 * order; 0 if the bound overflows. */
size_t cadet_attn_bwd_ds_bytes(const cadet_attn_config* cfg_h, int32_t n_seqs, int32_t total_tokens,
                               int32_t max_seqlen);
size_t cadet_heads_workspace_bytes(const cadet_head_config* h_h, int32_t n_rows);

/* ------------------------------------------------------------------ A1: mask plan
 * Validates the batch and builds, in ws: per row kv_end[i] (exclusive end of the visible
 * off-diagonal prefix, global index), the row -> sequence map, per 128-row tile the visit
 * bounds, and the cost-ordered (LPT) tile work lists.  The mask is never materialised. */
cadet_status cadet_mask_plan(const cadet_attn_config* cfg_h, const cadet_batch* b_h, void* ws, size_t ws_bytes,
                             cadet_stream_t stream);
/* Test hook (bit-exact targets): kv_end [T] int32 (global; pad rows hold kv_end = i); tile_class int8,
 * per sequence a row-major nq_s x nq_s block (nq_s = ceil(len_s/128), tiles anchored at the sequence
 * start), blocks concatenated in sequence order, 0 = SKIP 1 = PARTIAL 2 = FULL; n_pairs [1] int64 =
 * number of allowed (i, j) cells (head-independent).  tile_class_cap = capacity in entries
 * (>= sum nq_s^2; excess entries are not written).  Requires a prior cadet_mask_plan on ws. */
cadet_status cadet_mask_export(const cadet_attn_config* cfg_h, const cadet_batch* b_h, const void* ws,
                               int32_t* kv_end, int8_t* tile_class, int64_t tile_class_cap, int64_t* n_pairs,
                               cadet_stream_t stream);

/* ------------------------------------------------------------------ A5 / A10: attention core (Eq. 7)
 * Qr, Kr, V: bf16 [T, H*hd] (= [T, H, hd]); Qr/Kr already gated and rotated.
 * O: [T, H*hd] bf16 (fp32 if cfg.out_f32); lse: fp32 [H, T] = ln sum_{j visible} exp(Qr_i.Kr_j / sqrt(hd)).
 * Runs cadet_mask_plan internally. */
cadet_status cadet_attn_core_forward(const cadet_attn_config* cfg_h, const cadet_batch* b_h, const void* Qr,
                                     const void* Kr, const void* V, void* O, float* lse, void* ws, size_t ws_bytes,
                                     cadet_stream_t stream);
/* dO: bf16 [T, H*hd]; O must be the bf16 output of the forward.  Outputs: dQr fp32 [T, H*hd]
 * (always fp32: atomically accumulated), dKr and dV [T, H*hd] bf16 (fp32 if cfg.out_f32). */
cadet_status cadet_attn_core_backward(const cadet_attn_config* cfg_h, const cadet_batch* b_h, const void* Qr,
                                      const void* Kr, const void* V, const void* O, const float* lse, const void* dO,
                                      float* dQr, void* dKr, void* dV, void* ws, size_t ws_bytes,
                                      cadet_stream_t stream);

/* ------------------------------------------------------------------ A2-A6: full gated layer forward
 * X: bf16 [T, d].  Y: bf16 [T, d] = O . W_o (+ resid if resid != NULL, bf16 [T, d]).
 * saved: cadet_attn_saved_bytes; consumed by cadet_attn_backward.  Runs cadet_mask_plan. */
cadet_status cadet_attn_forward(const cadet_attn_config* cfg_h, const cadet_batch* b_h, const cadet_attn_weights* w_h,
                                const void* X, void* Y, const void* resid, void* saved, void* ws, size_t ws_bytes,
                                cadet_stream_t stream);
/* A9-A12: dY bf16 [T, d] -> dX bf16 [T, d] (+ dresid, bf16 [T, d], if non-NULL: the residual-path
 * gradient is added, i.e. dX = dresid + dX_attn) and the 7 fp32 weight gradients (overwritten).
 * ws must be the same workspace as the forward's (the plan is reused) or re-planned. */
cadet_status cadet_attn_backward(const cadet_attn_config* cfg_h, const cadet_batch* b_h,
                                 const cadet_attn_weights* w_h, const void* X, const void* saved, const void* dY,
                                 void* dX, const void* dresid, const cadet_attn_grads* g_h, void* ws, size_t ws_bytes,
                                 cadet_stream_t stream);
/* As cadet_attn_backward, and (grad_events non-NULL) records grad_events[i] (a cudaEvent_t, entries
 * may be NULL) on `stream` right after the launch that completes weight-gradient group i:
 * 0 = dW_o, 1 = dW_qg and dW_kg, 2 = dW_q, dW_k and dW_v, 3 = dW_xg (recorded even when an ablation
 * switch removes the group).  A data-parallel caller all-reduces each group as soon as its event
 * fires, overlapping the reduction with the rest of the backward. */
cadet_status cadet_attn_backward_ev(const cadet_attn_config* cfg_h, const cadet_batch* b_h,
                                    const cadet_attn_weights* w_h, const void* X, const void* saved, const void* dY,
                                    void* dX, const void* dresid, const cadet_attn_grads* g_h, void* ws,
                                    size_t ws_bytes, cadet_stream_t stream, void* const* grad_events);

/* ------------------------------------------------------------------ parity views of the layer (SURVEY 8(c) iii)
 * Stage-by-stage parity needs (a) each stage's value before its bf16 storage rounding and (b) the bf16
 * tensors the next stage consumed.  cadet_attn_stage_views fills views_h[CADET_N_VIEWS] (host array of
 * device pointers into ws, the layer workspace of cadet_attn_forward / cadet_attn_backward with the
 * same cfg, n_seqs and T):
 *   [CADET_TAP_*]  fp32 [T, d] taps, written by the layer calls only when cfg.out_f32 = 1 (else NULL);
 *                  ablated stages are not written;
 *   [CADET_WS_*]   bf16 [T, d] backward intermediates (valid after cadet_attn_backward) and D fp32 [H, T].
 * The forward's bf16 stage outputs are in `saved` (Zx, X~, Q, K, Zq, Zk, Qr, Kr, V, O, LSE; see above). */
enum {
  /* forward (A2-A6): Z_x = X W_xg, X~, Q, K, V, Z_q, Z_k, Q_r, K_r, O, Y */
  CADET_TAP_ZX = 0, CADET_TAP_XT, CADET_TAP_Q, CADET_TAP_K, CADET_TAP_V, CADET_TAP_ZQ, CADET_TAP_ZK, CADET_TAP_QR,
  CADET_TAP_KR, CADET_TAP_O, CADET_TAP_Y,
  /* backward (A9-A12): dO = dY W_o^T, dQ_r, dK_r, dV (attention), u_q, r_q, u_k, r_k (A11 elementwise:
     u = R(-a) dQ_r * Q * g (1 - g), r = R(-a) dQ_r * g), dQ = r_q + u_q W_qg^T, dK, u_x, r_x (A12 gate
     backward of dX~), dX */
  CADET_TAP_DO, CADET_TAP_DQR, CADET_TAP_DKR, CADET_TAP_DV, CADET_TAP_UQ, CADET_TAP_RQ, CADET_TAP_UK, CADET_TAP_RK,
  CADET_TAP_DQ, CADET_TAP_DK, CADET_TAP_UX, CADET_TAP_RX, CADET_TAP_DX,
  CADET_N_TAPS,
  /* bf16 backward intermediates in ws, then D = rowsum(dO * O) per head (fp32 [H, T]) */
  CADET_WS_DO = 32, CADET_WS_DQR, CADET_WS_DKR, CADET_WS_DV, CADET_WS_UQ, CADET_WS_RQ, CADET_WS_UK, CADET_WS_RK,
  CADET_WS_DQ, CADET_WS_DK, CADET_WS_UX, CADET_WS_RX, CADET_WS_D,
  CADET_N_VIEWS
};
cadet_status cadet_attn_stage_views(const cadet_attn_config* cfg_h, int32_t n_seqs, int32_t total_tokens, void* ws,
                                    size_t ws_bytes, void** views_h);

/* ------------------------------------------------------------------ A7 / A8: towers + routed loss (Eqs. 8-9)
 * Hs: bf16 [T, d] transformer output; rows: int32 [n] packed row index of each scored token
 * (impression rows in training, candidate rows at serving).  logits: fp32 [n, K].
 * pre_out (nullable): bf16 [n, K*dh] pre-activations kept for the backward. */
cadet_status cadet_heads_forward(const cadet_head_config* h_h, const cadet_head_weights* w_h, const void* Hs,
                                 const int32_t* rows, int32_t n, float* logits, void* pre_out, void* ws,
                                 size_t ws_bytes, cadet_stream_t stream);
/* Routed BCE with logits, summed (Eq. 9, R15): loss = sum_t softplus(z_{k_t}) - y_t z_{k_t};
 * dz_{k_t} = sigma(z_{k_t}) - y_t, other towers 0.  bucket int32 [n] in [0, K) (else
 * CADET_E_BUCKET via cadet_poll), label fp32 [n].  Writes loss_sum[1], dHs (bf16 [T, d], rows not
 * in `rows` set to 0) and the head gradients.  pre must be the forward's pre_out. */
cadet_status cadet_heads_loss_backward(const cadet_head_config* h_h, const cadet_head_weights* w_h, const void* Hs,
                                       const int32_t* rows, int32_t n, int32_t T, const float* logits,
                                       const void* pre, const int32_t* bucket, const float* label, float* loss_sum,
                                       void* dHs, const cadet_head_grads* g_h, void* ws, size_t ws_bytes,
                                       cadet_stream_t stream);

/* ------------------------------------------------------------------ NEXT-2: full loss (Eqs. 10-12)
 * Auxiliary heads (Eq. 10) run through cadet_heads_forward with their own weight set (K = J
 * towers, d_hidden = the aux width, never routed).  One training step:
 *   cadet_routed_logits -> (data parallel: all-gather z and labels over the ranks) ->
 *   cadet_pairwise_loss -> cadet_full_loss_grads -> cadet_heads_backward (towers, accumulate 0)
 *   -> cadet_heads_backward (aux heads, accumulate 1) -> layers backward.
 * Readings: R29 the RankNet term pairs the routed tower logits z_{k_t} of the whole
 * (global) batch, positives y = 1 vs negatives y = 0; R30 aux heads are 2-layer ReLU MLPs; R31 aux
 * losses are BCE with logits or squared error (z - y)^2, summed over impressions like L_ctx. */
typedef struct {
  int32_t J;              /* auxiliary tasks, 0..8 */
  int32_t aux_kind[8];    /* 0 = BCE with logits, 1 = squared error */
  float lambda_ctx, lambda_pair;
  float lambda_aux[8];    /* Eq. 11 weights; defaults 1.0, 0.1 each, 0.1 */
} cadet_loss_config;
void cadet_default_loss_config(cadet_loss_config* lc_h, int32_t J); /* kinds: task 0 BCE, others SE */
/* z_out [n] = logits[i, bucket[i]] (fp32), the logit the pairwise term compares (R29). */
cadet_status cadet_routed_logits(const float* logits, int32_t K, const int32_t* bucket, int32_t n, float* z_out,
                                 cadet_stream_t stream);
/* RankNet (Eq. 12) of this rank's n samples (routed logits z, labels in {0, 1}) against the batch
 * z_all / label_all [n_all] (all ranks' samples, gathered in rank order; pass z / label themselves on
 * one rank).  loss_share[1] = sum over LOCAL positives i and ALL negatives j of
 * softplus(z_j - z_i) / (N+ N-), so the ranks' shares sum to Eq. 12; dz_pair [n] = dL_pair / dz of
 * the local samples (overwritten).  N+, N- are counted on label_all; either empty -> 0.
 * Deterministic (fixed-order reductions).  ws: cadet_pairwise_workspace_bytes(n, n_all). */
size_t cadet_pairwise_workspace_bytes(int32_t n, int32_t n_all);
cadet_status cadet_pairwise_loss(const float* z, const float* label, int32_t n, const float* z_all,
                                 const float* label_all, int32_t n_all, float* loss_share, float* dz_pair, void* ws,
                                 size_t ws_bytes, cadet_stream_t stream);
/* Logit gradients and loss terms of Eq. 11 on this rank: dz_ctx [n, K] = lambda_ctx (sigma(z_kt) - y)
 * + lambda_pair dz_pair[i] on the routed tower, 0 elsewhere; dz_aux [n, J] = lambda_j dL_j/dz.
 * losses [J + 3] = (L_ctx, L_aux_0 .. L_aux_{J-1}, L_pair share, weighted total), overwritten.
 * dz_pair / pair_share may be NULL (no pairwise term). */
cadet_status cadet_full_loss_grads(const cadet_loss_config* lc_h, const float* logits, int32_t K,
                                   const int32_t* bucket, const float* label, const float* dz_pair,
                                   const float* pair_share, const float* aux_out, const float* aux_label, int32_t n,
                                   float* losses, float* dz_ctx, float* dz_aux, cadet_stream_t stream);
/* Tower backward from given logit gradients dz fp32 [n, K] (every tower; the towers of
 * cadet_heads_loss_backward or the aux heads).  dHs bf16 [T, d]: accumulate = 0 -> overwritten
 * (rows not in `rows` 0), 1 -> dHs[rows] += (other rows untouched).  Gradients overwritten. */
cadet_status cadet_heads_backward(const cadet_head_config* h_h, const cadet_head_weights* w_h, const void* Hs,
                                  const int32_t* rows, int32_t n, int32_t T, const void* pre, const float* dz,
                                  int32_t accumulate, void* dHs, const cadet_head_grads* g_h, void* ws,
                                  size_t ws_bytes, cadet_stream_t stream);

/* ------------------------------------------------------------------ NEXT-3: the CADET block
 * Pre-norm block ("two normalization layers" + "feed-forward network", readings R32/R33):
 *   Xn = RMSNorm_1(X);  H = X + Attn(Xn)     cadet_rmsnorm_forward, cadet_attn_forward(X := Xn, resid := X)
 *   Hn = RMSNorm_2(H);  Y = H + FFN(Hn)      cadet_rmsnorm_forward, cadet_ffn_forward(resid := H)
 * Backward in reverse: cadet_ffn_backward(dresid NULL) -> dHn; cadet_rmsnorm_backward(H, dHn, dresid := dY)
 * -> dH; cadet_attn_backward(dY := dH) -> dXn; cadet_rmsnorm_backward(X, dXn, dresid := dH) -> dX.
 *
 * RMSNorm (R32): Y = X / sqrt(mean_row(X^2) + 1e-6) * gamma.  X, Y bf16 [T, d] row-major, gamma fp32
 * [d], rstd fp32 [T] (saved for the backward).  d % 8 == 0, d <= 1024; else CADET_E_ARG. */
cadet_status cadet_rmsnorm_forward(const void* X, const float* gamma, int32_t T, int32_t d, void* Y, float* rstd,
                                   cadet_stream_t stream);
/* dX = rstd gamma dY - X rstd^3 mean_row(X gamma dY) (+ dresid, nullable), bf16 [T, d];
 * dgamma fp32 [d] = sum_rows dY X rstd, OVERWRITTEN (column sums: fp32 atomics, order not fixed). */
cadet_status cadet_rmsnorm_backward(const void* X, const float* gamma, const float* rstd, const void* dY,
                                    const void* dresid, int32_t T, int32_t d, void* dX, float* dgamma,
                                    cadet_stream_t stream);
/* FFN (R33): U = X W1, G = GELU(U) (exact, erf), Y = G W2 (+ resid, nullable).  X, Y, resid bf16 [T, d];
 * W1 bf16 [d, m d], W2 bf16 [m d, d] (row-vector convention y = x W, R1); U and G bf16 [T, m d] are
 * written for the backward.  d % 32 == 0.  Two tcgen05 GEMM launches, GELU in the first's epilogue. */
cadet_status cadet_ffn_forward(const void* X, const void* W1, const void* W2, const void* resid, int32_t T, int32_t d,
                               int32_t m, void* Y, void* U, void* G, cadet_stream_t stream);
/* dU = (dY W2^T) * GELU'(U) (in ws), dX = dU W1^T (+ dresid, nullable) bf16 [T, d]; dW1 fp32 [d, m d]
 * = X^T dU and dW2 fp32 [m d, d] = G^T dY, OVERWRITTEN.  ws >= cadet_ffn_workspace_bytes(T, d, m). */
size_t cadet_ffn_workspace_bytes(int32_t T, int32_t d, int32_t m);
cadet_status cadet_ffn_backward(const void* X, const void* W1, const void* W2, const void* U, const void* G,
                                const void* dY, const void* dresid, int32_t T, int32_t d, int32_t m, void* dX,
                                float* dW1, float* dW2, void* ws, size_t ws_bytes, cadet_stream_t stream);

/* ------------------------------------------------------------------ NEXT-3: input embeddings (Eq. 1)
 * x = [M; I_1, (C_1, A_1); ...; I_L] (Eq. 1): each token's input row is the sum of its id embeddings and its
 * token-type embedding (reading R37): F tables E_f bf16 [vocab[f], d], token t uses row
 * ids[t * F + f] of table f (an id < 0 = the field is absent for this token kind, e.g. no ad id on an
 * action token).  X[t] = sum_f E_f[ids[t, f]] (fp32 sum, bf16 out) for t < *n_valid (device scalar; NULL
 * = all T rows), rows [*n_valid, T) are 0 (pad rows).  An id >= vocab[f] latches CADET_E_BUCKET and is
 * skipped.  Backward: dE_f[v] = sum_{t : ids[t, f] = v} dX[t], fp32 [vocab[f], d], OVERWRITTEN,
 * deterministic (no order-dependent float atomics: tables with vocab <= 16 reduce per-CTA register
 * partials in a fixed order, larger ones add 64-bit fixed-point values, 2^-24 resolution).
 * d % 8 == 0, 1 <= n_tables <= 8; ws >= cadet_embed_workspace_bytes (the first 256 B: error word). */
#define CADET_EMBED_MAX_TABLES 8
typedef struct {
  int32_t n_tables;
  int32_t d_model;
  int32_t vocab[CADET_EMBED_MAX_TABLES];
} cadet_embed_config;
size_t cadet_embed_workspace_bytes(const cadet_embed_config* c_h);
cadet_status cadet_embed_forward(const cadet_embed_config* c_h, const void* const* tables_h, const int32_t* ids,
                                 int32_t T, const int32_t* n_valid, void* X, void* ws, size_t ws_bytes,
                                 cadet_stream_t stream);
cadet_status cadet_embed_backward(const cadet_embed_config* c_h, const int32_t* ids, int32_t T,
                                  const int32_t* n_valid, const void* dX, float* const* dtables_h, void* ws,
                                  size_t ws_bytes, cadet_stream_t stream);

/* ------------------------------------------------------------------ NEXT-4: HSDP optimizer step
 * HSDP shards parameters, gradients and optimizer state within a node: each rank
 * reduce-scatters the flat fp32 gradient buffer (NCCL, the caller), updates ITS shard with
 * cadet_adamw_step, and the bf16 compute copies are all-gathered (NCCL, the caller).  Reading R35:
 * AdamW, bias-corrected, eps outside the square root, decoupled weight decay:
 *   m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
 *   p = p (1 - lr wd) - lr (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps). */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
} cadet_adamw_config;
void cadet_default_adamw_config(cadet_adamw_config* c_h); /* lr 1e-4, (0.9, 0.999), eps 1e-8, wd 0 */
/* One AdamW step over n fp32 elements (grad read; param, m, v updated in place; step >= 1 counts
 * from 1).  param_bf16 (nullable) receives bf16(param) — the compute copy.  fp32 buffers 16-byte
 * aligned, param_bf16 8-byte aligned; else CADET_E_ARG.  Elementwise: any shard split gives the
 * same result as the whole buffer. */
cadet_status cadet_adamw_step(const cadet_adamw_config* c_h, int64_t step, const float* grad, float* param, float* m,
                              float* v, void* param_bf16, int64_t n, cadet_stream_t stream);
/* dst[i] = (float)src[i] for n bf16 elements (fp32-consumed parameters after a bf16 all-gather).
 * Both buffers 16-byte aligned. */
cadet_status cadet_bf16_to_f32(const void* src, float* dst, int64_t n, cadet_stream_t stream);

/* ------------------------------------------------------------------ context buckets
 * "we partition the context space into K discrete buckets"; the deployed choice is K = 2,
 * "positions 1--4, and 5+", i.e. boundaries {4}.  bucket[i] = #{j : raw_position[i] >
 * boundaries_h[j]} (0-based: SPEC S:142-150's 1-based k minus one), so K = nb + 1 towers.
 * raw_position int32 [n] (device, >= 1: a feed position); boundaries_h host, strictly increasing, 1 <= nb
 * <= 32 (else CADET_E_ARG, synchronously); bucket int32 [n] (device, overwritten).  A position < 1 latches
 * CADET_E_BUCKET in the error word at ws (>= 256 B; cadet_poll) and gets bucket 0. */
cadet_status cadet_bucketize(const int32_t* raw_position, int32_t n, const int32_t* boundaries_h, int32_t nb,
                             int32_t* bucket, void* ws, cadet_stream_t stream);

/* ------------------------------------------------------------------ A0 / A13: chunk and pack
 * Chunk: split each sequence [a, e) of cu_in at e - L, e - 2L, ... (newest chunk full, oldest may be
 * short) and write the refined offsets in buffer order to cu_out (capacity cap entries);
 * n_out[0] (device) = number of chunks.  Chunks stay contiguous: no data moves. */
cadet_status cadet_chunk(const int32_t* cu_in, int32_t n_in, int32_t L_chunk, int32_t* cu_out, int32_t cap,
                         int32_t* n_out, void* ws, cadet_stream_t stream); /* ws >= 256 B: error word (cadet_poll) */
/* Pack: greedy arrival-order packing into one fixed budget: sequences 0..k-1 are
 * copied while their running total fits `budget`; rows [total, budget) are zero-filled.
 * src: bf16 [*, d]; sequence s occupies src rows [src_row[s], src_row[s] + lens[s]) (padded input
 * [B, Lmax, d]: src_row[s] = s * Lmax; contiguous histories: src_row = NULL means the exclusive
 * prefix sum of lens).  t_src (nullable) int64 and s_src (nullable) int32 are per src row and are
 * packed alongside into t_out / s_out ([budget]).
 * Outputs: packed [budget, d], cu_out [B+1] (entries past n_packed repeat the total), n_packed[0].
 * src = packed = NULL packs only the offsets and t / s (one thread per row), and t_out = s_out =
 * NULL only the rows, so the row move can run on another stream than the metadata the plan needs.
 * ws (>= cadet_pack_workspace_bytes) holds the error word read by cadet_poll. */
cadet_status cadet_pack(const void* src, const int64_t* src_row, const int32_t* lens, int32_t B, int32_t d,
                        int32_t budget, const int64_t* t_src, const int32_t* s_src, void* packed, int64_t* t_out,
                        int32_t* s_out, int32_t* cu_out, int32_t* n_packed, void* ws, size_t ws_bytes,
                        cadet_stream_t stream);
size_t cadet_pack_workspace_bytes(int32_t B);

/* ------------------------------------------------------------------ stage hook (tests / building block)
 * C[M, N] = A . B (+ resid) with the tcgen05 GEMM.  A: bf16, storage [M, K] (a_mn = 0) or [K, M]
 * (a_mn = 1); B: bf16, storage [N, K] (b_mn = 0) or [K, N] (b_mn = 1).  C fp32 (c_f32 = 1) or bf16,
 * [M, N]; resid (nullable) same dtype as C.  N % 32 == 0, K % 8 == 0, M % 8 == 0 when MN-major. */
cadet_status cadet_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t a_mn, const void* B, int32_t b_mn,
                        void* C, int32_t c_f32, const void* resid, cadet_stream_t stream);

/* 3xTF32 GEMM of the CADET_FP32 mode (building block / test hook): C[M, N] = op(A) op(B) (+ resid), all fp32,
 * op(A) [M, K] = A stored [M][K] (a_t = 0) or [K][M] (a_t = 1); op(B) [K, N] = B stored [K][N] (b_t = 0, the
 * x . W case) or [N][K] (b_t = 1, the g . W^T case).  Each operand is split once into hi = tf32(x) and
 * lo = x - hi, and C = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulates in fp32 on the tensor cores
 * (kind::tf32).  N % 32 == 0; ws >= cadet_gemm_fp32_workspace_bytes(M, N, K) (the split operands). */
size_t cadet_gemm_fp32_workspace_bytes(int32_t M, int32_t N, int32_t K);
cadet_status cadet_gemm_fp32(int32_t M, int32_t N, int32_t K, const float* A, int32_t a_t, const float* B,
                             int32_t b_t, float* C, const float* resid, void* ws, size_t ws_bytes,
                             cadet_stream_t stream);

/* ------------------------------------------------------------------ instrumentation (bench / tests)
 * cadet_launch_count: number of libcadet kernels launched by this process so far.
 * cadet_prof_enable(classes, max_pairs): from now on every launch of a kernel in `classes`
 * (bit 0 GEMM, bit 1 attention forward, bit 2 attention backward, bit 3 everything else) is
 * bracketed by a cudaEvent pair on its stream (no host sync).  cadet_prof_read synchronises those
 * events and returns, per class, the summed milliseconds and the number of launches; it disables
 * profiling.  Used by bench.py to time the dominant kernel live inside the timed region. */
int64_t cadet_launch_count(void);
cadet_status cadet_prof_enable(int32_t classes, int32_t max_pairs);
cadet_status cadet_prof_read(double* ms_h /*[4]*/, int64_t* launches_h /*[4]*/);

/* ------------------------------------------------------------------ errors
 * Synchronises `stream`, then returns and clears the device-latched error word in ws. */
cadet_status cadet_poll(void* ws, cadet_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CADET_H */
