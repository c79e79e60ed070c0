// libcadet host side, attention core and full gated layer (rows A2-A12).
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include "../../include/cadet.h"
#include "fp32.cuh"
#include "gemm.cuh"
#include "layer.cuh"
#include "misc.cuh"

using namespace cadet;

namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
cadet_status cuda_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CADET_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  set_error(buf);
  return CADET_E_CUDA;
}
cadet_status ws_err(size_t have, size_t need) {
  char buf[128];
  snprintf(buf, sizeof(buf), "workspace %zu < required %zu", have, need);
  set_error(buf);
  return CADET_E_WORKSPACE;
}

AttnParams attn_params(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v) {
  AttnParams p;
  memset(&p, 0, sizeof(p));
  p.fwd_splits = 1;
  p.T = b->total_tokens;
  p.H = c->n_heads;
  p.hd = c->head_dim;
  p.d = c->d_model;
  p.n = b->n_seqs;
  p.scale = 1.0f / sqrtf((float)c->head_dim);
  p.scale_log2 = (float)(1.4426950408889634 / sqrt((double)c->head_dim));
  p.out_f32 = c->out_f32;
  p.cu = b->cu_seqlens;
  p.plan = v;
  return p;
}

// Forward split-KV: when one wave of two CTAs per SM would not be filled by
// the (q-tile, head) grid (a single serving request), each q-tile's visit list is split over 4
// CTAs; the fp32 partials live at the END of the caller's workspace when it is large enough
// (cadet_attn_workspace_bytes includes them; otherwise the kernel runs unsplit).
int fwd_splits_for(const cadet_attn_config* c, int n, int T) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long nq = (long long)(T + 127) / 128 + n;
  if (T <= 0) return 1;
  const long long S = (2LL * sms) / (nq * c->n_heads);  // fill one wave of two CTAs per SM
  return (int)(S < 1 ? 1 : (S > 4 ? 4 : S));
}
size_t fwd_split_bytes(const cadet_attn_config* c, int n, int T) {
  const int S = fwd_splits_for(c, n, T);
  if (S <= 1) return 0;
  return a256((size_t)S * T * c->d_model * 4) + 2 * a256((size_t)S * c->n_heads * T * 4) + 256;
}
void set_fwd_split(AttnParams& p, const cadet_attn_config* c, int n, int T, void* ws, size_t ws_bytes,
                   size_t base_need) {
  const int S = fwd_splits_for(c, n, T);
  const size_t sb = fwd_split_bytes(c, n, T);
  p.fwd_splits = 1;
  if (S <= 1 || ws_bytes < base_need + sb) return;
  uint8_t* e = reinterpret_cast<uint8_t*>(ws) + ((ws_bytes - sb + 255) & ~size_t(255));
  p.Opart = reinterpret_cast<float*>(e);
  e += a256((size_t)S * T * c->d_model * 4);
  p.Mpart = reinterpret_cast<float*>(e);
  e += a256((size_t)S * c->n_heads * T * 4);
  p.Lpart = reinterpret_cast<float*>(e);
  p.fwd_splits = S;
}
}  // namespace

extern "C" {

cadet_status cadet_attn_core_forward(const cadet_attn_config* cfg, const cadet_batch* b, const void* Qr,
                                     const void* Kr, const void* V, void* O, float* lse, void* ws, size_t ws_bytes,
                                     cadet_stream_t stream) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!Qr || !Kr || !V || !O || !lse || !ws) {
    set_error("cadet_attn_core_forward: null pointer");
    return CADET_E_ARG;
  }
  const size_t need = plan_bytes(b->n_seqs, b->total_tokens, b->total_tokens);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!cfg->plan_ready && (s = cadet_mask_plan(cfg, b, ws, ws_bytes, stream))) return s;
  PlanView v = plan_carve(ws, b->n_seqs, b->total_tokens, b->total_tokens);
  if (cfg->dtype == CADET_FP32)  // fp32 Qr, Kr, V in; fp32 O out
    return cuda_err(attn_fwd_f32(cfg, b, v, (const float*)Qr, (const float*)Kr, (const float*)V, (float*)O, lse, st),
                    "attention forward (fp32)");
  AttnParams p = attn_params(cfg, b, v);
  p.O = O;
  p.lse = lse;
  set_fwd_split(p, cfg, b->n_seqs, b->total_tokens, ws, ws_bytes, need);
  const int T = b->total_tokens, d = cfg->d_model;
  // pad rows: O = 0, LSE = 0 (R17)
  cudaError_t e = zero_pad_rows_launch(O, d * (cfg->out_f32 ? 4 : 2), T, b->cu_seqlens, b->n_seqs, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(lse, 0, sizeof(float) * (size_t)T * cfg->n_heads, st);
  if (e == cudaSuccess) e = attn_fwd_launch(Qr, Kr, V, p, st);
  return cuda_err(e, "attention forward");
}


cadet_status cadet_attn_core_backward(const cadet_attn_config* cfg, const cadet_batch* b, const void* Qr,
                                      const void* Kr, const void* V, const void* O, const float* lse, const void* dO,
                                      float* dQr, void* dKr, void* dV, void* ws, size_t ws_bytes,
                                      cadet_stream_t stream) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!Qr || !Kr || !V || !O || !lse || !dO || !dQr || !dKr || !dV || !ws) {
    set_error("cadet_attn_core_backward: null pointer");
    return CADET_E_ARG;
  }
  const int T = b->total_tokens, d = cfg->d_model, H = cfg->n_heads;
  const size_t pb = plan_bytes(b->n_seqs, T, T);
  const size_t need = pb + a256((size_t)4 * H * T);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!cfg->plan_ready && (s = cadet_mask_plan(cfg, b, ws, ws_bytes, stream))) return s;
  PlanView v = plan_carve(ws, b->n_seqs, T, T);
  float* D = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pb);
  if (cfg->dtype == CADET_FP32)  // every tensor fp32
    return cuda_err(attn_bwd_f32(cfg, b, v, (const float*)Qr, (const float*)Kr, (const float*)V, (const float*)O, lse,
                                 (const float*)dO, D, dQr, (float*)dKr, (float*)dV, st),
                    "attention backward (fp32)");
  AttnParams p = attn_params(cfg, b, v);
  p.lse = const_cast<float*>(lse);
  p.D = D;
  p.dQ = dQr;
  p.dK = dKr;
  p.dV = dV;
  const int ob = d * (cfg->out_f32 ? 4 : 2);
  cudaError_t e = attn_bwd_pre_launch(O, dO, D, dQr, T, H, cfg->head_dim, st);
  if (e == cudaSuccess) e = zero_pad_rows_launch(dQr, d * 4, T, b->cu_seqlens, b->n_seqs, st);
  if (e == cudaSuccess) {
    void* pads[2] = {dKr, dV};
    e = zero_pad_rows_multi_launch(pads, 2, ob, T, b->cu_seqlens, b->n_seqs, st);
  }
  if (e == cudaSuccess) e = attn_bwd_launch(Qr, Kr, V, dO, p, st);
  return cuda_err(e, "attention backward");
}

}  // extern "C"

// =====================================================================================
// Full gated layer (rows A2-A12)
// =====================================================================================
namespace {

struct LayerBufs {  // carved from `saved`
  void *Zx, *Xt, *Q, *K, *Zq, *Zk, *Qr, *Kr, *V, *O;
  float* lse;
};
// Parity taps (cfg.out_f32 = 1 on the layer calls): fp32 [T, d] copies of every stage's value before
// its bf16 rounding, in the order of the CADET_TAP_* views of include/cadet.h.
enum { TAP_ZX, TAP_XT, TAP_Q, TAP_K, TAP_V, TAP_ZQ, TAP_ZK, TAP_QR, TAP_KR, TAP_O, TAP_Y, TAP_DO, TAP_DQR, TAP_DKR,
       TAP_DV, TAP_UQ, TAP_RQ, TAP_UK, TAP_RK, TAP_DQ, TAP_DK, TAP_UX, TAP_RX, TAP_DX, N_TAPS };
static_assert(N_TAPS == CADET_N_TAPS, "tap list out of sync with cadet.h");
struct LayerWs {    // carved from `ws` after the plan
  float* D;
  void *dO, *dKr, *dV, *uq, *uk, *dQ, *dK, *ux;
  float *dQacc, *rq, *rk, *rx;
  float* tap[N_TAPS];  // all null unless cfg.out_f32
  float* slab;         // deterministic mode: split-K partial slabs (null otherwise)
};

size_t bf_sz(int T, int d) { return a256((size_t)T * d * 2); }
size_t f_sz(int T, int d) { return a256((size_t)T * d * 4); }

LayerBufs carve_saved(void* saved, const cadet_attn_config* c, int T) {
  uint8_t* p = reinterpret_cast<uint8_t*>(saved);
  const size_t z = bf_sz(T, c->d_model);
  LayerBufs L;
  void** slots[10] = {&L.Zx, &L.Xt, &L.Q, &L.K, &L.Zq, &L.Zk, &L.Qr, &L.Kr, &L.V, &L.O};
  for (int i = 0; i < 10; ++i) *slots[i] = p + i * z;
  L.lse = reinterpret_cast<float*>(p + 10 * z);
  return L;
}
size_t saved_bytes(const cadet_attn_config* c, int T) {
  if (c->dtype == CADET_FP32) return f32_saved_bytes(c, T);
  return 10 * bf_sz(T, c->d_model) + a256((size_t)4 * c->n_heads * T);
}
int pick_bn_wgrad(int N);
int pick_split(int M, int N, int bn, int K);
// deterministic mode: fp32 split-K partial slabs of up to 3 weight gradients of one launch
size_t det_slab_bytes(const cadet_attn_config* c, int T) {
  if (!c->deterministic) return 0;
  const int d = c->d_model;
  return 3 * a256((size_t)pick_split(d, d, pick_bn_wgrad(d), T) * d * d * 4);
}
size_t layer_ws_base_bytes(const cadet_attn_config* c, int n, int T) {
  const int d = c->d_model;
  return plan_bytes(n, T, T) + a256((size_t)4 * c->n_heads * T) + 8 * bf_sz(T, d) + 4 * f_sz(T, d) + (c->out_f32 ? N_TAPS * f_sz(T, d) : 0) +
         det_slab_bytes(c, T);
}
size_t layer_ws_bytes(const cadet_attn_config* c, int n, int T) {
  if (c->dtype == CADET_FP32) return f32_layer_ws_bytes(c, n, T);
  return layer_ws_base_bytes(c, n, T) + fwd_split_bytes(c, n, T);
}
// Two-pass attention backward: dS^T tile slots (sum over sequences of nq_s (nq_s + 1) / 2, bounded
// with nq_s <= max_seqlen / 128 + 3 exactly like the plan's visit lists) x H x [128 x 128] bf16.
int32_t ds_slots_of(int n, int T, int max_seqlen) {
  const long long nq = (T + 127) / 128 + n, hm = (max_seqlen + 127) / 128 + 3;
  const long long s = nq * (hm + 1) / 2 + hm;
  return s > (1LL << 24) ? 0 : (int32_t)s;
}
size_t ds_bytes_of(const cadet_attn_config* c, int n, int T, int max_seqlen) {
  const int32_t s = ds_slots_of(n, T, max_seqlen);
  return s ? a256((size_t)s * c->n_heads * 128 * 128 * 2) : 0;
}
LayerWs carve_ws(void* ws, const cadet_attn_config* c, int n, int T) {
  const int d = c->d_model;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws) + plan_bytes(n, T, T);
  LayerWs W;
  W.D = reinterpret_cast<float*>(p);
  p += a256((size_t)4 * c->n_heads * T);
  void** bf[8] = {&W.dO, &W.dKr, &W.dV, &W.uq, &W.uk, &W.dQ, &W.dK, &W.ux};
  for (int i = 0; i < 8; ++i) {
    *bf[i] = p;
    p += bf_sz(T, d);
  }
  float** fp[4] = {&W.dQacc, &W.rq, &W.rk, &W.rx};
  for (int i = 0; i < 4; ++i) {
    *fp[i] = reinterpret_cast<float*>(p);
    p += f_sz(T, d);
  }
  for (int i = 0; i < N_TAPS; ++i) {
    W.tap[i] = c->out_f32 ? reinterpret_cast<float*>(p) : nullptr;
    if (c->out_f32) p += f_sz(T, d);
  }
  W.slab = c->deterministic ? reinterpret_cast<float*>(p) : nullptr;
  return W;
}

// Timestamp RoPE of the layer, evaluated on the fly by the kernels that rotate
RopeOTF rope_of(const cadet_attn_config* cfg, const cadet_batch* b, const PlanView& v) {
  (void)b;
  RopeOTF r;
  r.dt = v.rope_dt;
  r.theta = v.theta;
  r.on = cfg->use_rope;
  return r;
}

int pick_bn(int M, int N) {
  if (N % 256 == 0 && (long long)((M + 127) / 128) * (N / 256) >= 148) return 256;
  if (N <= 128) return 128;
  const int w256 = (N + 255) / 256 * 256 - N, w128 = (N + 127) / 128 * 128 - N;
  return (w256 <= w128 && (long long)((M + 127) / 128) * ((N + 255) / 256) >= 148) ? 256 : 128;
}
// Weight gradients are split-K, so tile count is never the limit: prefer BN = 256 (BN = 128 with
// both operands from smem needs 128 B/clk of smem bandwidth per SM, the whole budget).
int pick_bn_wgrad(int N) { return (N >= 256 && ((N + 255) / 256 * 256 - N) <= ((N + 127) / 128 * 128 - N) + 64) ? 256 : 128; }
int pick_split(int M, int N, int bn, int K) {
  const long long tiles = (long long)((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = (K + 63) / 64;
  long long split = (2 * 148 + tiles - 1) / tiles;
  if (split > kb / 4) split = kb / 4;
  return split < 1 ? 1 : (int)split;
}

OperandDesc act(const void* p, int T, int d) { return OperandDesc{p, T, d, 0}; }       // [T, d] as K-major A
OperandDesc act_t(const void* p, int T, int d) { return OperandDesc{p, T, d, 1}; }     // [T, d] as MN-major (wgrad)
OperandDesc w_fwd(const void* W, int din, int dout) { return OperandDesc{W, din, dout, 1}; }  // x.W: B MN-major
OperandDesc w_bwd(const void* W, int din, int dout) { return OperandDesc{W, din, dout, 0}; }  // g.W^T: B K-major

GemmProblem prob(int M, int N, int K, OperandDesc A, OperandDesc B, int mode) {
  GemmProblem g;
  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.nseg = 1;
  g.K[0] = K;
  g.A[0] = A;
  g.B[0] = B;
  g.split_k = 1;
  g.epi.mode = mode;
  g.epi.ldo = N;
  return g;
}

// dW = A^T . G over T rows, fp32, split-K with atomics into a zeroed output; with a slab (deterministic
// mode) each split stores its partial into slab + ks din dout and slab_reduce sums them in order.
GemmProblem wgrad(const void* A, const void* G, float* dW, int T, int din, int dout, int bn, float* slab = nullptr) {
  GemmProblem g = prob(din, dout, T, act_t(A, T, din), act_t(G, T, dout), EPI_ATOMIC);
  g.split_k = pick_split(din, dout, bn, T);
  g.epi.out = slab ? slab : dW;
  g.epi.out_f32 = 1;
  g.epi.split_stride = slab ? (int64_t)din * dout : 0;
  return g;
}

// Two independent groups of GEMMs (e.g. an input gradient and the weight gradient that shares its
// operand) as ONE persistent launch when they use the same N tile: one ramp-up / tail instead of two.
cudaError_t gemm_launch2(const GemmProblem* a, int na, int bna, const GemmProblem* b, int nb, int bnb,
                         cudaStream_t st) {
  if (bna == bnb && na + nb <= GEMM_MAX_PROB) {
    GemmProblem g[GEMM_MAX_PROB];
    for (int i = 0; i < na; ++i) g[i] = a[i];
    for (int i = 0; i < nb; ++i) g[na + i] = b[i];
    return gemm_launch(g, na + nb, bna, st);
  }
  cudaError_t e = gemm_launch(a, na, bna, st);
  return e == cudaSuccess ? gemm_launch(b, nb, bnb, st) : e;
}

}  // namespace

extern "C" {

size_t cadet_attn_workspace_bytes(const cadet_attn_config* c, int32_t n, int32_t T) {
  if (check_cfg(c)) return 0;
  return layer_ws_bytes(c, n, T);
}
size_t cadet_attn_bwd_ds_bytes(const cadet_attn_config* c, int32_t n, int32_t T, int32_t max_seqlen) {
  if (check_cfg(c) || n < 0 || T < 0 || max_seqlen < 1 || c->dtype == CADET_FP32) return 0;
  return ds_bytes_of(c, n, T, max_seqlen);
}
size_t cadet_attn_saved_bytes(const cadet_attn_config* c, int32_t T) {
  if (check_cfg(c)) return 0;
  return saved_bytes(c, T);
}

cadet_status cadet_attn_stage_views(const cadet_attn_config* cfg, int32_t n, int32_t T, void* ws, size_t ws_bytes,
                                    void** views_h) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if (!ws || !views_h || n < 0 || T < 0) {
    set_error("cadet_attn_stage_views: null pointer or negative size");
    return CADET_E_ARG;
  }
  if (cfg->dtype == CADET_FP32) {
    set_error("cadet_attn_stage_views: bf16 layer only (the fp32 mode stores every stage in fp32)");
    return CADET_E_UNSUPPORTED;
  }
  const size_t need = layer_ws_bytes(cfg, n, T);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  LayerWs W = carve_ws(ws, cfg, n, T);
  for (int i = 0; i < CADET_N_VIEWS; ++i) views_h[i] = nullptr;
  for (int i = 0; i < N_TAPS; ++i) views_h[i] = W.tap[i];
  void* bf[12] = {W.dO, W.dQacc, W.dKr, W.dV, W.uq, W.rq, W.uk, W.rk, W.dQ, W.dK, W.ux, W.rx};
  for (int i = 0; i < 12; ++i) views_h[CADET_WS_DO + i] = bf[i];
  views_h[CADET_WS_D] = W.D;
  return CADET_OK;
}

cadet_status cadet_attn_forward(const cadet_attn_config* cfg, const cadet_batch* b, const cadet_attn_weights* w,
                                const void* X, void* Y, const void* resid, void* saved, void* ws, size_t ws_bytes,
                                cadet_stream_t stream) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!w || !X || !Y || !saved || !ws || !w->W_q || !w->W_k || !w->W_v || (cfg->use_rep_gate && !w->W_xg) ||
      (cfg->use_int_gate && (!w->W_qg || !w->W_kg)) || (cfg->use_out_proj && !w->W_o)) {
    set_error("cadet_attn_forward: null pointer");
    return CADET_E_ARG;
  }
  const int T = b->total_tokens, d = cfg->d_model, n = b->n_seqs, hd = cfg->head_dim;
  const size_t need = layer_ws_bytes(cfg, n, T);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  if (T == 0) return CADET_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!cfg->plan_ready && (s = cadet_mask_plan(cfg, b, ws, ws_bytes, stream))) return s;
  if (cfg->dtype == CADET_FP32)  // X, Y, resid, weights fp32 (3xTF32 GEMMs)
    return cuda_err(layer_forward_f32(cfg, b, w, (const float*)X, (float*)Y, (const float*)resid, saved, ws, st),
                    "attention layer forward (fp32)");
  PlanView v = plan_carve(ws, n, T, T);
  LayerBufs L = carve_saved(saved, cfg, T);
  LayerWs W = carve_ws(ws, cfg, n, T);
  cudaError_t e = cudaSuccess;
  const RopeOTF rp = rope_of(cfg, b, v);
  const int bn = pick_bn(T, d);
  // A2: representation gate  Xt = X * sigma(X W_xg)   (Eq. 4)
  const void* Xt = X;
  if (e == cudaSuccess && cfg->use_rep_gate) {
    GemmProblem g = prob(T, d, d, act(X, T, d), w_fwd(w->W_xg, d, d), EPI_GATE);
    g.epi.out = L.Xt;
    g.epi.src = X;
    g.epi.aux = L.Zx;
    g.epi.tap = W.tap[TAP_XT];
    g.epi.tap2 = W.tap[TAP_ZX];
    e = gemm_launch(&g, 1, bn, st);
    Xt = L.Xt;
  }
  // A3: Q, K, V = Xt W_{q,k,v}   (Eq. 3; R2)
  if (e == cudaSuccess) {
    GemmProblem g[3];
    const void* Ws[3] = {w->W_q, w->W_k, w->W_v};
    void* outs[3] = {L.Q, L.K, L.V};
    for (int i = 0; i < 3; ++i) {
      g[i] = prob(T, d, d, act(Xt, T, d), w_fwd(Ws[i], d, d), EPI_STORE);
      g[i].epi.out = outs[i];
      g[i].epi.tap = W.tap[TAP_Q + i];
    }
    e = gemm_launch(g, 3, bn, st);
  }
  // A4: interaction gates + timestamp RoPE  (Eq. 5)
  if (e == cudaSuccess) {
    if (cfg->use_int_gate) {
      // Zq = Q W_qg, Zk = K W_kg stored plainly (saved for the backward); sigma, the product with Q, K
      // and the rotation run in one HBM pass after (a fused gate+RoPE epilogue made these GEMMs
      // epilogue-bound at 0.66 of their mainloop rate)
      GemmProblem g[2];
      const void* Ws[2] = {w->W_qg, w->W_kg};
      const void* src[2] = {L.Q, L.K};
      void* zs[2] = {L.Zq, L.Zk};
      for (int i = 0; i < 2; ++i) {
        g[i] = prob(T, d, d, act(src[i], T, d), w_fwd(Ws[i], d, d), EPI_STORE);
        g[i].epi.out = zs[i];
        g[i].epi.tap = W.tap[TAP_ZQ + i];
      }
      e = gemm_launch(g, 2, bn, st);
      if (e == cudaSuccess)
        e = gate_rope_fwd_launch(L.Q, L.K, L.Zq, L.Zk, rp, L.Qr, L.Kr, T, d, hd, st,
                                 W.tap[TAP_QR], W.tap[TAP_KR]);
    } else if (cfg->use_rope) {
      e = rope_apply_launch(L.Q, L.Qr, T, d, hd, rp, st);
      if (e == cudaSuccess) e = rope_apply_launch(L.K, L.Kr, T, d, hd, rp, st);
    } else {
      e = cudaMemcpyAsync(L.Qr, L.Q, (size_t)T * d * 2, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(L.Kr, L.K, (size_t)T * d * 2, cudaMemcpyDeviceToDevice, st);
    }
  }
  // A5: attention core
  if (e == cudaSuccess) {
    AttnParams p = attn_params(cfg, b, v);
    p.out_f32 = 0;
    p.O = L.O;
    p.lse = L.lse;
    set_fwd_split(p, cfg, n, T, ws, ws_bytes, layer_ws_base_bytes(cfg, n, T));
    e = zero_pad_rows_launch(L.O, d * 2, T, b->cu_seqlens, n, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(L.lse, 0, sizeof(float) * (size_t)T * cfg->n_heads, st);
    if (e == cudaSuccess) e = attn_fwd_launch(L.Qr, L.Kr, L.V, p, st);
    if (e == cudaSuccess && W.tap[TAP_O]) {  // parity tap: the same (deterministic) kernel, fp32 O
      p.out_f32 = 1;
      p.O = W.tap[TAP_O];
      e = zero_pad_rows_launch(W.tap[TAP_O], d * 4, T, b->cu_seqlens, n, st);
      if (e == cudaSuccess) e = attn_fwd_launch(L.Qr, L.Kr, L.V, p, st);
    }
  }
  // A6: Y = O W_o (+ resid)
  if (e == cudaSuccess) {
    if (cfg->use_out_proj) {
      GemmProblem g = prob(T, d, d, act(L.O, T, d), w_fwd(w->W_o, d, d), EPI_STORE);
      g.epi.out = Y;
      g.epi.resid = resid;
      g.epi.tap = W.tap[TAP_Y];
      e = gemm_launch(&g, 1, bn, st);
    } else {
      e = add_bf16_launch(L.O, resid, Y, (size_t)T * d, st);
    }
  }
  return cuda_err(e, "attention layer forward");
}

cadet_status cadet_attn_backward_ev(const cadet_attn_config* cfg, const cadet_batch* b, const cadet_attn_weights* w,
                                 const void* X, const void* saved, const void* dY, void* dX, const void* dresid,
                                 const cadet_attn_grads* gr, void* ws, size_t ws_bytes, cadet_stream_t stream,
                                    void* const* grad_events) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!w || !X || !saved || !dY || !dX || !gr || !ws || !gr->dW_q || !gr->dW_k || !gr->dW_v ||
      (cfg->use_rep_gate && !gr->dW_xg) || (cfg->use_int_gate && (!gr->dW_qg || !gr->dW_kg)) ||
      (cfg->use_out_proj && !gr->dW_o)) {
    set_error("cadet_attn_backward: null pointer");
    return CADET_E_ARG;
  }
  const int T = b->total_tokens, d = cfg->d_model, n = b->n_seqs, hd = cfg->head_dim, H = cfg->n_heads;
  const size_t need = layer_ws_bytes(cfg, n, T);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  if (T == 0) return CADET_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!cfg->plan_ready && (s = cadet_mask_plan(cfg, b, ws, ws_bytes, stream))) return s;
  if (cfg->dtype == CADET_FP32)  // X, dY, dX, dresid, weights fp32 (3xTF32 GEMMs)
    return cuda_err(layer_backward_f32(cfg, b, w, (const float*)X, saved, (const float*)dY, (float*)dX,
                                       (const float*)dresid, gr, ws, st, grad_events),
                    "attention layer backward (fp32)");
  PlanView v = plan_carve(ws, n, T, T);
  LayerBufs L = carve_saved(const_cast<void*>(saved), cfg, T);
  LayerWs W = carve_ws(ws, cfg, n, T);
  const int bn = pick_bn(T, d);
  const int bnw = pick_bn_wgrad(d);
  const size_t wbytes = (size_t)d * d * 4;
  cudaError_t e = cudaSuccess;
  const RopeOTF cs = rope_of(cfg, b, v);
  float* gws[7] = {gr->dW_xg, gr->dW_q, gr->dW_k, gr->dW_v, gr->dW_qg, gr->dW_kg, gr->dW_o};
  // deterministic mode: no fp32 atomics anywhere in the layer backward -- split-K weight-gradient partials
  // go to slabs summed in a fixed order, and D comes from the (fixed-order) preprocess kernel
  const bool det = cfg->deterministic != 0;
  const int wsplit = pick_split(d, d, bnw, T);
  auto slab = [&](int j) { return det ? W.slab + (size_t)j * wsplit * d * d : nullptr; };
  auto reduce = [&](float* const* dWs, int count) {
    for (int j = 0; j < count && det && e == cudaSuccess; ++j)
      e = slab_reduce_launch(slab(j), wsplit, (size_t)d * d, dWs[j], st);
  };
  // A10's preprocess D = rowsum(dO * O) per head comes out of the A9 GEMM's epilogue when it exists
  const bool d_in_a9 = cfg->use_out_proj && hd >= 32 && !det;
  if (e == cudaSuccess) {  // the 7 weight gradients (split-K accumulated) and D (atomics): one launch
    ZeroSpan zs[8];
    for (int i = 0; i < 7; ++i) zs[i] = ZeroSpan{gws[i], wbytes};
    zs[7] = ZeroSpan{d_in_a9 ? W.D : nullptr, sizeof(float) * (size_t)H * T};
    e = zero_many_launch(zs, 8, st);
  }
  auto mark = [&](int i) {  // grad group i complete on `st` (SURVEY 8(e) overlap)
    if (e == cudaSuccess && grad_events && grad_events[i]) e = cudaEventRecord((cudaEvent_t)grad_events[i], st);
  };
  const void* Xt = cfg->use_rep_gate ? L.Xt : X;
  // A9: dO = dY W_o^T ; dW_o = O^T dY
  const void* dO = dY;
  if (e == cudaSuccess && cfg->use_out_proj) {
    GemmProblem g = prob(T, d, d, act(dY, T, d), w_bwd(w->W_o, d, d), EPI_STORE);
    g.epi.out = W.dO;
    g.epi.tap = W.tap[TAP_DO];
    if (d_in_a9) {
      g.epi.dot_src = L.O;
      g.epi.dot_out = W.D;
      g.epi.dot_T = T;
      g.epi.hd = hd;
    }
    GemmProblem gw = wgrad(L.O, dY, gr->dW_o, T, d, d, bnw, slab(0));
    e = gemm_launch2(&g, 1, bn, &gw, 1, bnw, st);
    reduce(&gr->dW_o, 1);
    dO = W.dO;
  }
  mark(0);
  // A10: attention core backward
  if (e == cudaSuccess) {
    AttnParams p = attn_params(cfg, b, v);
    p.out_f32 = 0;
    p.lse = L.lse;
    p.D = W.D;
    p.dQ = W.dQacc;
    p.dq_bf16 = 1;  // dQ_r rounded to bf16 like dK_r before R(-alpha) and the gate backward
    p.dK = W.dKr;
    p.dV = W.dV;
    // two-pass backward when the caller's workspace holds the dS region (after the layer's own
    // buffers, before the forward split partials at the end; cadet_attn_bwd_ds_bytes)
    const size_t dsb = ds_bytes_of(cfg, n, T, b->max_seqlen);
    if (dsb && ws_bytes >= layer_ws_bytes(cfg, n, T) + dsb) {
      p.dS = reinterpret_cast<uint8_t*>(ws) + layer_ws_base_bytes(cfg, n, T);
      p.ds_slots = ds_slots_of(n, T, b->max_seqlen);
    }
    if (!d_in_a9) e = attn_bwd_pre_launch(L.O, dO, W.D, W.dQacc, T, H, hd, st);
    if (e == cudaSuccess) {  // pad rows of the attention gradients: one launch for the three
      void* pads[3] = {W.dQacc, W.dKr, W.dV};
      e = zero_pad_rows_multi_launch(pads, 3, d * 2, T, b->cu_seqlens, n, st);
    }
    if (e == cudaSuccess) e = attn_bwd_launch(L.Qr, L.Kr, L.V, dO, p, st);
    if (e == cudaSuccess && W.tap[TAP_DQR]) {  // parity taps: the same (deterministic) kernels, fp32 outputs
      p.out_f32 = 1;
      p.dq_bf16 = 0;
      p.dQ = W.tap[TAP_DQR];
      p.dK = W.tap[TAP_DKR];
      p.dV = W.tap[TAP_DV];
      void* pads[3] = {W.tap[TAP_DQR], W.tap[TAP_DKR], W.tap[TAP_DV]};
      e = zero_pad_rows_multi_launch(pads, 3, d * 4, T, b->cu_seqlens, n, st);
      if (e == cudaSuccess) e = attn_bwd_launch(L.Qr, L.Kr, L.V, dO, p, st);
    }
  }
  // A11: R(-alpha) + interaction-gate backward
  const void* dQ = W.dQ;
  const void* dK = W.dK;
  if (e == cudaSuccess) {
    if (cfg->use_int_gate) {
      {  // Q and K sides in one launch
        const void* drs[2] = {W.dQacc, W.dKr};
        const void* xs[2] = {L.Q, L.K};
        const void* zs[2] = {L.Zq, L.Zk};
        void* us[2] = {W.uq, W.uk};
        void* rs[2] = {W.rq, W.rk};
        float* tu[2] = {W.tap[TAP_UQ], W.tap[TAP_UK]};
        float* tr[2] = {W.tap[TAP_RQ], W.tap[TAP_RK]};
        e = rope_gate_bwd_launch2(drs, xs, zs, us, rs, 2, 0, 1, T, d, hd, cs, st, tu, tr);
      }
      if (e == cudaSuccess) {  // dQ = rq + uq W_qg^T ; dK = rk + uk W_kg^T
        GemmProblem g[2];
        const void* us[2] = {W.uq, W.uk};
        const void* rs[2] = {W.rq, W.rk};  // bf16
        const void* Ws[2] = {w->W_qg, w->W_kg};
        void* outs[2] = {W.dQ, W.dK};
        for (int i = 0; i < 2; ++i) {
          g[i] = prob(T, d, d, act(us[i], T, d), w_bwd(Ws[i], d, d), EPI_STORE);
          g[i].epi.out = outs[i];
          g[i].epi.resid = rs[i];
          g[i].epi.resid_f32 = 0;
          g[i].epi.tap = W.tap[TAP_DQ + i];
        }
        // dW_qg = Q^T uq ; dW_kg = K^T uk share the u operands: same launch
        GemmProblem gw[2] = {wgrad(L.Q, W.uq, gr->dW_qg, T, d, d, bnw, slab(0)),
                             wgrad(L.K, W.uk, gr->dW_kg, T, d, d, bnw, slab(1))};
        e = gemm_launch2(g, 2, bn, gw, 2, bnw, st);
        float* dws[2] = {gr->dW_qg, gr->dW_kg};
        reduce(dws, 2);
      }
    } else {
      e = rope_gate_bwd_launch(W.dQacc, 0, nullptr, nullptr, nullptr, W.dQ, 1, T, d, hd, cs, st);
      if (e == cudaSuccess)
        e = rope_gate_bwd_launch(W.dKr, 0, nullptr, nullptr, nullptr, W.dK, 1, T, d, hd, cs, st);
    }
  }
  mark(1);
  // A12: dXt = dQ W_q^T + dK W_k^T + dV W_v^T (one K = 3d accumulation), weight grads, rep-gate bwd
  if (e == cudaSuccess) {
    GemmProblem g;
    memset(&g, 0, sizeof(g));
    g.M = T;
    g.N = d;
    g.nseg = 3;
    const void* gs[3] = {dQ, dK, W.dV};
    const void* Ws[3] = {w->W_q, w->W_k, w->W_v};
    for (int i = 0; i < 3; ++i) {
      g.K[i] = d;
      g.A[i] = act(gs[i], T, d);
      g.B[i] = w_bwd(Ws[i], d, d);
    }
    g.split_k = 1;
    g.epi.ldo = d;
    if (cfg->use_rep_gate) {  // ux = dXt * X * g (1 - g) ; rx = dXt * g (+ dresid)
      g.epi.mode = EPI_GATE_BWD;
      g.epi.out = W.ux;
      g.epi.out2 = W.rx;  // bf16 (like r_q, r_k): rounded once before the bf16 dX it feeds
      g.epi.out2_f32 = 0;
      g.epi.src = X;
      g.epi.aux = L.Zx;
      g.epi.resid = dresid;
      g.epi.tap = W.tap[TAP_UX];
      g.epi.tap2 = W.tap[TAP_RX];
    } else {
      g.epi.mode = EPI_STORE;
      g.epi.out = dX;
      g.epi.resid = dresid;
      g.epi.tap = W.tap[TAP_DX];
    }
    {  // with the weight gradients of W_q, W_k, W_v (same dQ, dK, dV operands) in one launch
      GemmProblem gw[3] = {wgrad(Xt, dQ, gr->dW_q, T, d, d, bnw, slab(0)), wgrad(Xt, dK, gr->dW_k, T, d, d, bnw, slab(1)),
                           wgrad(Xt, W.dV, gr->dW_v, T, d, d, bnw, slab(2))};
      e = gemm_launch2(&g, 1, bn, gw, 3, bnw, st);
      float* dws[3] = {gr->dW_q, gr->dW_k, gr->dW_v};
      reduce(dws, 3);
    }
    mark(2);
    if (e == cudaSuccess && cfg->use_rep_gate) {  // dX = rx + ux W_xg^T ; dW_xg = X^T ux
      GemmProblem g2 = prob(T, d, d, act(W.ux, T, d), w_bwd(w->W_xg, d, d), EPI_STORE);
      g2.epi.out = dX;
      g2.epi.resid = W.rx;
      g2.epi.resid_f32 = 0;
      g2.epi.tap = W.tap[TAP_DX];
      GemmProblem gw = wgrad(X, W.ux, gr->dW_xg, T, d, d, bnw, slab(0));
      e = gemm_launch2(&g2, 1, bn, &gw, 1, bnw, st);
      reduce(&gr->dW_xg, 1);
    }
  }
  mark(3);
  if (e == cudaSuccess) e = zero_pad_rows_launch(dX, d * 2, T, b->cu_seqlens, n, st);
  return cuda_err(e, "attention layer backward");
}

cadet_status cadet_attn_backward(const cadet_attn_config* cfg, const cadet_batch* b, const cadet_attn_weights* w,
                                 const void* X, const void* saved, const void* dY, void* dX, const void* dresid,
                                 const cadet_attn_grads* gr, void* ws, size_t ws_bytes, cadet_stream_t stream) {
  return cadet_attn_backward_ev(cfg, b, w, X, saved, dY, dX, dresid, gr, ws, ws_bytes, stream, nullptr);
}

// =====================================================================================
// Heads (rows A7 / A8)
// =====================================================================================
static cadet_status check_head(const cadet_head_config* h, const cadet_head_weights* w) {
  if (!h || !w || !w->W1 || !w->b1 || !w->w2 || !w->b2) {
    set_error("heads: null pointer");
    return CADET_E_ARG;
  }
  if (h->K < 1 || h->d_model <= 0 || h->d_model % 8 || h->d_hidden < 32 || h->d_hidden % 8 ||
      (h->K * h->d_hidden) % 32) {
    set_error("heads: K >= 1, d_model % 8 == 0, d_hidden % 8 == 0 and >= 32, K*d_hidden % 32 == 0 required");
    return CADET_E_ARG;
  }
  if (h->dtype != CADET_BF16 && h->dtype != CADET_FP32) {
    set_error("heads: dtype must be CADET_BF16 or CADET_FP32");
    return CADET_E_ARG;
  }
  return CADET_OK;
}

size_t cadet_heads_workspace_bytes(const cadet_head_config* h, int32_t n) {
  if (!h || n < 0) return 0;
  if (h->dtype == CADET_FP32) return f32_heads_ws_bytes(h, n);
  const int N = h->K * h->d_hidden;
  return 256 + a256((size_t)n * h->d_model * 2) + a256((size_t)n * N * 2) * 2 + a256((size_t)n * 4) +
         a256((size_t)h->d_model * N * 2);
}
// fp16 copy of W1 in the heads workspace (after the error word, H_r, pre / spare, dhid and dz)
static void* heads_w1h(void* ws, const cadet_head_config* h, int n) {
  const int N = h->K * h->d_hidden;
  return reinterpret_cast<uint8_t*>(ws) + 256 + a256((size_t)n * h->d_model * 2) + a256((size_t)n * N * 2) * 2 +
         a256((size_t)n * 4);
}

cadet_status cadet_heads_forward(const cadet_head_config* h, const cadet_head_weights* w, const void* Hs,
                                 const int32_t* rows, int32_t n, float* logits, void* pre_out, void* ws,
                                 size_t ws_bytes, cadet_stream_t stream) {
  cadet_status s = check_head(h, w);
  if (s) return s;
  if (!Hs || !rows || !logits || !ws || n < 0) {
    set_error("heads_forward: null pointer");
    return CADET_E_ARG;
  }
  const size_t need = cadet_heads_workspace_bytes(h, n);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  if (n == 0) return CADET_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (h->dtype == CADET_FP32)
    return cuda_err(heads_forward_f32(h, w, (const float*)Hs, rows, n, logits, (float*)pre_out, ws, st),
                    "heads forward (fp32)");
  const int d = h->d_model, N = h->K * h->d_hidden;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  uint32_t* err = reinterpret_cast<uint32_t*>(p);
  void* Hr = p + 256;
  void* pre = pre_out ? pre_out : (void*)(p + 256 + a256((size_t)n * d * 2));
  // the towers' GEMMs run on fp16 operands (R27): H_r gathered as fp16, W1 converted once per call
  void* W1h = heads_w1h(ws, h, n);
  cudaError_t e = gather_rows_launch(Hs, rows, n, 1 << 30, d, Hr, err, st, 1);
  if (e == cudaSuccess) e = bf16_to_f16_launch(w->W1, W1h, (size_t)d * N, st);
  if (e == cudaSuccess) e = head_init_launch(logits, w->b2, n, h->K, st);
  if (e == cudaSuccess) {
    GemmProblem g = prob(n, N, d, act(Hr, n, d), w_fwd(W1h, d, N), EPI_HEAD);
    g.f16 = 1;
    g.epi.aux = pre;
    g.epi.b1 = w->b1;
    g.epi.w2 = w->w2;
    g.epi.logits = logits;
    g.epi.hd = h->d_hidden;
    g.epi.n_towers = h->K;
    e = gemm_launch(&g, 1, pick_bn(n, N), st);
  }
  return cuda_err(e, "heads forward");
}

cadet_status cadet_heads_backward(const cadet_head_config* h, const cadet_head_weights* w, const void* Hs,
                                  const int32_t* rows, int32_t n, int32_t T, const void* pre, const float* dz,
                                  int32_t accumulate, void* dHs, const cadet_head_grads* gr, void* ws, size_t ws_bytes,
                                  cadet_stream_t stream) {
  cadet_status s = check_head(h, w);
  if (s) return s;
  if (!Hs || !rows || !pre || !dz || !dHs || !gr || !gr->dW1 || !gr->db1 || !gr->dw2 || !gr->db2 || !ws || n < 0 ||
      T < 0) {
    set_error("heads_backward: null pointer");
    return CADET_E_ARG;
  }
  const size_t need = cadet_heads_workspace_bytes(h, n);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (h->dtype == CADET_FP32)
    return cuda_err(heads_backward_f32(h, w, (const float*)Hs, rows, n, T, (const float*)pre, dz, nullptr, nullptr,
                                       nullptr, nullptr, accumulate, (float*)dHs, gr, ws, st),
                    "heads backward (fp32)");
  const int d = h->d_model, N = h->K * h->d_hidden;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  uint32_t* err = reinterpret_cast<uint32_t*>(p);
  void* Hr = p + 256;
  void* dhid = p + 256 + a256((size_t)n * d * 2) + a256((size_t)n * N * 2);
  const ZeroSpan zs[5] = {{gr->dW1, (size_t)d * N * 4}, {gr->db1, (size_t)N * 4}, {gr->dw2, (size_t)N * 4},
                          {gr->db2, (size_t)h->K * 4}, {accumulate ? nullptr : dHs, (size_t)T * d * 2}};
  cudaError_t e = zero_many_launch(zs, 5, st);
  if (n == 0) return cuda_err(e, "heads backward");
  if (e == cudaSuccess)
    e = head_dhid_full_launch(pre, dz, w->w2, n, h->K, h->d_hidden, dhid, nullptr, gr->db1, gr->dw2, gr->db2, st);
  void* W1h = heads_w1h(ws, h, n);
  if (e == cudaSuccess && !h->rows_in_ws) {  // else ws holds the forward's fp16 H_r and W1 copies
    e = gather_rows_launch(Hs, rows, n, T, d, Hr, err, st, 1);
    if (e == cudaSuccess) e = bf16_to_f16_launch(w->W1, W1h, (size_t)d * N, st);
  }
  if (e == cudaSuccess) {  // dW1 = H_r^T dhid and dHs[rows] (+)= dhid W1^T (fp16 operands, R27): one launch
    const int bnw = pick_bn_wgrad(N);
    GemmProblem gw = prob(d, N, n, act_t(Hr, n, d), act_t(dhid, n, N), EPI_ATOMIC);
    gw.f16 = 1;
    gw.split_k = pick_split(d, N, bnw, n);
    gw.epi.out = gr->dW1;
    gw.epi.out_f32 = 1;
    GemmProblem g = prob(n, d, N, act(dhid, n, N), w_bwd(W1h, d, N), EPI_STORE);
    g.f16 = 1;
    g.epi.out = dHs;
    g.epi.ldo = d;
    g.epi.row_map = rows;
    g.epi.row_map_max = T;  // invalid rows (latched by the gather) never scatter out of bounds
    if (accumulate) {  // in place: dHs[rows] = dHs[rows] + (...)
      g.epi.resid = dHs;
      g.epi.resid_f32 = 0;
      g.epi.resid_at_out = 1;
    }
    e = gemm_launch2(&g, 1, pick_bn(n, d), &gw, 1, bnw, st);
  }
  return cuda_err(e, "heads backward");
}

cadet_status cadet_heads_loss_backward(const cadet_head_config* h, const cadet_head_weights* w, const void* Hs,
                                       const int32_t* rows, int32_t n, int32_t T, const float* logits,
                                       const void* pre, const int32_t* bucket, const float* label, float* loss_sum,
                                       void* dHs, const cadet_head_grads* gr, void* ws, size_t ws_bytes,
                                       cadet_stream_t stream) {
  cadet_status s = check_head(h, w);
  if (s) return s;
  if (!Hs || !rows || !logits || !pre || !bucket || !label || !loss_sum || !dHs || !gr || !gr->dW1 || !gr->db1 ||
      !gr->dw2 || !gr->db2 || !ws || n < 0 || T < 0) {
    set_error("heads_loss_backward: null pointer");
    return CADET_E_ARG;
  }
  const size_t need = cadet_heads_workspace_bytes(h, n);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (h->dtype == CADET_FP32)
    return cuda_err(heads_backward_f32(h, w, (const float*)Hs, rows, n, T, (const float*)pre, nullptr, logits, bucket,
                                       label, loss_sum, 0, (float*)dHs, gr, ws, st),
                    "heads backward (fp32)");
  const int d = h->d_model, N = h->K * h->d_hidden;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  uint32_t* err = reinterpret_cast<uint32_t*>(p);
  void* Hr = p + 256;
  void* dhid = p + 256 + a256((size_t)n * d * 2) + a256((size_t)n * N * 2);
  float* dz = reinterpret_cast<float*>(p + 256 + a256((size_t)n * d * 2) + 2 * a256((size_t)n * N * 2));
  const ZeroSpan zs[6] = {{loss_sum, 4},          {gr->dW1, (size_t)d * N * 4}, {gr->db1, (size_t)N * 4},
                          {gr->dw2, (size_t)N * 4}, {gr->db2, (size_t)h->K * 4}, {dHs, (size_t)T * d * 2}};
  cudaError_t e = zero_many_launch(zs, 6, st);
  if (n == 0) return cuda_err(e, "heads backward");
  if (e == cudaSuccess) e = head_dz_launch(logits, bucket, label, n, h->K, dz, loss_sum, gr->db2, err, st);
  if (e == cudaSuccess) e = head_dhid_launch(pre, dz, bucket, w->w2, n, h->K, h->d_hidden, dhid, nullptr, gr->db1, gr->dw2, st);
  void* W1h = heads_w1h(ws, h, n);
  if (e == cudaSuccess && !h->rows_in_ws) {  // else ws holds the forward's fp16 H_r and W1 copies
    e = gather_rows_launch(Hs, rows, n, T, d, Hr, err, st, 1);
    if (e == cudaSuccess) e = bf16_to_f16_launch(w->W1, W1h, (size_t)d * N, st);
  }
  if (e == cudaSuccess) {  // dW1 = H_r^T dhid and dHs[rows] (+)= dhid W1^T (fp16 operands, R27): one launch
    const int bnw = pick_bn_wgrad(N);
    GemmProblem gw = prob(d, N, n, act_t(Hr, n, d), act_t(dhid, n, N), EPI_ATOMIC);
    gw.f16 = 1;
    gw.split_k = pick_split(d, N, bnw, n);
    gw.epi.out = gr->dW1;
    gw.epi.out_f32 = 1;
    GemmProblem g = prob(n, d, N, act(dhid, n, N), w_bwd(W1h, d, N), EPI_STORE);
    g.f16 = 1;
    g.epi.out = dHs;
    g.epi.ldo = d;
    g.epi.row_map = rows;
    g.epi.row_map_max = T;  // invalid rows (latched by the gather) never scatter out of bounds
    e = gemm_launch2(&g, 1, pick_bn(n, d), &gw, 1, bnw, st);
  }
  return cuda_err(e, "heads backward");
}

// ------------------------------------------------------------------ NEXT-3: FFN of the CADET block (R33)
static cadet_status check_ffn(int T, int d, int m, const void* p0, const void* p1, const void* p2) {
  if (T < 0 || d <= 0 || m <= 0 || d % 32 || (T > 0 && !p0) || !p1 || !p2) {
    set_error("ffn: bad argument (d % 32 == 0, m >= 1, non-null operands)");
    return CADET_E_ARG;
  }
  return CADET_OK;
}

size_t cadet_ffn_workspace_bytes(int32_t T, int32_t d, int32_t m) { return a256((size_t)T * d * m * 2); }

cadet_status cadet_ffn_forward(const void* X, const void* W1, const void* W2, const void* resid, int32_t T, int32_t d,
                               int32_t m, void* Y, void* U, void* G, cadet_stream_t stream) {
  cadet_status s = check_ffn(T, d, m, X, W1, W2);
  if (s) return s;
  if (T == 0) return CADET_OK;
  if (!Y || !U || !G) return check_ffn(T, d, m, nullptr, nullptr, nullptr);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int N = d * m;
  // U = X W1 (saved pre-activation), G = GELU(U): one GEMM, the activation in its epilogue
  GemmProblem g1 = prob(T, N, d, act(X, T, d), w_fwd(W1, d, N), EPI_GELU);
  g1.epi.out = G;
  g1.epi.aux = U;
  cudaError_t e = gemm_launch(&g1, 1, pick_bn(T, N), st);
  if (e == cudaSuccess) {  // Y = G W2 (+ resid)
    GemmProblem g2 = prob(T, d, N, act(G, T, N), w_fwd(W2, N, d), EPI_STORE);
    g2.epi.out = Y;
    g2.epi.resid = resid;
    e = gemm_launch(&g2, 1, pick_bn(T, d), st);
  }
  return cuda_err(e, "ffn forward");
}

cadet_status cadet_ffn_backward(const void* X, const void* W1, const void* W2, const void* U, const void* G,
                                const void* dY, const void* dresid, int32_t T, int32_t d, int32_t m, void* dX,
                                float* dW1, float* dW2, void* ws, size_t ws_bytes, cadet_stream_t stream) {
  cadet_status s = check_ffn(T, d, m, X, W1, W2);
  if (s) return s;
  if (!dW1 || !dW2 || (T > 0 && (!U || !G || !dY || !dX || !ws))) return check_ffn(T, d, m, nullptr, nullptr, nullptr);
  const size_t need = cadet_ffn_workspace_bytes(T, d, m);
  if (ws_bytes < need) return ws_err(ws_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int N = d * m;
  const ZeroSpan zs[2] = {{dW1, (size_t)d * N * 4}, {dW2, (size_t)N * d * 4}};
  cudaError_t e = zero_many_launch(zs, 2, st);
  if (T == 0) return cuda_err(e, "ffn backward");
  void* dU = ws;
  if (e == cudaSuccess) {  // dU = (dY W2^T) * GELU'(U)  with  dW2 = G^T dY  in the same launch
    GemmProblem g = prob(T, N, d, act(dY, T, d), w_bwd(W2, N, d), EPI_GELU_BWD);
    g.epi.out = dU;
    g.epi.aux = const_cast<void*>(U);
    const int bnw = pick_bn_wgrad(d);
    GemmProblem gw = wgrad(G, dY, dW2, T, N, d, bnw);
    e = gemm_launch2(&g, 1, pick_bn(T, N), &gw, 1, bnw, st);
  }
  if (e == cudaSuccess) {  // dX = dU W1^T (+ dresid)  with  dW1 = X^T dU
    GemmProblem g = prob(T, d, N, act(dU, T, N), w_bwd(W1, d, N), EPI_STORE);
    g.epi.out = dX;
    g.epi.resid = dresid;
    const int bnw = pick_bn_wgrad(N);
    GemmProblem gw = wgrad(X, dU, dW1, T, d, N, bnw);
    e = gemm_launch2(&g, 1, pick_bn(T, d), &gw, 1, bnw, st);
  }
  return cuda_err(e, "ffn backward");
}

}  // extern "C"

namespace cadet {
// cadet_mask_plan's extension (plan_ready = 2): formerly the per-step RoPE table; RoPE angles are now
// evaluated on the fly, so there is nothing to prepare.
cudaError_t layer_plan_extras(const cadet_attn_config*, const cadet_batch*, void*, size_t, cudaStream_t) {
  return cudaSuccess;
}
}  // namespace cadet
