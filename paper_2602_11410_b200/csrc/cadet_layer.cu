// libcadet host side, attention core and full gated layer (rows A2-A12).
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include "../../include/cadet.h"
#include "gemm.cuh"
#include "layer.cuh"

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
  if ((s = cadet_mask_plan(cfg, b, ws, ws_bytes, stream))) return s;
  PlanView v = plan_carve(ws, b->n_seqs, b->total_tokens, b->total_tokens);
  AttnParams p = attn_params(cfg, b, v);
  p.O = O;
  p.lse = lse;
  const int T = b->total_tokens, d = cfg->d_model;
  // pad rows: O = 0, LSE = 0 (R17)
  cudaError_t e = zero_pad_rows_launch(O, d * (cfg->out_f32 ? 4 : 2), T, b->cu_seqlens, b->n_seqs, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(lse, 0, sizeof(float) * (size_t)T * cfg->n_heads, st);
  if (e == cudaSuccess) e = attn_fwd_launch(Qr, Kr, V, p, st);
  return cuda_err(e, "attention forward");
}

}  // extern "C"
