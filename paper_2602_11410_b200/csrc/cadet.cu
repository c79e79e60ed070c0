// libcadet host side: the C ABI of include/cadet.h — validation, workspace carving,
// TMA descriptor encoding and launch sequencing.  Every call is asynchronous on the
// caller's stream; nothing here allocates device memory.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <string>

#include "../../include/cadet.h"
#include "fp32.cuh"
#include "gemm.cuh"
#include "layer.cuh"
#include "plan.cuh"
#include "misc.cuh"

using namespace cadet;

namespace {
thread_local std::string g_err;

cadet_status fail(cadet_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
cadet_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CADET_OK;
  return fail(CADET_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

namespace cadet {
cadet_status check_cfg(const cadet_attn_config* c) {
  if (!c) return fail(CADET_E_ARG, "null config");
  if (c->d_model <= 0 || c->n_heads <= 0 || c->d_model % c->n_heads)
    return fail(CADET_E_ARG, "d_model %d not divisible by n_heads %d", c->d_model, c->n_heads);
  const int hd = c->d_model / c->n_heads;
  if (c->head_dim != hd) return fail(CADET_E_ARG, "head_dim %d != d_model / n_heads = %d", c->head_dim, hd);
  // the kernels are built and parity-tested for these head dims (88 runs padded to 96 by TMA zero-fill)
  if (hd != 32 && hd != 64 && hd != 88 && hd != 96 && hd != 128)
    return fail(CADET_E_ARG, "head_dim %d must be one of 32, 64, 88, 96, 128", hd);
  // per-row head sums (attn_bwd_pre_kernel) and the per-head plan arrays hold at most 128 heads
  if (c->n_heads > 128) return fail(CADET_E_ARG, "n_heads %d > 128", c->n_heads);
  if (c->d_model % 32) return fail(CADET_E_ARG, "d_model %d must be a multiple of 32", c->d_model);
  if (c->dtype != CADET_BF16 && c->dtype != CADET_FP32) return fail(CADET_E_ARG, "dtype %d unknown", c->dtype);
  if (c->deterministic && c->dtype != CADET_BF16)
    return fail(CADET_E_UNSUPPORTED, "deterministic mode: bf16 layer only (the fp32 parity mode reduces with atomics)");
  if (c->delta_delay_ms < 0 || c->delta_cand_ms < 0) return fail(CADET_E_ARG, "negative delta");
  if (c->use_rope && (c->rope_delta_t_max_ms <= 0 || c->rope_phi_min <= 0 || c->rope_base <= 1.0))
    return fail(CADET_E_ARG, "invalid RoPE constants");
  return CADET_OK;
}
cadet_status check_batch(const cadet_batch* b, const cadet_attn_config* c) {
  if (!b) return fail(CADET_E_ARG, "null batch");
  if (b->n_seqs < 0 || b->total_tokens < 0 || b->max_seqlen <= 0) return fail(CADET_E_ARG, "bad batch scalars");
  if (b->n_seqs > 0 && (!b->cu_seqlens || !b->timestamps_ms)) return fail(CADET_E_ARG, "null cu_seqlens/timestamps");
  if (c && (c->mask_flags & CADET_MASK_SESSION) && !b->session_ids)
    return fail(CADET_E_ARG, "CADET_MASK_SESSION needs session_ids");
  return CADET_OK;
}
PlanArgs plan_args(const cadet_attn_config* c, const cadet_batch* b) {
  PlanArgs a;
  a.n = b->n_seqs;
  a.T = b->total_tokens;
  a.max_seqlen = b->max_seqlen;
  a.mask_flags = c->mask_flags;
  a.delta_ctx = c->delta_delay_ms;
  a.delta_cand = c->delta_cand_ms;
  a.cu = b->cu_seqlens;
  a.t = b->timestamps_ms;
  a.sess = b->session_ids;
  a.ncand = b->n_candidates;
  a.nstatic = b->n_static;
  a.flags = b->token_flags;
  a.rope_phi_min = c->rope_phi_min;
  a.rope_dt_max = (double)c->rope_delta_t_max_ms;
  a.rope_base = c->rope_base;
  a.head_dim = c->head_dim;
  return a;
}
void set_error(const char* msg) { g_err = msg; }
}  // namespace cadet

extern "C" {

int32_t cadet_abi_version(void) { return CADET_ABI_VERSION; }
const char* cadet_last_error(void) { return g_err.c_str(); }

const char* cadet_status_string(cadet_status s) {
  switch (s) {
    case CADET_OK: return "CADET_OK";
    case CADET_E_ARG: return "CADET_E_ARG";
    case CADET_E_OFFSETS: return "CADET_E_OFFSETS";
    case CADET_E_ORDER: return "CADET_E_ORDER";
    case CADET_E_TOO_LONG: return "CADET_E_TOO_LONG";
    case CADET_E_CAND: return "CADET_E_CAND";
    case CADET_E_BUCKET: return "CADET_E_BUCKET";
    case CADET_E_NONFINITE: return "CADET_E_NONFINITE";
    case CADET_E_WORKSPACE: return "CADET_E_WORKSPACE";
    case CADET_E_UNSUPPORTED: return "CADET_E_UNSUPPORTED";
    case CADET_E_CUDA: return "CADET_E_CUDA";
  }
  return "CADET_E_UNKNOWN";
}

void cadet_default_attn_config(cadet_attn_config* c, int32_t d_model, int32_t n_heads) {
  memset(c, 0, sizeof(*c));
  c->d_model = d_model;
  c->n_heads = n_heads;
  c->head_dim = n_heads > 0 ? d_model / n_heads : 0;
  c->dtype = CADET_BF16;
  c->mask_flags = CADET_MASK_TIME;
  c->use_rope = c->use_rep_gate = c->use_int_gate = c->use_out_proj = 1;
  c->delta_delay_ms = 3600000LL;
  c->delta_cand_ms = 0;
  c->rope_delta_t_max_ms = 31536000000LL;
  c->rope_phi_min = 1e-4;
  c->rope_base = 600000.0;
}

void cadet_tile_shape(int32_t* bm, int32_t* bn) {
  if (bm) *bm = TILE;
  if (bn) *bn = TILE;
}

size_t cadet_plan_workspace_bytes(int32_t n_seqs, int32_t T) {
  // max_seqlen is only needed for the cost histogram; bound it by T.
  return plan_bytes(n_seqs, T, T > 0 ? T : 1) + a256((size_t)4 * T * 128 /* D for core bwd, H <= 128 */);
}

cadet_status cadet_mask_plan(const cadet_attn_config* cfg, const cadet_batch* b, void* ws, size_t ws_bytes,
                             cadet_stream_t stream) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!ws) return fail(CADET_E_ARG, "null workspace");
  if (ws_bytes < plan_bytes(b->n_seqs, b->total_tokens, b->total_tokens))
    return fail(CADET_E_WORKSPACE, "workspace %zu < %zu", ws_bytes, plan_bytes(b->n_seqs, b->total_tokens, b->total_tokens));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PlanView v = plan_carve(ws, b->n_seqs, b->total_tokens, b->total_tokens);
  cudaError_t e = plan_launch(plan_args(cfg, b), v, st);
  if (e == cudaSuccess) e = layer_plan_extras(cfg, b, ws, ws_bytes, st);  // RoPE table (plan_ready = 2)
  return cuda_check(e, "mask plan");
}

cadet_status cadet_mask_export(const cadet_attn_config* cfg, const cadet_batch* b, const void* ws, int32_t* kv_end,
                               int8_t* tile_class, int64_t tile_class_cap, int64_t* n_pairs, cadet_stream_t stream) {
  cadet_status s = check_cfg(cfg);
  if (s) return s;
  if ((s = check_batch(b, cfg))) return s;
  if (!ws) return fail(CADET_E_ARG, "null workspace");
  PlanView v = plan_carve(const_cast<void*>(ws), b->n_seqs, b->total_tokens, b->total_tokens);
  return cuda_check(plan_export_launch(plan_args(cfg, b), v, kv_end, tile_class, tile_class_cap, n_pairs,
                                       reinterpret_cast<cudaStream_t>(stream)),
                    "mask export");
}

cadet_status cadet_poll(void* ws, cadet_stream_t stream) {
  if (!ws) return fail(CADET_E_ARG, "null workspace");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint32_t word = 0;
  cudaError_t e = cudaMemcpyAsync(&word, ws, sizeof(word), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_check(e, "poll");
  if (word) {
    e = cudaMemsetAsync(ws, 0, sizeof(word), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (word & ERRBIT_OFFSETS) return fail(CADET_E_OFFSETS, "invalid cu_seqlens (device)");
  if (word & ERRBIT_ORDER) return fail(CADET_E_ORDER, "timestamps/session ids decrease inside a sequence (device)");
  if (word & ERRBIT_TOO_LONG) return fail(CADET_E_TOO_LONG, "sequence longer than max_seqlen / budget (device)");
  if (word & ERRBIT_CAND) return fail(CADET_E_CAND, "n_candidates out of range (device)");
  if (word & ERRBIT_BUCKET) return fail(CADET_E_BUCKET, "bucket / position / embedding id out of range (device)");
  if (word & ERRBIT_NONFINITE) return fail(CADET_E_NONFINITE, "non-finite loss (device)");
  if (word & ERRBIT_CAPACITY) return fail(CADET_E_WORKSPACE, "output capacity too small (device)");
  return CADET_OK;
}

cadet_status cadet_chunk(const int32_t* cu_in, int32_t n_in, int32_t L_chunk, int32_t* cu_out, int32_t cap,
                         int32_t* n_out, void* ws, cadet_stream_t stream) {
  if (!cu_in || !cu_out || !n_out || n_in < 0 || L_chunk <= 0 || cap < 1 || !ws) return fail(CADET_E_ARG, "cadet_chunk args");
  return cuda_check(chunk_launch(cu_in, n_in, L_chunk, cu_out, cap, n_out, reinterpret_cast<uint32_t*>(ws),
                                 reinterpret_cast<cudaStream_t>(stream)),
                    "chunk");
}

size_t cadet_pack_workspace_bytes(int32_t B) { (void)B; return 256; }

cadet_status cadet_pack(const void* src, const int64_t* src_row, const int32_t* lens, int32_t B, int32_t d,
                        int32_t budget, const int64_t* t_src, const int32_t* s_src, void* packed, int64_t* t_out,
                        int32_t* s_out, int32_t* cu_out, int32_t* n_packed, void* ws, size_t ws_bytes,
                        cadet_stream_t stream) {
  if (!lens || (!src != !packed) || !cu_out || !n_packed || B < 0 || d <= 0 || budget <= 0 || !ws)
    return fail(CADET_E_ARG, "cadet_pack args");
  if (d % 8) return fail(CADET_E_ARG, "d must be a multiple of 8");
  if (ws_bytes < 256) return fail(CADET_E_WORKSPACE, "pack workspace");
  return cuda_check(pack_launch(src, src_row, lens, B, d, budget, t_src, s_src, packed, t_out, s_out, cu_out,
                                n_packed, reinterpret_cast<uint32_t*>(ws), reinterpret_cast<cudaStream_t>(stream)),
                    "pack");
}

cadet_status cadet_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t a_mn, const void* B, int32_t b_mn,
                        void* C, int32_t c_f32, const void* resid, cadet_stream_t stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0) return fail(CADET_E_ARG, "cadet_gemm args");
  if (N % 32 || K % 8 || (a_mn && M % 8)) return fail(CADET_E_ARG, "cadet_gemm shape constraints");
  GemmProblem g;
  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.nseg = 1;
  g.K[0] = K;
  g.A[0] = a_mn ? OperandDesc{A, K, M, 1} : OperandDesc{A, M, K, 0};
  g.B[0] = b_mn ? OperandDesc{B, K, N, 1} : OperandDesc{B, N, K, 0};
  g.split_k = 1;
  g.epi.mode = EPI_STORE;
  g.epi.out = C;
  g.epi.out_f32 = c_f32;
  g.epi.ldo = N;
  g.epi.resid = resid;
  g.epi.resid_f32 = c_f32;
  const int bn = (N % 256 == 0 && M >= 256) ? 256 : 128;  // 256 -> CTA-pair (cta_group::2) kernel
  return cuda_check(gemm_launch(&g, 1, bn, reinterpret_cast<cudaStream_t>(stream)), "gemm");
}

cadet_status cadet_bucketize(const int32_t* raw_position, int32_t n, const int32_t* boundaries_h, int32_t nb,
                             int32_t* bucket, void* ws, cadet_stream_t stream) {
  if (n < 0 || (n > 0 && (!raw_position || !bucket)) || !ws || !boundaries_h) return fail(CADET_E_ARG, "cadet_bucketize args");
  if (nb < 1 || nb > 32) return fail(CADET_E_ARG, "cadet_bucketize: 1 <= nb <= 32 boundaries");
  Bounds bd;
  memset(&bd, 0, sizeof(bd));
  bd.nb = nb;
  for (int j = 0; j < nb; ++j) {
    if (j > 0 && boundaries_h[j] <= boundaries_h[j - 1]) return fail(CADET_E_ARG, "boundaries not strictly increasing");
    bd.b[j] = boundaries_h[j];
  }
  return cuda_check(bucketize_launch(raw_position, n, bd, bucket, reinterpret_cast<uint32_t*>(ws),
                                     reinterpret_cast<cudaStream_t>(stream)),
                    "bucketize");
}

static cadet_status check_embed(const cadet_embed_config* c) {
  if (!c || c->n_tables < 1 || c->n_tables > CADET_EMBED_MAX_TABLES || c->d_model <= 0 || c->d_model % 8)
    return fail(CADET_E_ARG, "embed: 1 <= n_tables <= 8, d_model % 8 == 0");
  for (int f = 0; f < c->n_tables; ++f)
    if (c->vocab[f] < 1) return fail(CADET_E_ARG, "embed: vocab[%d] < 1", f);
  return CADET_OK;
}
size_t cadet_embed_workspace_bytes(const cadet_embed_config* c) { return check_embed(c) ? 0 : embed_ws_bytes(c); }
cadet_status cadet_embed_forward(const cadet_embed_config* c, const void* const* tables, const int32_t* ids, int32_t T,
                                 const int32_t* n_valid, void* X, void* ws, size_t ws_bytes, cadet_stream_t stream) {
  cadet_status s = check_embed(c);
  if (s) return s;
  if (T < 0 || !tables || (T > 0 && (!ids || !X)) || !ws) return fail(CADET_E_ARG, "embed_forward: null pointer");
  for (int f = 0; f < c->n_tables; ++f)
    if (!tables[f]) return fail(CADET_E_ARG, "embed_forward: null table %d", f);
  if (ws_bytes < embed_ws_bytes(c)) return fail(CADET_E_WORKSPACE, "embed workspace too small");
  return cuda_check(embed_forward_launch(c, tables, ids, T, n_valid, X, ws, reinterpret_cast<cudaStream_t>(stream)),
                    "embed forward");
}
cadet_status cadet_embed_backward(const cadet_embed_config* c, const int32_t* ids, int32_t T, const int32_t* n_valid,
                                  const void* dX, float* const* dtables, void* ws, size_t ws_bytes,
                                  cadet_stream_t stream) {
  cadet_status s = check_embed(c);
  if (s) return s;
  if (T < 0 || !dtables || (T > 0 && (!ids || !dX)) || !ws) return fail(CADET_E_ARG, "embed_backward: null pointer");
  for (int f = 0; f < c->n_tables; ++f)
    if (!dtables[f]) return fail(CADET_E_ARG, "embed_backward: null gradient %d", f);
  if (ws_bytes < embed_ws_bytes(c)) return fail(CADET_E_WORKSPACE, "embed workspace too small");
  return cuda_check(embed_backward_launch(c, ids, T, n_valid, dX, dtables, ws, reinterpret_cast<cudaStream_t>(stream)),
                    "embed backward");
}

size_t cadet_gemm_fp32_workspace_bytes(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  return gemm3x_scratch_bytes(M, N, K);
}

cadet_status cadet_gemm_fp32(int32_t M, int32_t N, int32_t K, const float* A, int32_t a_t, const float* B,
                             int32_t b_t, float* C, const float* resid, void* ws, size_t ws_bytes,
                             cadet_stream_t stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0 || (!ws && ws_bytes)) return fail(CADET_E_ARG, "cadet_gemm_fp32 args");
  if (N % 32) return fail(CADET_E_ARG, "cadet_gemm_fp32: N %% 32 != 0");
  const size_t need = gemm3x_scratch_bytes(M, N, K);
  if (ws_bytes < need) return fail(CADET_E_WORKSPACE, "workspace %zu < required %zu", ws_bytes, need);
  return cuda_check(gemm3x(M, N, K, A, a_t, B, b_t, C, resid, ws, reinterpret_cast<cudaStream_t>(stream)),
                    "gemm fp32");
}

}  // extern "C"
