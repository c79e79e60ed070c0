// CADET_FP32 parity mode (fp32.cu): 3xTF32 GEMMs, exact fp32 elementwise and attention kernels.
#pragma once
#include <cuda_runtime.h>
#include "../../include/cadet.h"
#include "gemm.cuh"
#include "plan.cuh"

namespace cadet {
size_t gemm3x_scratch_bytes(int M, int N, int K);
cudaError_t gemm3x(int M, int N, int K, const float* A, int a_t, const float* B, int b_t, float* C,
                   const float* resid, void* scratch, cudaStream_t st);
size_t f32_saved_bytes(const cadet_attn_config* c, int T);
size_t f32_layer_ws_bytes(const cadet_attn_config* c, int n, int T);
cudaError_t attn_fwd_f32(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v, const float* Qr,
                         const float* Kr, const float* V, float* O, float* lse, cudaStream_t st);
cudaError_t attn_bwd_f32(const cadet_attn_config* c, const cadet_batch* b, const PlanView& v, const float* Qr,
                         const float* Kr, const float* V, const float* O, const float* lse, const float* dO, float* D,
                         float* dQ, float* dK, float* dV, cudaStream_t st);
cudaError_t layer_forward_f32(const cadet_attn_config* c, const cadet_batch* b, const cadet_attn_weights* w,
                              const float* X, float* Y, const float* resid, void* saved, void* ws, cudaStream_t st);
cudaError_t layer_backward_f32(const cadet_attn_config* c, const cadet_batch* b, const cadet_attn_weights* w,
                               const float* X, const void* saved, const float* dY, float* dX, const float* dresid,
                               const cadet_attn_grads* g, void* ws, cudaStream_t st, void* const* grad_events);
size_t f32_heads_ws_bytes(const cadet_head_config* h, int n);
cudaError_t heads_forward_f32(const cadet_head_config* h, const cadet_head_weights* w, const float* Hs,
                              const int32_t* rows, int n, float* logits, float* pre_out, void* ws, cudaStream_t st);
cudaError_t heads_backward_f32(const cadet_head_config* h, const cadet_head_weights* w, const float* Hs,
                               const int32_t* rows, int n, int T, const float* pre, const float* dz_in,
                               const float* logits, const int32_t* bucket, const float* label, float* loss,
                               int accumulate, float* dHs, const cadet_head_grads* g, void* ws, cudaStream_t st);
}  // namespace cadet
