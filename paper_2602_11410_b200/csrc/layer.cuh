// Internal declarations shared by the host-side layer code.
#pragma once
#include <cuda_runtime.h>
#include "../../include/cadet.h"
#include "attn_common.cuh"
#include "plan.cuh"

namespace cadet {
cadet_status check_cfg(const cadet_attn_config* c);
cadet_status check_batch(const cadet_batch* b, const cadet_attn_config* c);
PlanArgs plan_args(const cadet_attn_config* c, const cadet_batch* b);
void set_error(const char* msg);

cudaError_t attn_fwd_launch(const void* Qr, const void* Kr, const void* V, const AttnParams& p, cudaStream_t st);
cudaError_t attn_bwd_launch(const void* Qr, const void* Kr, const void* V, const void* dO, const AttnParams& p,
                            cudaStream_t st);
cudaError_t attn_bwd_pre_launch(const void* O, const void* dO, float* D, float* dQacc, int T, int H, int hd,
                                cudaStream_t st);
cudaError_t layer_plan_extras(const cadet_attn_config* cfg, const cadet_batch* b, void* ws, size_t ws_bytes,
                              cudaStream_t st);
}  // namespace cadet
