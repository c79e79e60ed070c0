// Host/device interface of the tcgen05 GEMM with CADET fused epilogues.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cadet {

enum EpiMode : int32_t {
  EPI_STORE = 0,      // out = acc (+ resid)                                        (A3, A6, A9, A12 ...)
  EPI_GATE = 1,       // out = src * sigma(acc); aux = acc                          (Eq. 4)
  // 2: formerly the fused gate + RoPE epilogue (A4 now stores Z and runs gate_rope_fwd_kernel)
  EPI_GATE_BWD = 3,   // g = sigma(aux); out = acc*src*g*(1-g); out2 = acc*g + resid (A12)
  EPI_ATOMIC = 4,     // out += acc (fp32 red.add; split-K weight gradients)
  EPI_HEAD = 5,       // pre = acc + b1; aux = pre; logits[row, n/dh] += relu(pre).w2 (Eq. 8)
  EPI_GELU = 6,       // NEXT-3 FFN: aux = acc (pre-activation); out = GELU(acc) (R33)
  EPI_GELU_BWD = 7,   // NEXT-3 FFN: out = acc * GELU'(aux)
};
// Not a mode: the bit of the compile-time mode set that enables the parity taps (tap / tap2 below).
constexpr int EPI_TAPS = 8;

struct EpiParams {
  int32_t mode;
  int32_t out_f32;  // out dtype: 1 = fp32, 0 = bf16
  int32_t ldo;      // leading dim of out / resid / src / aux (elements)
  int32_t resid_f32;
  int32_t aux_f32;
  int32_t hd;       // head dim (EPI_STORE dot_out) or head hidden width dh (EPI_HEAD)
  int32_t n_towers; // EPI_HEAD: K
  void* out;
  const void* resid;
  const void* src;   // bf16
  void* aux;
  void* out2;        // EPI_GATE_BWD second output: fp32 if out2_f32 else bf16
  int32_t out2_f32;
  const int32_t* row_map;  // optional output-row remap (scatter); < 0 = drop row
  int32_t resid_at_out;    // row_map stores: resid read at the output row (in-place accumulate)
  int32_t row_map_max;     // row_map stores: rows >= this are dropped (0 = no bound)
  // EPI_STORE extra (A9 -> A10 preprocess): dot_out[(n / hd) * dot_T + row] += sum over the slice's
  // columns of acc * dot_src (bf16, same layout as out), per head (hd >= 32); dot_out zeroed
  const void* dot_src;
  float* dot_out;
  int32_t dot_T;
  // parity taps (SURVEY 8(c) protocol iii, cadet_attn_stage_views): fp32 copies, [rows][ldo], of the
  // value stored to out (tap) and of aux (EPI_GATE: Z) / out2 (EPI_GATE_BWD: r) (tap2) BEFORE their
  // bf16 rounding; null = off.  Only the warp-cooperative epilogue (no row_map) writes them.
  float* tap;
  float* tap2;
  // EPI_ATOMIC in deterministic mode (cfg.deterministic): split ks stores its fp32 partial at
  // out + ks * split_stride (plain stores, no atomics); a fixed-order reduction sums the slabs after
  int64_t split_stride;
  // heads (EPI_HEAD)
  const float* b1;
  const float* w2;
  float* logits;
};

struct OperandDesc {
  const void* ptr;  // bf16 (fp32 for tf32 problems), row-major storage [rows][cols] (row stride ld if > 0)
  int32_t rows, cols;
  int32_t mn_major; // 0: storage is [MN][K] (K-major); 1: storage is [K][MN] (MN-major)
  int32_t ld;       // row stride in elements (0 = cols)
};

constexpr int GEMM_MAX_PROB = 4;
constexpr int GEMM_MAX_SEG = 3;

struct GemmProblem {
  int32_t M, N;
  int32_t nseg;
  int32_t K[GEMM_MAX_SEG];
  OperandDesc A[GEMM_MAX_SEG], B[GEMM_MAX_SEG];
  int32_t split_k;   // > 1 only with EPI_ATOMIC
  int32_t f16;       // operands are fp16 instead of bf16 (both A and B)
  int32_t tf32;      // operands are fp32 (both K-major), multiplied as TF32 (kind::tf32; CADET_FP32 mode)
  EpiParams epi;
};

// Enqueue: returns cudaError_t.  BN chosen by the host (128 or 256).
cudaError_t gemm_launch(const GemmProblem* probs, int nprob, int bn, cudaStream_t stream);

}  // namespace cadet
