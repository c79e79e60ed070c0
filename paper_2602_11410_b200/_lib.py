"""ctypes binding of libcadet (include/cadet.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  There is no fallback: if libcadet.so is
missing or a call fails, an exception is raised."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CADET_LIB") or os.path.join(HERE, "libcadet.so")  # CADET_LIB: A/B builds

CADET_MASK_TIME = 1
CADET_MASK_SESSION = 2
CADET_MASK_PAIR_PREV = 4

# cadet_attn_stage_views indices (include/cadet.h)
TAP_NAMES = ["Zx", "Xt", "Q", "K", "V", "Zq", "Zk", "Qr", "Kr", "O", "Y", "dO", "dQr", "dKr", "dV", "uq", "rq", "uk",
             "rk", "dQ", "dK", "ux", "rx", "dX"]
CADET_N_TAPS = 24
WS_NAMES = ["dO", "dQr", "dKr", "dV", "uq", "rq", "uk", "rk", "dQ", "dK", "ux", "rx"]
CADET_WS_DO = 32
CADET_WS_D = 44
CADET_N_VIEWS = 45

STATUS = {0: "CADET_OK", 1: "CADET_E_ARG", 2: "CADET_E_OFFSETS", 3: "CADET_E_ORDER", 4: "CADET_E_TOO_LONG",
          5: "CADET_E_CAND", 6: "CADET_E_BUCKET", 7: "CADET_E_NONFINITE", 8: "CADET_E_WORKSPACE",
          9: "CADET_E_UNSUPPORTED", 10: "CADET_E_CUDA"}


class CadetError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class AttnConfig(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("n_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("mask_flags", C.c_int32), ("out_f32", C.c_int32), ("use_rope", C.c_int32),
                ("use_rep_gate", C.c_int32), ("use_int_gate", C.c_int32), ("use_out_proj", C.c_int32),
                ("deterministic", C.c_int32), ("plan_ready", C.c_int32), ("delta_delay_ms", C.c_int64),
                ("delta_cand_ms", C.c_int64), ("rope_delta_t_max_ms", C.c_int64), ("rope_phi_min", C.c_double),
                ("rope_base", C.c_double)]


class BatchStruct(C.Structure):
    _fields_ = [("n_seqs", C.c_int32), ("total_tokens", C.c_int32), ("max_seqlen", C.c_int32),
                ("reserved0", C.c_int32), ("cu_seqlens", C.c_void_p), ("timestamps_ms", C.c_void_p),
                ("session_ids", C.c_void_p), ("n_candidates", C.c_void_p), ("n_static", C.c_void_p),
                ("token_flags", C.c_void_p)]


class AttnWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("W_xg", "W_q", "W_k", "W_v", "W_qg", "W_kg", "W_o")]


class AttnGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("dW_xg", "dW_q", "dW_k", "dW_v", "dW_qg", "dW_kg", "dW_o")]


class LossConfig(C.Structure):
    _fields_ = [("J", C.c_int32), ("aux_kind", C.c_int32 * 8), ("lambda_ctx", C.c_float), ("lambda_pair", C.c_float),
                ("lambda_aux", C.c_float * 8)]


class EmbedConfig(C.Structure):
    _fields_ = [("n_tables", C.c_int32), ("d_model", C.c_int32), ("vocab", C.c_int32 * 8)]


class AdamWConfig(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float)]


class HeadConfig(C.Structure):
    _fields_ = [("K", C.c_int32), ("d_model", C.c_int32), ("d_hidden", C.c_int32), ("dtype", C.c_int32),
                ("rows_in_ws", C.c_int32)]


class HeadWeights(C.Structure):
    _fields_ = [("W1", C.c_void_p), ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p)]


class HeadGrads(C.Structure):
    _fields_ = [("dW1", C.c_void_p), ("db1", C.c_void_p), ("dw2", C.c_void_p), ("db2", C.c_void_p)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
SZ = C.c_size_t
PCFG = C.POINTER(AttnConfig)
PB = C.POINTER(BatchStruct)

# name -> (restype, argtypes); the binding exports exactly these names (tests check the .so exports them).
SIGNATURES = {
    "cadet_abi_version": (I32, []),
    "cadet_last_error": (C.c_char_p, []),
    "cadet_status_string": (C.c_char_p, [I32]),
    "cadet_default_attn_config": (None, [PCFG, I32, I32]),
    "cadet_tile_shape": (None, [C.POINTER(I32), C.POINTER(I32)]),
    "cadet_plan_workspace_bytes": (SZ, [I32, I32]),
    "cadet_attn_workspace_bytes": (SZ, [PCFG, I32, I32]),
    "cadet_attn_saved_bytes": (SZ, [PCFG, I32]),
    "cadet_attn_bwd_ds_bytes": (SZ, [C.POINTER(AttnConfig), I32, I32, I32]),
    "cadet_heads_workspace_bytes": (SZ, [C.POINTER(HeadConfig), I32]),
    "cadet_attn_stage_views": (I32, [PCFG, I32, I32, P, SZ, C.POINTER(C.c_void_p)]),
    "cadet_mask_plan": (I32, [PCFG, PB, P, SZ, P]),
    "cadet_mask_export": (I32, [PCFG, PB, P, P, P, I64, P, P]),
    "cadet_attn_core_forward": (I32, [PCFG, PB, P, P, P, P, P, P, SZ, P]),
    "cadet_attn_core_backward": (I32, [PCFG, PB, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "cadet_attn_forward": (I32, [PCFG, PB, C.POINTER(AttnWeights), P, P, P, P, P, SZ, P]),
    "cadet_attn_backward": (I32, [PCFG, PB, C.POINTER(AttnWeights), P, P, P, P, P, C.POINTER(AttnGrads), P, SZ, P]),
    "cadet_attn_backward_ev": (I32, [PCFG, PB, C.POINTER(AttnWeights), P, P, P, P, P, C.POINTER(AttnGrads), P, SZ, P,
                                     C.POINTER(C.c_void_p)]),
    "cadet_heads_forward": (I32, [C.POINTER(HeadConfig), C.POINTER(HeadWeights), P, P, I32, P, P, P, SZ, P]),
    "cadet_heads_loss_backward": (I32, [C.POINTER(HeadConfig), C.POINTER(HeadWeights), P, P, I32, I32, P, P, P, P,
                                        P, P, C.POINTER(HeadGrads), P, SZ, P]),
    "cadet_default_loss_config": (None, [C.POINTER(LossConfig), I32]),
    "cadet_routed_logits": (I32, [P, I32, P, I32, P, P]),
    "cadet_pairwise_workspace_bytes": (SZ, [I32, I32]),
    "cadet_pairwise_loss": (I32, [P, P, I32, P, P, I32, P, P, P, SZ, P]),
    "cadet_full_loss_grads": (I32, [C.POINTER(LossConfig), P, I32, P, P, P, P, P, P, I32, P, P, P, P]),
    "cadet_heads_backward": (I32, [C.POINTER(HeadConfig), C.POINTER(HeadWeights), P, P, I32, I32, P, P, I32, P,
                                   C.POINTER(HeadGrads), P, SZ, P]),
    "cadet_rmsnorm_forward": (I32, [P, P, I32, I32, P, P, P]),
    "cadet_rmsnorm_backward": (I32, [P, P, P, P, P, I32, I32, P, P, P]),
    "cadet_ffn_workspace_bytes": (SZ, [I32, I32, I32]),
    "cadet_ffn_forward": (I32, [P, P, P, P, I32, I32, I32, P, P, P, P]),
    "cadet_ffn_backward": (I32, [P, P, P, P, P, P, P, I32, I32, I32, P, P, P, P, SZ, P]),
    "cadet_embed_workspace_bytes": (SZ, [C.POINTER(EmbedConfig)]),
    "cadet_embed_forward": (I32, [C.POINTER(EmbedConfig), C.POINTER(C.c_void_p), P, I32, P, P, P, SZ, P]),
    "cadet_embed_backward": (I32, [C.POINTER(EmbedConfig), P, I32, P, P, C.POINTER(C.c_void_p), P, SZ, P]),
    "cadet_default_adamw_config": (None, [C.POINTER(AdamWConfig)]),
    "cadet_adamw_step": (I32, [C.POINTER(AdamWConfig), C.c_int64, P, P, P, P, P, C.c_int64, P]),
    "cadet_bf16_to_f32": (I32, [P, P, C.c_int64, P]),
    "cadet_chunk": (I32, [P, I32, I32, P, I32, P, P, P]),
    "cadet_bucketize": (I32, [P, I32, C.POINTER(I32), I32, P, P, P]),
    "cadet_pack": (I32, [P, P, P, I32, I32, I32, P, P, P, P, P, P, P, P, SZ, P]),
    "cadet_pack_workspace_bytes": (SZ, [I32]),
    "cadet_gemm": (I32, [I32, I32, I32, P, I32, P, I32, P, I32, P, P]),
    "cadet_gemm_fp32_workspace_bytes": (SZ, [I32, I32, I32]),
    "cadet_gemm_fp32": (I32, [I32, I32, I32, P, I32, P, I32, P, P, P, SZ, P]),
    "cadet_poll": (I32, [P, P]),
    "cadet_launch_count": (I64, []),
    "cadet_prof_enable": (I32, [I32, I32]),
    "cadet_prof_read": (I32, [C.POINTER(C.c_double), C.POINTER(I64)]),
}

_lib = None


def lib():
    """Load libcadet.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libcadet.so not built at {LIB_PATH}; run python -m paper_2602_11410_b200.build")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def has(name: str) -> bool:
    return getattr(lib(), name, None) is not None


def check(status: int):
    if status != 0:
        raise CadetError(status, lib().cadet_last_error().decode(errors="replace"))


def default_config(d_model: int, n_heads: int, **kw) -> AttnConfig:
    cfg = AttnConfig()
    lib().cadet_default_attn_config(C.byref(cfg), d_model, n_heads)
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise AttributeError(k)
        setattr(cfg, k, v)
    return cfg
