"""Torch-facing wrappers over the libcadet C ABI (same names as include/cadet.h without the
`cadet_` prefix).  PyTorch supplies device memory and the current stream only; every
computation is a libcadet kernel.  All tensors must be CUDA tensors; nothing falls back to
PyTorch or the CPU."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L

BF16 = torch.bfloat16


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libcadet ops take CUDA tensors only (no CPU fallback)")


def config(d_model: int, n_heads: int, **kw) -> L.AttnConfig:
    return L.default_config(d_model, n_heads, **kw)


@dataclass
class PackedBatch:
    """Device-side packed batch: cu_seqlens [n+1] int32, timestamps [T] int64, ..."""
    cu_seqlens: torch.Tensor
    timestamps_ms: torch.Tensor
    total_tokens: int
    max_seqlen: int
    session_ids: torch.Tensor | None = None
    n_candidates: torch.Tensor | None = None
    n_static: torch.Tensor | None = None
    token_flags: torch.Tensor | None = None

    @property
    def n_seqs(self) -> int:
        return int(self.cu_seqlens.numel()) - 1

    def struct(self) -> L.BatchStruct:
        b = L.BatchStruct()
        b.n_seqs = self.n_seqs
        b.total_tokens = self.total_tokens
        b.max_seqlen = self.max_seqlen
        b.cu_seqlens = self.cu_seqlens.data_ptr()
        b.timestamps_ms = self.timestamps_ms.data_ptr()
        b.session_ids = None if self.session_ids is None else self.session_ids.data_ptr()
        b.n_candidates = None if self.n_candidates is None else self.n_candidates.data_ptr()
        b.n_static = None if self.n_static is None else self.n_static.data_ptr()
        b.token_flags = None if self.token_flags is None else self.token_flags.data_ptr()
        return b


def workspace(nbytes: int, device="cuda") -> torch.Tensor:
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def plan_workspace(batch: PackedBatch) -> torch.Tensor:
    return workspace(L.lib().cadet_plan_workspace_bytes(batch.n_seqs, batch.total_tokens),
                     batch.cu_seqlens.device)


def mask_plan(cfg, batch: PackedBatch, ws: torch.Tensor):
    L.check(L.lib().cadet_mask_plan(C.byref(cfg), C.byref(batch.struct()), _p(ws), ws.numel(), _stream()))


def mask_export(cfg, batch: PackedBatch, ws: torch.Tensor, tile_class_cap: int):
    dev = batch.cu_seqlens.device
    kv_end = torch.empty(batch.total_tokens, dtype=torch.int32, device=dev)
    tc = torch.full((max(tile_class_cap, 1),), -1, dtype=torch.int8, device=dev)
    pairs = torch.zeros(1, dtype=torch.int64, device=dev)
    L.check(L.lib().cadet_mask_export(C.byref(cfg), C.byref(batch.struct()), _p(ws), _p(kv_end), _p(tc),
                                      tile_class_cap, _p(pairs), _stream()))
    return kv_end, tc[:tile_class_cap], pairs


def poll(ws: torch.Tensor):
    L.check(L.lib().cadet_poll(_p(ws), _stream()))


def attn_core_forward(cfg, batch: PackedBatch, Qr, Kr, V, ws=None):
    _need_cuda(Qr, Kr, V)
    T, d = Qr.shape
    ws = plan_workspace(batch) if ws is None else ws
    O = torch.empty(T, d, dtype=torch.float32 if cfg.out_f32 else BF16, device=Qr.device)
    lse = torch.empty(cfg.n_heads, T, dtype=torch.float32, device=Qr.device)
    L.check(L.lib().cadet_attn_core_forward(C.byref(cfg), C.byref(batch.struct()), _p(Qr), _p(Kr), _p(V), _p(O),
                                            _p(lse), _p(ws), ws.numel(), _stream()))
    return O, lse


def attn_core_backward(cfg, batch: PackedBatch, Qr, Kr, V, O, lse, dO, ws=None):
    _need_cuda(Qr, Kr, V, O, lse, dO)
    T, d = Qr.shape
    ws = plan_workspace(batch) if ws is None else ws
    odt = torch.float32 if cfg.out_f32 else BF16
    dQ = torch.empty(T, d, dtype=torch.float32, device=Qr.device)
    dK = torch.empty(T, d, dtype=odt, device=Qr.device)
    dV = torch.empty(T, d, dtype=odt, device=Qr.device)
    L.check(L.lib().cadet_attn_core_backward(C.byref(cfg), C.byref(batch.struct()), _p(Qr), _p(Kr), _p(V), _p(O),
                                             _p(lse), _p(dO), _p(dQ), _p(dK), _p(dV), _p(ws), ws.numel(),
                                             _stream()))
    return dQ, dK, dV


def gemm(A, B, a_mn: bool = False, b_mn: bool = False, out_f32: bool = True, resid=None):
    """C = A_op . B_op with A_op = A (a_mn=False, A [M,K]) or A^T storage (a_mn=True, A [K,M]);
    B_op from B [N,K] (b_mn=False) or B [K,N] (b_mn=True)."""
    _need_cuda(A, B, resid)
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    out = torch.empty(M, N, dtype=torch.float32 if out_f32 else BF16, device=A.device)
    L.check(L.lib().cadet_gemm(M, N, K, _p(A), int(a_mn), _p(B), int(b_mn), _p(out), int(out_f32), _p(resid),
                               _stream()))
    return out


def rmsnorm_forward(X, gamma, Y=None, rstd=None):
    """NEXT-3 (R32): Y = X / sqrt(mean(X^2) + 1e-6) * gamma; returns (Y bf16, rstd fp32 [T])."""
    _need_cuda(X, gamma)
    T, d = X.shape
    Y = torch.empty_like(X) if Y is None else Y
    rstd = torch.empty(T, dtype=torch.float32, device=X.device) if rstd is None else rstd
    L.check(L.lib().cadet_rmsnorm_forward(_p(X), _p(gamma), T, d, _p(Y), _p(rstd), _stream()))
    return Y, rstd


def rmsnorm_backward(X, gamma, rstd, dY, dresid=None, dX=None, dgamma=None):
    """dX (+ dresid) and dgamma (fp32 [d], overwritten)."""
    _need_cuda(X, gamma, rstd, dY, dresid)
    T, d = X.shape
    dX = torch.empty_like(X) if dX is None else dX
    dgamma = torch.empty(d, dtype=torch.float32, device=X.device) if dgamma is None else dgamma
    L.check(L.lib().cadet_rmsnorm_backward(_p(X), _p(gamma), _p(rstd), _p(dY), _p(dresid), T, d, _p(dX), _p(dgamma),
                                           _stream()))
    return dX, dgamma


def ffn_forward(X, W1, W2, resid=None, Y=None, U=None, Gt=None):
    """NEXT-3 (R33): U = X W1, G = GELU(U), Y = G W2 (+ resid); returns (Y, U, G)."""
    _need_cuda(X, W1, W2, resid)
    T, d = X.shape
    m = W1.shape[1] // d
    Y = torch.empty_like(X) if Y is None else Y
    U = torch.empty(T, m * d, dtype=BF16, device=X.device) if U is None else U
    Gt = torch.empty(T, m * d, dtype=BF16, device=X.device) if Gt is None else Gt
    L.check(L.lib().cadet_ffn_forward(_p(X), _p(W1), _p(W2), _p(resid), T, d, m, _p(Y), _p(U), _p(Gt), _stream()))
    return Y, U, Gt


def ffn_backward(X, W1, W2, U, Gt, dY, dresid=None, dX=None, dW1=None, dW2=None, ws=None):
    """Returns (dX, dW1, dW2, ws); ws[: T m d bf16] holds dU after the call."""
    _need_cuda(X, W1, W2, U, Gt, dY, dresid)
    T, d = X.shape
    m = W1.shape[1] // d
    dX = torch.empty_like(X) if dX is None else dX
    dW1 = torch.empty(d, m * d, dtype=torch.float32, device=X.device) if dW1 is None else dW1
    dW2 = torch.empty(m * d, d, dtype=torch.float32, device=X.device) if dW2 is None else dW2
    ws = workspace(L.lib().cadet_ffn_workspace_bytes(T, d, m)) if ws is None else ws
    L.check(L.lib().cadet_ffn_backward(_p(X), _p(W1), _p(W2), _p(U), _p(Gt), _p(dY), _p(dresid), T, d, m, _p(dX),
                                       _p(dW1), _p(dW2), _p(ws), ws.numel(), _stream()))
    return dX, dW1, dW2, ws


def adamw_config(**kw) -> L.AdamWConfig:
    c = L.AdamWConfig()
    L.lib().cadet_default_adamw_config(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def adamw_step(cfg, step: int, grad, param, m, v, param_bf16=None):
    """NEXT-4 (R35): fused AdamW over fp32 (grad, param, m, v) in place; param_bf16 gets bf16(param)."""
    _need_cuda(grad, param, m, v, param_bf16)
    n = param.numel()
    assert grad.numel() == n and m.numel() == n and v.numel() == n
    assert param_bf16 is None or param_bf16.numel() == n
    L.check(L.lib().cadet_adamw_step(C.byref(cfg), int(step), _p(grad), _p(param), _p(m), _p(v), _p(param_bf16), n,
                                     _stream()))


def bf16_to_f32(src, dst=None):
    _need_cuda(src, dst)
    dst = torch.empty(src.shape, dtype=torch.float32, device=src.device) if dst is None else dst
    L.check(L.lib().cadet_bf16_to_f32(_p(src), _p(dst), src.numel(), _stream()))
    return dst


def chunk(cu_in: torch.Tensor, L_chunk: int, cap: int, ws=None):
    _need_cuda(cu_in)
    ws = workspace(256, cu_in.device) if ws is None else ws
    cu_out = torch.full((cap,), -1, dtype=torch.int32, device=cu_in.device)
    n_out = torch.zeros(1, dtype=torch.int32, device=cu_in.device)
    L.check(L.lib().cadet_chunk(_p(cu_in), cu_in.numel() - 1, L_chunk, _p(cu_out), cap, _p(n_out), _p(ws),
                                _stream()))
    return cu_out, n_out, ws


def pack(src, lens, budget: int, src_row=None, t_src=None, s_src=None, ws=None):
    """A13: greedy arrival-order packing into a fixed budget.  src [rows, d] bf16 with
    sequence s at rows [src_row[s], src_row[s] + lens[s]) (src_row None = back to back)."""
    _need_cuda(src, lens, src_row, t_src, s_src)
    d = src.shape[-1]
    B = lens.numel()
    dev = src.device
    ws = workspace(L.lib().cadet_pack_workspace_bytes(B), dev) if ws is None else ws
    packed = torch.empty(budget, d, dtype=src.dtype, device=dev)
    t_out = torch.empty(budget, dtype=torch.int64, device=dev) if t_src is not None else None
    s_out = torch.empty(budget, dtype=torch.int32, device=dev) if s_src is not None else None
    cu = torch.empty(B + 1, dtype=torch.int32, device=dev)
    n_packed = torch.zeros(1, dtype=torch.int32, device=dev)
    L.check(L.lib().cadet_pack(_p(src), _p(src_row), _p(lens), B, d, budget, _p(t_src), _p(s_src), _p(packed),
                               _p(t_out), _p(s_out), _p(cu), _p(n_packed), _p(ws), ws.numel(), _stream()))
    return packed, t_out, s_out, cu, n_packed, ws


def launch_count() -> int:
    return int(L.lib().cadet_launch_count())


def prof_enable(classes: int = 15, max_pairs: int = 4096):
    L.check(L.lib().cadet_prof_enable(classes, max_pairs))


PROF_CLASSES = ("gemm", "attn_fwd", "attn_bwd", "other")


def prof_read():
    ms = (C.c_double * 4)()
    n = (C.c_int64 * 4)()
    L.check(L.lib().cadet_prof_read(ms, n))
    return {k: (ms[i], int(n[i])) for i, k in enumerate(PROF_CLASSES)}
