"""CADET hot-path training step over the libcadet C ABI (one process per GPU).

A step (in order):
  A13 pack   contiguous user histories -> fixed budget T (cadet_pack)
  A0  chunk  refine offsets so no sequence exceeds L_chunk (cadet_chunk)
  A1-A6      L residual layers of self-gated attention forward (cadet_attn_forward; plan inside)
  A7-A8      context-conditioned towers + routed BCE + tower backward (cadet_heads_*)
  A9-A12     layers backward (cadet_attn_backward), weight gradients into one flat fp32 buffer
  DP         torch.distributed all_reduce(SUM) of the flat gradient buffer (NCCL) when world > 1
Every computation is a libcadet kernel; PyTorch only allocates memory, provides the stream and
runs the NCCL collective.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import ops


@dataclass
class StackConfig:
    d_model: int = 1024
    n_heads: int = 8
    n_layers: int = 1
    budget: int = 65536          # T: packed rows per step
    L_chunk: int = 2048
    K: int = 2                   # towers
    d_hidden: int = 0            # 0 -> d_model // 2
    delta_delay_ms: int = 3_600_000
    mask_flags: int = L.CADET_MASK_TIME

    @property
    def dh(self) -> int:
        return self.d_hidden or self.d_model // 2


@dataclass
class StepInputs:
    """Device (or pinned host) tensors of one step plus host-side counts known to the loader."""
    X_hist: torch.Tensor     # [R, d] bf16, histories back to back (arrival order)
    t_hist: torch.Tensor     # [R] int64 Unix ms
    s_hist: torch.Tensor     # [R] int32 session ids
    lens: torch.Tensor       # [B] int32 history lengths
    rows: torch.Tensor       # [n_imp] int32 packed rows of impression tokens
    bucket: torch.Tensor     # [n_imp] int32 realised context bucket k_t
    label: torch.Tensor      # [n_imp] fp32 click label y_t
    n_hist: int
    n_chunks: int
    tokens: int              # real tokens T_r

    def to(self, device, non_blocking=True) -> "StepInputs":
        f = lambda t: t.to(device, non_blocking=non_blocking)
        return StepInputs(f(self.X_hist), f(self.t_hist), f(self.s_hist), f(self.lens), f(self.rows),
                          f(self.bucket), f(self.label), self.n_hist, self.n_chunks, self.tokens)

    def copy_(self, src: "StepInputs"):
        for a in ("X_hist", "t_hist", "s_hist", "lens", "rows", "bucket", "label"):
            getattr(self, a).copy_(getattr(src, a), non_blocking=True)

    def nbytes(self) -> int:
        return sum(getattr(self, a).numel() * getattr(self, a).element_size()
                   for a in ("X_hist", "t_hist", "s_hist", "lens", "rows", "bucket", "label"))


def make_inputs(users, d: int, L_chunk: int, seed: int, pin: bool = False) -> StepInputs:
    """Host-side data loader output for one batch of generator users (synth/ Appendix B)."""
    from synth import generator as G
    lens = np.array([u.length for u in users], dtype=np.int32)
    R = int(lens.sum())
    X = G.normal_bf16(seed, 11, (R, d))
    t = np.concatenate([u.timestamps for u in users]).astype(np.int64)
    s = np.concatenate([u.session_ids for u in users]).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    rows = np.concatenate([st + u.impression_rows for st, u in zip(starts, users)]).astype(np.int32)
    bucket = np.concatenate([u.buckets[u.impression_rows] for u in users]).astype(np.int32)
    label = np.concatenate([u.labels[u.impression_rows] for u in users]).astype(np.float32)
    n_chunks = int(sum(-(-int(m) // L_chunk) for m in lens))
    mk = lambda a, dt: (torch.from_numpy(np.ascontiguousarray(a)).to(dt))
    Xt = torch.from_numpy(X).to(torch.bfloat16)
    inp = StepInputs(Xt, mk(t, torch.int64), mk(s, torch.int32), mk(lens, torch.int32), mk(rows, torch.int32),
                     mk(bucket, torch.int32), mk(label, torch.float32), len(users), n_chunks, R)
    if pin:
        inp = StepInputs(*[x.pin_memory() for x in (inp.X_hist, inp.t_hist, inp.s_hist, inp.lens, inp.rows,
                                                    inp.bucket, inp.label)], inp.n_hist, inp.n_chunks, inp.tokens)
    return inp


def dp_reduce(grads: torch.Tensor, loss: torch.Tensor, group=None):
    """the routed loss is a SUM over impressions (Eq. 9, R15), so summing the ranks'
    flat fp32 gradient buffers (one NCCL all-reduce bucket) gives exactly the union-batch gradient."""
    if group is None:
        return grads, loss
    torch.distributed.all_reduce(grads, group=group)
    torch.distributed.all_reduce(loss, group=group)
    return grads, loss


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class CadetStack:
    """Weights, activations and workspaces for L layers + towers on one GPU."""

    def __init__(self, cfg: StackConfig, seed: int = 0, device="cuda", peaky: bool = False):
        from synth import generator as G
        self.cfg = cfg
        self.dev = torch.device(device)
        d, T, nl = cfg.d_model, cfg.budget, cfg.n_layers
        self.acfg = ops.config(d, cfg.n_heads, delta_delay_ms=cfg.delta_delay_ms, mask_flags=cfg.mask_flags)
        bf = lambda a: torch.from_numpy(a).to(torch.bfloat16).to(self.dev)
        self.W = [[bf(w) for w in G.layer_weights(seed, l, d, peaky).as_list()] for l in range(nl)]
        hw = G.head_weights(seed, cfg.K, d, cfg.dh)
        self.W1 = bf(np.concatenate([hw.W1[k] for k in range(cfg.K)], axis=1))
        self.b1 = torch.from_numpy(hw.b1.reshape(-1).copy()).to(self.dev)
        self.w2 = torch.from_numpy(hw.w2.reshape(-1).copy()).to(self.dev)
        self.b2 = torch.from_numpy(hw.b2.copy()).to(self.dev)
        # flat fp32 gradient buffer: 7 d^2 per layer + towers (one NCCL all-reduce bucket)
        N = cfg.K * cfg.dh
        self.n_grad = nl * 7 * d * d + d * N + 2 * N + cfg.K
        self.grads = torch.zeros(self.n_grad, dtype=torch.float32, device=self.dev)
        off = 0
        self.gW = []
        for _ in range(nl):
            gl = []
            for _ in range(7):
                gl.append(self.grads[off:off + d * d])
                off += d * d
            self.gW.append(gl)
        self.gW1 = self.grads[off:off + d * N]; off += d * N
        self.gb1 = self.grads[off:off + N]; off += N
        self.gw2 = self.grads[off:off + N]; off += N
        self.gb2 = self.grads[off:off + cfg.K]
        lib = L.lib()
        self.saved_bytes = lib.cadet_attn_saved_bytes(C.byref(self.acfg), T)
        self.saved = [torch.empty(self.saved_bytes, dtype=torch.uint8, device=self.dev) for _ in range(nl)]
        self.Hs = [torch.empty(T, d, dtype=torch.bfloat16, device=self.dev) for _ in range(nl + 1)]
        self.dHs = [torch.empty(T, d, dtype=torch.bfloat16, device=self.dev) for _ in range(nl + 1)]
        self.t_p = torch.empty(T, dtype=torch.int64, device=self.dev)
        self.s_p = torch.empty(T, dtype=torch.int32, device=self.dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.small_ws = ops.workspace(4096, self.dev)
        self._ws = None
        self._hws = None
        self._bufs_for = None

    # -------------------------------------------------------------- buffers sized per batch
    def _ensure(self, n_chunks: int, n_imp: int, n_hist: int):
        key = (n_chunks, n_imp, n_hist)
        if self._bufs_for == key:
            return
        lib = L.lib()
        cfg = self.cfg
        wsb = lib.cadet_attn_workspace_bytes(C.byref(self.acfg), n_chunks, cfg.budget)
        if self._ws is None or self._ws.numel() < wsb:
            self._ws = ops.workspace(wsb, self.dev)
        hc = L.HeadConfig(cfg.K, cfg.d_model, cfg.dh, 0)
        hwb = lib.cadet_heads_workspace_bytes(C.byref(hc), n_imp)
        if self._hws is None or self._hws.numel() < hwb:
            self._hws = ops.workspace(hwb, self.dev)
        self.logits = torch.empty(n_imp, cfg.K, dtype=torch.float32, device=self.dev)
        self.pre = torch.empty(n_imp, cfg.K * cfg.dh, dtype=torch.bfloat16, device=self.dev)
        self.cu_hist = torch.empty(n_hist + 1, dtype=torch.int32, device=self.dev)
        self.cu = torch.empty(n_chunks + 8, dtype=torch.int32, device=self.dev)
        self.n_out = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.n_packed = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._bufs_for = key

    def batch(self, inp: StepInputs) -> ops.PackedBatch:
        return ops.PackedBatch(cu_seqlens=self.cu[: inp.n_chunks + 1], timestamps_ms=self.t_p,
                               total_tokens=self.cfg.budget, max_seqlen=self.cfg.L_chunk, session_ids=self.s_p)

    # -------------------------------------------------------------- the step
    def step(self, inp: StepInputs, group=None, backward: bool = True) -> torch.Tensor:
        cfg, lib = self.cfg, L.lib()
        d, T = cfg.d_model, cfg.budget
        n_imp = inp.rows.numel()
        self._ensure(inp.n_chunks, n_imp, inp.n_hist)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        chk = L.check
        # A13 pack (contiguous histories, src_row = NULL) and A0 chunk
        chk(lib.cadet_pack(_vp(inp.X_hist), None, _vp(inp.lens), inp.n_hist, d, T, _vp(inp.t_hist),
                           _vp(inp.s_hist), _vp(self.Hs[0]), _vp(self.t_p), _vp(self.s_p), _vp(self.cu_hist),
                           _vp(self.n_packed), _vp(self.small_ws), 256, st))
        chk(lib.cadet_chunk(_vp(self.cu_hist), inp.n_hist, cfg.L_chunk, _vp(self.cu), inp.n_chunks + 8,
                            _vp(self.n_out), C.c_void_p(self.small_ws.data_ptr() + 256), st))
        b = self.batch(inp).struct()
        ws, wsn = _vp(self._ws), self._ws.numel()
        # A1: one mask plan per step, shared by every layer's forward and backward
        self.acfg.plan_ready = 0
        chk(lib.cadet_mask_plan(C.byref(self.acfg), C.byref(b), ws, wsn, st))
        self.acfg.plan_ready = 1
        # A1-A6: residual layers  H[l+1] = H[l] + Attn(H[l])
        for l in range(cfg.n_layers):
            w = L.AttnWeights(*[x.data_ptr() for x in self.W[l]])
            chk(lib.cadet_attn_forward(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(self.Hs[l]),
                                       _vp(self.Hs[l + 1]), _vp(self.Hs[l]), _vp(self.saved[l]), ws, wsn, st))
        # A7-A8: towers on impression rows + routed BCE
        hc = L.HeadConfig(cfg.K, d, cfg.dh, 0)
        hw = L.HeadWeights(self.W1.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr(), self.b2.data_ptr())
        chk(lib.cadet_heads_forward(C.byref(hc), C.byref(hw), _vp(self.Hs[-1]), _vp(inp.rows), n_imp,
                                    _vp(self.logits), _vp(self.pre), _vp(self._hws), self._hws.numel(), st))
        if not backward:
            return self.logits
        hg = L.HeadGrads(self.gW1.data_ptr(), self.gb1.data_ptr(), self.gw2.data_ptr(), self.gb2.data_ptr())
        chk(lib.cadet_heads_loss_backward(C.byref(hc), C.byref(hw), _vp(self.Hs[-1]), _vp(inp.rows), n_imp, T,
                                          _vp(self.logits), _vp(self.pre), _vp(inp.bucket), _vp(inp.label),
                                          _vp(self.loss), _vp(self.dHs[-1]), C.byref(hg), _vp(self._hws),
                                          self._hws.numel(), st))
        # A9-A12: layers backward; dX_l = dX_{l+1} (residual) + Attn_l^T(dX_{l+1})
        for l in reversed(range(cfg.n_layers)):
            w = L.AttnWeights(*[x.data_ptr() for x in self.W[l]])
            g = L.AttnGrads(*[x.data_ptr() for x in self.gW[l]])
            chk(lib.cadet_attn_backward(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(self.Hs[l]),
                                        _vp(self.saved[l]), _vp(self.dHs[l + 1]), _vp(self.dHs[l]),
                                        _vp(self.dHs[l + 1]), C.byref(g), ws, wsn, st))
        dp_reduce(self.grads, self.loss, group)
        return self.loss

    def pairs(self, inp: StepInputs) -> int:
        """Allowed (i, j) pairs of the planned mask (head-independent), from the plan's export hook."""
        self.step(inp, backward=False)
        self.acfg.plan_ready = 0
        kv, tc, pairs = ops.mask_export(self.acfg, self.batch(inp), self._ws, 0)
        return int(pairs.item())

    def poll(self):
        """Raise if any device-side input check latched an error (offsets, ordering, buckets...)."""
        ops.poll(self._ws)
        ops.poll(self._hws)
        ops.poll(self.small_ws)            # pack error word
        ops.poll(self.small_ws[256:])      # chunk error word
