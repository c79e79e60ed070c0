"""Stage-by-stage parity of one gated layer (SURVEY 8(c) protocol iii) from the layer's parity taps.

Every GPU stage value before its bf16 rounding (cadet_attn_stage_views taps, cfg.out_f32 = 1) is
compared with the fp64 oracle stage fed the bf16 tensors that GPU stage consumed (saved activations,
the backward's bf16 intermediates), at the north-star tolerance max-abs 1e-2 / mean-abs 1e-3 (R19
normalisation) with no storage allowance.  Used at oracle-sized shapes (test_gpu_stages.py, every
sequence) and at BASELINE's full sizes in the bench's launch configuration (test_gpu_fullsize.py,
sampled sequences; the weight gradients always over all rows).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle import cadet_oracle as O
from tests.helpers import assert_close, err_stats, to_np


class DevArr:
    """A device tensor read lazily: a[rows] / a[:, cols] copy only that slice to the host (fp64)."""

    def __init__(self, t):
        self.t = t

    def __getitem__(self, idx):
        return self.t[idx].float().cpu().numpy().astype(np.float64)

    @property
    def shape(self):
        return tuple(self.t.shape)


def read_views(lib_mod, cfg, n_seqs, T, ws, H, lazy=False):
    """Taps (fp32 [T, d]), bf16 backward intermediates and D [H, T] of the layer workspace ws
    (device views wrapped in DevArr when lazy, else host fp64 arrays)."""
    import torch
    L = lib_mod
    d = cfg.d_model
    views = (C.c_void_p * L.CADET_N_VIEWS)()
    L.check(L.lib().cadet_attn_stage_views(C.byref(cfg), n_seqs, T, C.c_void_p(ws.data_ptr()), ws.numel(), views))
    base = ws.data_ptr()

    def at(ptr, nbytes):
        off = ptr - base
        assert 0 <= off and off + nbytes <= ws.numel()
        return ws[off: off + nbytes]

    wrap = DevArr if lazy else (lambda x: x.float().cpu().numpy().astype(np.float64))
    taps = {n: wrap(at(views[i], T * d * 4).view(torch.float32).view(T, d)) for i, n in enumerate(L.TAP_NAMES)}
    wsb = {n: wrap(at(views[L.CADET_WS_DO + i], T * d * 2).view(torch.bfloat16).view(T, d))
           for i, n in enumerate(L.WS_NAMES)}
    D = wrap(at(views[L.CADET_WS_D], H * T * 4).view(torch.float32).view(H, T))
    return taps, wsb, D


def saved_dev(saved, T, d, H):
    """The layer's saved activations (bf16 [T, d] each, LSE fp32 [H, T]) as lazy device views."""
    import torch
    z = ((T * d * 2 + 255) // 256) * 256
    names = ["Zx", "Xt", "Q", "K", "Zq", "Zk", "Qr", "Kr", "V", "O"]
    out = {n: DevArr(saved[i * z: i * z + T * d * 2].view(torch.bfloat16).view(T, d)) for i, n in enumerate(names)}
    out["lse"] = DevArr(saved[10 * z: 10 * z + 4 * H * T].view(torch.float32).view(H, T))
    return out


def _core_tol(name, got, ref, peaky):
    if not peaky:
        return assert_close(got, ref, what=name)
    # R23: in the peaky regime P and dS are bf16 MMA operands: 1e-1 / 5e-3 for the attention core
    mx, mn, rms = err_stats(got, ref)
    print(f"[parity] {name} (peaky): max {mx:.3e} mean {mn:.3e} (rms ref {rms:.3e})")
    assert mx <= 1e-1 and mn <= 5e-3, (name, mx, mn)
    return mx, mn


def check_layer_stages(X, W, sv, tp, wb, D, dY, meta, ocfg, seqs, resid=None, dresid=None, peaky=False,
                       forward=True, backward=True, weight_grads=None, wg_sample=None, d_from_stored=False,
                       tag=""):
    """X: the layer input (bf16 values) [T, d]; W: the 7 weights (fp64); sv: saved views; tp: taps;
    wb / D: backward intermediates; dY: the upstream gradient; meta / ocfg: the batch for the oracle;
    seqs: sequence indices to check row-wise; resid / dresid: the residual added to Y / to dX (or
    None); weight_grads: the GPU's 7 fp32 weight gradients (checked over all real rows: every entry, or
    wg_sample random entries at full size) or None.  Arrays may be host fp64 or DevArr."""
    Wxg, Wq, Wk, Wv, Wqg, Wkg, Wo = W
    H = ocfg.n_heads
    d = ocfg.d_model
    hd = d // H
    cu = np.asarray(meta.cu, np.int64)
    t = np.asarray(meta.t_ms, np.int64)
    for k in seqs:
        a, e = int(cu[k]), int(cu[k + 1])
        tg = f"{tag} seq {k} len {e - a}"
        A = O.seq_mask(meta, k, ocfg)
        trel = t[a:e] - t[a]   # the GPU rotates by times rebased to the sequence start (R21)
        sl = slice(a, e)
        x = X[sl]
        if forward:
            # A2 (Eq. 4) fed the bf16 X
            Zx = x @ Wxg
            assert_close(tp["Zx"][sl], Zx, what=f"A2 Zx {tg}")
            assert_close(tp["Xt"][sl], x * O.sigmoid(Zx), what=f"A2 Xt {tg}")
            # A3 (Eq. 3; R2) fed the bf16 Xt
            for nm, Wi in (("Q", Wq), ("K", Wk), ("V", Wv)):
                assert_close(tp[nm][sl], sv["Xt"][sl] @ Wi, what=f"A3 {nm} {tg}")
            # A4 (Eq. 5; RoPE P:274): Z from the bf16 Q / K, the rotation of Q * sigma(bf16 Z)
            for nm, src, Wg, zn in (("Qr", "Q", Wqg, "Zq"), ("Kr", "K", Wkg, "Zk")):
                assert_close(tp[zn][sl], sv[src][sl] @ Wg, what=f"A4 {zn} {tg}")
                assert_close(tp[nm][sl], O.rope_heads(sv[src][sl] * O.sigmoid(sv[zn][sl]), trel, ocfg),
                             what=f"A4 {nm} {tg}")
            # A5 (Eq. 7) fed the bf16 Qr, Kr, V
            o, l, _ = O.attention_core_forward(sv["Qr"][sl], sv["Kr"][sl], sv["V"][sl], A, H)
            _core_tol(f"A5 O {tg}", tp["O"][sl], o, peaky)
            assert_close(sv["lse"][:, sl], l, what=f"A5 LSE {tg}")
            # A6 fed the bf16 O (+ the residual)
            y = sv["O"][sl] @ Wo + (0 if resid is None else resid[sl])
            assert_close(tp["Y"][sl], y, what=f"A6 Y {tg}")
        if backward:
            g = dY[sl]
            # A9: dO = dY W_o^T; D = rowsum(dO * O) per head (dO's fp32 value, the bf16 O)
            dO = g @ Wo.T
            assert_close(tp["dO"][sl], dO, what=f"A9 dO {tg}")
            # (d_from_stored: D comes from the preprocess kernel fed the stored bf16 dO -- deterministic mode)
            dOD = wb["dO"][sl] if d_from_stored else dO
            Dr = np.stack([(dOD[:, h * hd:(h + 1) * hd] * sv["O"][sl][:, h * hd:(h + 1) * hd]).sum(1) for h in range(H)])
            assert_close(D[:, sl], Dr, what=f"A9 D {tg}")
            # A10 (adjoint of Eq. 7) fed the bf16 Qr, Kr, V and the bf16 dO it consumed
            ref = O.attention_core_backward(sv["Qr"][sl], sv["Kr"][sl], sv["V"][sl], A, wb["dO"][sl], H)
            for nm, rf in zip(("dQr", "dKr", "dV"), ref):
                _core_tol(f"A10 {nm} {tg}", tp[nm][sl], rf, peaky)
            # A11 (adjoints of the rotation and of Eq. 5) fed the bf16 dQr / dKr, Q / K and Z
            for side, src, zn, Wg in (("q", "Q", "Zq", Wqg), ("k", "K", "Zk", Wkg)):
                dT = O.rope_heads(wb["dQr" if side == "q" else "dKr"][sl], trel, ocfg, -1.0)
                gg = O.sigmoid(sv[zn][sl])
                assert_close(tp["u" + side][sl], dT * sv[src][sl] * gg * (1 - gg), what=f"A11 u_{side} {tg}")
                assert_close(tp["r" + side][sl], dT * gg, what=f"A11 r_{side} {tg}")
                dn = "dQ" if side == "q" else "dK"
                assert_close(tp[dn][sl], wb["r" + side][sl] + wb["u" + side][sl] @ Wg.T, what=f"A11 {dn} {tg}")
            # A12 (adjoint of Eqs. 3-4) fed the bf16 dQ, dK, dV, X and Zx
            dXt = wb["dQ"][sl] @ Wq.T + wb["dK"][sl] @ Wk.T + wb["dV"][sl] @ Wv.T
            gx = O.sigmoid(sv["Zx"][sl])
            assert_close(tp["ux"][sl], dXt * x * gx * (1 - gx), what=f"A12 u_x {tg}")
            assert_close(tp["rx"][sl], dXt * gx + (0 if dresid is None else dresid[sl]), what=f"A12 r_x {tg}")
            assert_close(tp["dX"][sl], wb["rx"][sl] + wb["ux"][sl] @ Wxg.T, what=f"A12 dX {tg}")
    if weight_grads is not None:
        n = int(cu[-1])
        gW = weight_grads
        pairs = [(6, sv["O"], dY, "A9 dW_o"), (4, sv["Q"], wb["uq"], "A11 dW_qg"), (5, sv["K"], wb["uk"], "A11 dW_kg"),
                 (1, sv["Xt"], wb["dQ"], "A12 dW_q"), (2, sv["Xt"], wb["dK"], "A12 dW_k"), (3, sv["Xt"], wb["dV"], "A12 dW_v"),
                 (0, X, wb["ux"], "A12 dW_xg")]
        for gi, A_, G_, nm in pairs:
            if wg_sample is None:   # every entry: dW = A^T G over the real rows
                assert_close(gW[gi], A_[:n].T @ G_[:n], what=f"{nm} {tag}")
            else:                   # sampled entries dW[i, j] = sum_t A[t, i] G[t, j], the oracle one by one
                rng = np.random.default_rng(gi)
                ii = rng.integers(0, d, size=wg_sample)
                jj = rng.integers(0, d, size=wg_sample)
                ref = np.zeros(wg_sample)
                for r0 in range(0, n, 8192):
                    r1 = min(n, r0 + 8192)
                    ref += np.einsum("ts,ts->s", A_[r0:r1][:, ii], G_[r0:r1][:, jj])
                got = np.asarray(gW[gi])[ii, jj] if not hasattr(gW[gi], "t") else gW[gi].t[ii, jj].cpu().numpy()
                # R19 scale of the whole gradient from the GPU's own entries (rms of the sample otherwise)
                mx, mn, rms = err_stats(got, ref)
                print(f"[parity] {nm} {tag} ({wg_sample} sampled entries): max {mx:.3e} mean {mn:.3e} (rms {rms:.3e})")
                assert mx <= 1e-2 and mn <= 1e-3, (nm, mx, mn)
