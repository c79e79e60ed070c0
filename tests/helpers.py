"""Shared test helpers: seeded cases from synth/, comparison with the R19 normalisation."""
from __future__ import annotations

import numpy as np

from synth import generator as G

MAX_ABS = 1e-2     # north-star bf16-in / fp32-accumulate tolerances
MEAN_ABS = 1e-3


def err_stats(got, ref):
    """R19: |gpu - ref| / max(1, rms(ref)); returns (max, mean, rms(ref))."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    e = np.abs(got - ref) / max(1.0, rms)
    return (float(e.max()) if e.size else 0.0, float(e.mean()) if e.size else 0.0, rms)


def assert_close(got, ref, max_abs=MAX_ABS, mean_abs=MEAN_ABS, what=""):
    mx, mn, rms = err_stats(got, ref)
    if what:
        print(f"[parity] {what}: max {mx:.3e} mean {mn:.3e} (rms ref {rms:.3e})")
    assert mx <= max_abs and mn <= mean_abs, f"{what}: max {mx:.3e} mean {mn:.3e} (rms ref {rms:.3e})"
    return mx, mn


def bf16_half_ulp(x):
    """Half a bf16 ulp of |x| (round-to-nearest storage error bound)."""
    a = np.abs(np.asarray(x, dtype=np.float64))
    e = np.floor(np.log2(np.maximum(a, 1e-38)))
    return np.where(a > 0, 0.5 * np.exp2(e - 7), 0.0)


def assert_close_stored(got_bf16, ref, max_abs=MAX_ABS, mean_abs=MEAN_ABS, what=""):
    """Protocol (iii) for a stage whose fp32 accumulator is stored as bf16: the storage
    rounding (<= half a bf16 ulp, deterministic) is removed before applying the tolerance,
    so what is gated is the accumulator's error (R22)."""
    got = np.asarray(got_bf16, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    allow = bf16_half_ulp(np.abs(ref))  # from the reference only: a wrong value never widens its own bound
    resid = np.maximum(np.abs(got - ref) - allow, 0.0) / max(1.0, rms)
    mx, mn = float(resid.max()), float(resid.mean())
    assert mx <= max_abs and mn <= mean_abs, f"{what}: accumulator max {mx:.3e} mean {mn:.3e} (rms ref {rms:.3e})"
    return mx, mn


def make_case(lengths, T=None, n_cand=None, stress=True, seed=0):
    """Packed batch metadata (host numpy) of given sequence lengths; T = budget (>= sum)."""
    cfgg = G.stress_config() if stress else G.GenConfig()
    b = G.fixed_lengths_batch(list(lengths), seed=seed, cfg=cfgg, n_cand=n_cand)
    n_real = b.n_tokens
    T = n_real if T is None else T
    cu = np.concatenate([[0], np.cumsum(b.lengths)]).astype(np.int32)
    t = np.zeros(T, np.int64)
    t[:n_real] = b.timestamps
    s = np.zeros(T, np.int32)
    s[:n_real] = b.session_ids
    nc = np.zeros(len(lengths), np.int32) if n_cand is None else np.asarray(n_cand, np.int32)
    return cu, t, s, nc, T


def to_dev_batch(cu, t, s, nc, T, max_seqlen=None, n_static=None, flags=None, with_sess=True):
    import torch
    from paper_2602_11410_b200 import ops
    dev = "cuda"
    return ops.PackedBatch(
        cu_seqlens=torch.tensor(cu, dtype=torch.int32, device=dev),
        timestamps_ms=torch.tensor(t, dtype=torch.int64, device=dev),
        total_tokens=int(T),
        max_seqlen=int(max_seqlen or max(1, int(np.max(np.diff(cu))) if len(cu) > 1 else 1)),
        session_ids=torch.tensor(s, dtype=torch.int32, device=dev) if with_sess else None,
        n_candidates=torch.tensor(nc, dtype=torch.int32, device=dev),
        n_static=None if n_static is None else torch.tensor(n_static, dtype=torch.int32, device=dev),
        token_flags=None if flags is None else torch.tensor(flags, dtype=torch.uint8, device=dev),
    )


def bf16_tensor(x, device="cuda"):
    import torch
    return torch.tensor(G.bf16_round(np.asarray(x, np.float32)), dtype=torch.float32).to(device).to(torch.bfloat16)


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)
