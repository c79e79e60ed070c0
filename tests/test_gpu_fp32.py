"""GPU parity of the CADET_FP32 mode (SURVEY 8(c) protocol ii; north star "1e-4 for an fp32 mode"):
the 3xTF32 GEMM, the fp32 attention core under every mask rule, and the WHOLE chain -- gated layer
forward (Eqs. 3-7), towers and routed BCE (Eqs. 8-9), layer backward -- end to
end against the fp64 oracle at max-abs 1e-4 / mean-abs 1e-5 (R19 normalisation).  Unlike the bf16
stage gates this checks the algorithm itself: nothing is re-fed from the GPU between stages.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G
from tests.helpers import assert_close, err_stats, to_dev_batch
from tests.test_gpu_core import meta_of, oracle_cfg
from tests.test_gpu_layer import layer_case
from tests.test_gpu_stages import pair_flags_for

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MAX32, MEAN32 = 1e-4, 1e-5
T_, S_, P_ = 1, 2, 4


@pytest.fixture(scope="module")
def ops():
    from paper_2602_11410_b200 import build, ops as _ops
    build.build()
    return _ops


def f32(x):
    return torch.tensor(np.asarray(x, np.float32), device="cuda")


def npf(t):
    return t.detach().cpu().numpy().astype(np.float64)


def st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("M,N,K,a_t,b_t", [(128, 128, 64, 0, 0), (300, 96, 30, 0, 1), (257, 512, 1024, 1, 0),
                                           (1000, 352, 352, 1, 1), (64, 1024, 4100, 1, 0)])
def test_gemm_3xtf32(ops, M, N, K, a_t, b_t):
    """cadet_gemm_fp32 against fp64: relative error ~2^-21 sqrt(K), far below one TF32 pass (2^-11)."""
    from paper_2602_11410_b200 import _lib as L
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    R = rng.standard_normal((M, N)).astype(np.float32)
    Ad, Bd, Rd = f32(A.T.copy() if a_t else A), f32(B.T.copy() if b_t else B), f32(R)
    Cd = torch.empty(M, N, dtype=torch.float32, device="cuda")
    wsb = L.lib().cadet_gemm_fp32_workspace_bytes(M, N, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    L.check(L.lib().cadet_gemm_fp32(M, N, K, C.c_void_p(Ad.data_ptr()), a_t, C.c_void_p(Bd.data_ptr()), b_t,
                                    C.c_void_p(Cd.data_ptr()), C.c_void_p(Rd.data_ptr()), C.c_void_p(ws.data_ptr()),
                                    wsb, st()))
    torch.cuda.synchronize()
    ref = A.astype(np.float64) @ B.astype(np.float64) + R
    rel = np.abs(npf(Cd) - ref).max() / np.abs(ref).max()
    print(f"[parity] 3xTF32 GEMM {M}x{N}x{K}: max rel {rel:.2e}")
    assert rel < 2e-6


CORE32 = [
    ([64, 1, 33, 17], 32, 1, None, T_, None, False),
    ([300, 129, 700], 128, 2, [0, 5, 64], T_ | S_, None, False),
    ([513, 257, 1, 300], 352, 4, [0, 30, 0, 0], T_ | P_, [130, 0, 1, 0], True),
    ([400, 300, 129], 256, 4, [0, 50, 0], T_ | S_ | P_, [2, 129, 0], True),
]


@pytest.mark.parametrize("case", range(len(CORE32)))
@pytest.mark.parametrize("scale", [0.55, 2.2])
def test_attn_core_fp32(ops, case, scale):
    """fp32 attention core (A5 + A10) vs fp64, flat and peaky score regimes, every mask rule."""
    from tests.test_gpu_core import core_case
    lengths, d, H, nc, flags, nst, use_pf = CORE32[case]
    cu, t, s, ncv, T, Qr, Kr, V = core_case(lengths, d, H, nc, scale, seed=80 + case)
    pf = pair_flags_for(cu, T) if use_pf else None
    nstv = None if nst is None else np.asarray(nst, np.int32)
    dO = np.random.default_rng(81 + case).standard_normal((T, d)).astype(np.float32)
    cfg = ops.config(d, H, mask_flags=flags, delta_delay_ms=120_000)
    cfg.dtype = 1
    b = to_dev_batch(cu, t, s, ncv, T, n_static=nstv, flags=pf)
    from paper_2602_11410_b200 import _lib as L
    lib = L.lib()
    q, k, v, g = f32(Qr), f32(Kr), f32(V), f32(dO)
    Od = torch.empty(T, d, dtype=torch.float32, device="cuda")
    lse = torch.empty(H, T, dtype=torch.float32, device="cuda")
    ws = ops.workspace(lib.cadet_plan_workspace_bytes(b.n_seqs, T) + 4 * H * T + 4096)
    L.check(lib.cadet_attn_core_forward(C.byref(cfg), C.byref(b.struct()), *[C.c_void_p(x.data_ptr()) for x in (q, k, v, Od, lse)],
                                        C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    dQ, dK, dV = (torch.empty(T, d, dtype=torch.float32, device="cuda") for _ in range(3))
    L.check(lib.cadet_attn_core_backward(C.byref(cfg), C.byref(b.struct()),
                                         *[C.c_void_p(x.data_ptr()) for x in (q, k, v, Od, lse, g, dQ, dK, dV)],
                                         C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    torch.cuda.synchronize()
    ops.poll(ws)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv, n_static=nstv, flags=pf)
    Oref, lref = np.zeros((T, d)), np.zeros((H, T))
    ref = [np.zeros((T, d)) for _ in range(3)]
    for i in range(len(lengths)):
        a, e = cu[i], cu[i + 1]
        A = O.seq_mask(meta, i, ocfg)
        args = (Qr[a:e].astype(np.float64), Kr[a:e].astype(np.float64), V[a:e].astype(np.float64))
        o, l, _ = O.attention_core_forward(*args, A, H)
        Oref[a:e], lref[:, a:e] = o, l
        for j, x in enumerate(O.attention_core_backward(*args, A, dO[a:e].astype(np.float64), H)):
            ref[j][a:e] = x
    assert_close(npf(Od), Oref, MAX32, MEAN32, what=f"fp32 O (scale {scale})")
    assert_close(npf(lse), lref, MAX32, MEAN32, what="fp32 LSE")
    for nm, got, rf in zip(("dQ", "dK", "dV"), (dQ, dK, dV), ref):
        assert_close(npf(got), rf, MAX32, MEAN32, what=f"fp32 {nm} (scale {scale})")


# lengths, d, H, n_cand, peaky, flags, n_static, pair flags, paper RoPE constants (Unix-ms times)
E2E32 = [
    ([64, 1, 33, 17], 32, 1, None, False, T_, None, False, False),
    ([200, 77, 300], 128, 2, [0, 7, 30], True, T_, None, False, False),
    ([513, 257, 1, 300], 352, 4, None, False, T_ | S_, None, False, True),
    ([260, 5, 700], 512, 8, [0, 2, 64], True, T_ | P_, [130, 0, 3], True, False),
    ([400, 300, 129], 256, 2, [0, 50, 0], False, T_ | S_ | P_, [2, 129, 0], True, True),
]


@pytest.mark.parametrize("case", range(len(E2E32)))
def test_layer_and_towers_fp32_end_to_end(ops, case):
    """X -> gated layer -> towers -> routed BCE -> towers backward -> layer backward, all fp32 on the
    GPU, vs the fp64 oracle chain: Y, logits, loss, dH, dX, the 7 weight gradients and the 4 tower
    gradients within 1e-4 (max) / 1e-5 (mean)."""
    from paper_2602_11410_b200 import _lib as L
    lib = L.lib()
    lengths, d, H, nc, peaky, flags, nst, use_pf, paper = E2E32[case]
    cu, t, s, ncv, T, X, W = layer_case(lengths, d, H, nc, seed=90 + case, peaky=peaky, stress=not paper)
    pf = pair_flags_for(cu, T) if use_pf else None
    nstv = None if nst is None else np.asarray(nst, np.int32)
    if paper:   # P:627 constants on absolute Unix-ms times, Delta_delay = 1 h
        cfg = ops.config(d, H, mask_flags=flags)
    else:       # stress constants (R7): RoPE visibly active
        cfg = ops.config(d, H, mask_flags=flags, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4,
                         rope_delta_t_max_ms=86_400_000)
    cfg.dtype = 1
    b = to_dev_batch(cu, t, s, ncv, T, n_static=nstv, flags=pf)
    n_real = int(cu[-1])
    Wl = [x.astype(np.float64) for x in W.as_list()]
    Xd = f32(X)
    Wd = [f32(x) for x in W.as_list()]
    w = L.AttnWeights(*[x.data_ptr() for x in Wd])
    saved = torch.zeros(lib.cadet_attn_saved_bytes(C.byref(cfg), T), dtype=torch.uint8, device="cuda")
    ws = ops.workspace(lib.cadet_attn_workspace_bytes(C.byref(cfg), b.n_seqs, T))
    Y = torch.empty(T, d, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_attn_forward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                   C.c_void_p(Y.data_ptr()), None, C.c_void_p(saved.data_ptr()),
                                   C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    # towers on a random subset of the real rows (impressions), K = 2, dh = d / 2
    rng = np.random.default_rng(95 + case)
    K, dh = 2, max(32, d // 2)
    rows = np.sort(rng.choice(n_real, size=max(1, n_real // 2), replace=False)).astype(np.int32)
    nr = len(rows)
    hw = G.head_weights(95 + case, K, d, dh)
    bucket = rng.integers(0, K, size=nr).astype(np.int32)
    label = (rng.random(nr) < 0.3).astype(np.float32)
    W1cat = np.concatenate([hw.W1[k] for k in range(K)], axis=1)
    hc = L.HeadConfig(K, d, dh, 1)
    tens = {k_: torch.tensor(v_, device="cuda") for k_, v_ in dict(
        W1=W1cat.astype(np.float32), b1=hw.b1.reshape(-1), w2=hw.w2.reshape(-1), b2=hw.b2, rows=rows, bucket=bucket,
        label=label).items()}
    hwst = L.HeadWeights(*[tens[k_].data_ptr() for k_ in ("W1", "b1", "w2", "b2")])
    hws = ops.workspace(lib.cadet_heads_workspace_bytes(C.byref(hc), nr))
    logits = torch.empty(nr, K, dtype=torch.float32, device="cuda")
    pre = torch.empty(nr, K * dh, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_heads_forward(C.byref(hc), C.byref(hwst), C.c_void_p(Y.data_ptr()),
                                    C.c_void_p(tens["rows"].data_ptr()), nr, C.c_void_p(logits.data_ptr()),
                                    C.c_void_p(pre.data_ptr()), C.c_void_p(hws.data_ptr()), hws.numel(), st()))
    loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    dH = torch.empty(T, d, dtype=torch.float32, device="cuda")
    hg = [torch.empty(d, K * dh, dtype=torch.float32, device="cuda"), torch.empty(K * dh, dtype=torch.float32, device="cuda"),
          torch.empty(K * dh, dtype=torch.float32, device="cuda"), torch.empty(K, dtype=torch.float32, device="cuda")]
    hgs = L.HeadGrads(*[x.data_ptr() for x in hg])
    L.check(lib.cadet_heads_loss_backward(C.byref(hc), C.byref(hwst), C.c_void_p(Y.data_ptr()),
                                          C.c_void_p(tens["rows"].data_ptr()), nr, T, C.c_void_p(logits.data_ptr()),
                                          C.c_void_p(pre.data_ptr()), C.c_void_p(tens["bucket"].data_ptr()),
                                          C.c_void_p(tens["label"].data_ptr()), C.c_void_p(loss.data_ptr()),
                                          C.c_void_p(dH.data_ptr()), C.byref(hgs), C.c_void_p(hws.data_ptr()),
                                          hws.numel(), st()))
    dX = torch.empty(T, d, dtype=torch.float32, device="cuda")
    gs = [torch.empty(d, d, dtype=torch.float32, device="cuda") for _ in range(7)]
    g = L.AttnGrads(*[x.data_ptr() for x in gs])
    L.check(lib.cadet_attn_backward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                    C.c_void_p(saved.data_ptr()), C.c_void_p(dH.data_ptr()), C.c_void_p(dX.data_ptr()),
                                    None, C.byref(g), C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    torch.cuda.synchronize()
    ops.poll(ws)
    ops.poll(hws)
    # the fp64 oracle chain (nothing re-fed from the GPU)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv, n_static=nstv, flags=pf)
    Yr, caches, _ = O.batch_forward(X.astype(np.float64), Wl, meta, ocfg)
    # the ReLU' decision is taken from the GPU's fp32 pre-activation (a value at the kink may round to
    # either sign; a floating-point decision is taken in the same precision on both sides)
    act = [npf(pre)[:, k * dh:(k + 1) * dh] > 0 for k in range(K)]
    Lr, zr, dHr, ghr = O.heads_loss_backward(Yr, rows, hw.W1.astype(np.float64), hw.b1.astype(np.float64),
                                             hw.w2.astype(np.float64), hw.b2.astype(np.float64), bucket,
                                             label.astype(np.float64), relu_active=act)
    _, pre_r, _ = O.heads_forward(Yr, rows, hw.W1.astype(np.float64), hw.b1.astype(np.float64),
                                  hw.w2.astype(np.float64), hw.b2.astype(np.float64))
    flips = sum(int(((pre_r[k] > 0) != act[k]).sum()) for k in range(K))
    assert flips <= 2 and all(np.abs(pre_r[k][(pre_r[k] > 0) != act[k]]).max(initial=0) < 1e-4 for k in range(K))
    dXr, gWr, _ = O.batch_backward(caches, Wl, meta, dHr, ocfg)
    assert_close(npf(Y), Yr, MAX32, MEAN32, what="fp32 e2e Y")
    assert_close(npf(logits), zr, MAX32, MEAN32, what="fp32 e2e logits")
    assert abs(loss.item() - Lr) <= MAX32 * max(1.0, abs(Lr)), (loss.item(), Lr)
    assert_close(npf(dH), dHr, MAX32, MEAN32, what="fp32 e2e dH")
    assert_close(npf(hg[0]), np.concatenate([ghr["dW1"][k] for k in range(K)], axis=1), MAX32, MEAN32, what="fp32 e2e dW1")
    assert_close(npf(hg[1]), ghr["db1"].reshape(-1), MAX32, MEAN32, what="fp32 e2e db1")
    assert_close(npf(hg[2]), ghr["dw2"].reshape(-1), MAX32, MEAN32, what="fp32 e2e dw2")
    assert_close(npf(hg[3]), ghr["db2"], MAX32, MEAN32, what="fp32 e2e db2")
    assert_close(npf(dX), dXr, MAX32, MEAN32, what="fp32 e2e dX")
    for nm, gg, rr in zip(G.NAMES, gs, gWr):
        assert_close(npf(gg), rr, MAX32, MEAN32, what="fp32 e2e d" + nm)
    assert (npf(Y)[n_real:] == 0).all() and (npf(dX)[n_real:] == 0).all()


@pytest.mark.parametrize("ablate", ["use_rep_gate", "use_int_gate", "use_rope", "use_out_proj"])
def test_layer_fp32_ablations(ops, ablate):
    """Table 1's ablation switches in the fp32 mode: each stage can be turned off and the layer forward /
    backward still matches the oracle (with the same switch) end to end within 1e-4."""
    from paper_2602_11410_b200 import _lib as L
    lib = L.lib()
    lengths, d, H = [300, 129, 77], 128, 2
    cu, t, s, ncv, T, X, W = layer_case(lengths, d, H, None, seed=7)
    cfg = ops.config(d, H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4, rope_delta_t_max_ms=86_400_000)
    cfg.dtype = 1
    setattr(cfg, ablate, 0)
    b = to_dev_batch(cu, t, s, ncv, T)
    Xd, Wd = f32(X), [f32(x) for x in W.as_list()]
    w = L.AttnWeights(*[x.data_ptr() for x in Wd])
    saved = torch.zeros(lib.cadet_attn_saved_bytes(C.byref(cfg), T), dtype=torch.uint8, device="cuda")
    ws = ops.workspace(lib.cadet_attn_workspace_bytes(C.byref(cfg), b.n_seqs, T))
    Y = torch.empty(T, d, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_attn_forward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                   C.c_void_p(Y.data_ptr()), None, C.c_void_p(saved.data_ptr()),
                                   C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    dY = np.random.default_rng(8).standard_normal((T, d)).astype(np.float32)
    dY[cu[-1]:] = 0
    dX = torch.empty(T, d, dtype=torch.float32, device="cuda")
    gs = [torch.empty(d, d, dtype=torch.float32, device="cuda") for _ in range(7)]
    g = L.AttnGrads(*[x.data_ptr() for x in gs])
    dYd = f32(dY)
    L.check(lib.cadet_attn_backward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                    C.c_void_p(saved.data_ptr()), C.c_void_p(dYd.data_ptr()), C.c_void_p(dX.data_ptr()),
                                    None, C.byref(g), C.c_void_p(ws.data_ptr()), ws.numel(), st()))
    torch.cuda.synchronize()
    ops.poll(ws)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv)
    Wl = [x.astype(np.float64) for x in W.as_list()]
    Yr, caches, _ = O.batch_forward(X.astype(np.float64), Wl, meta, ocfg)
    dXr, gWr, _ = O.batch_backward(caches, Wl, meta, dY.astype(np.float64), ocfg)
    assert_close(npf(Y), Yr, MAX32, MEAN32, what=f"fp32 {ablate}=0 Y")
    assert_close(npf(dX), dXr, MAX32, MEAN32, what=f"fp32 {ablate}=0 dX")
    for nm, gg, rr in zip(G.NAMES, gs, gWr):
        assert_close(npf(gg), rr, MAX32, MEAN32, what=f"fp32 {ablate}=0 d{nm}")
