"""GPU parity of the attention core backward, the full gated layer (forward stage by stage and
end to end, backward end to end) and the towers, against the fp64 oracle (SURVEY 8(c) protocol)."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G
from tests.helpers import assert_close, bf16_tensor, err_stats, make_case, to_dev_batch, to_np
from tests.test_gpu_core import core_case, meta_of, oracle_cfg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ops():
    from paper_2602_11410_b200 import build, ops as _ops
    build.build()
    return _ops


# Qr/Kr scale: 0.55 ~ the flat regime of a layer with sigma_w = 1/sqrt(d) (Var(Q) ~ 0.3);
# 2.2 ~ the peaky regime (sigma_w = 4/sqrt(d) for W_q, W_k).  SURVEY 8(c).
FLAT, PEAKY = 0.55, 2.2
BWD_CASES = [
    ([64, 1, 33, 17], 32, 1, None, FLAT),
    ([300, 129, 128, 127, 700], 128, 2, [0, 5, 0, 127, 64], FLAT),
    ([300, 129, 700], 256, 2, None, FLAT),
    ([513, 257, 1, 900], 352, 4, None, FLAT),
    ([400, 1000], 384, 4, [0, 100], FLAT),
    ([260, 5, 700], 512, 8, None, FLAT),
    ([300, 129, 700], 256, 2, None, PEAKY),
    ([260, 5, 700], 512, 8, [0, 2, 64], PEAKY),
]


@pytest.mark.parametrize("case", range(len(BWD_CASES)))
def test_attn_core_backward(ops, case):
    lengths, d, H, nc, scale = BWD_CASES[case]
    cu, t, s, ncv, T, Qr, Kr, V = core_case(lengths, d, H, nc, scale, seed=10 + case)
    rng = np.random.default_rng(77 + case)
    dO = G.bf16_round(rng.standard_normal((T, d)).astype(np.float32))
    cfg = ops.config(d, H, delta_delay_ms=120_000, out_f32=0)
    b = to_dev_batch(cu, t, s, ncv, T)
    q, k, v, g = bf16_tensor(Qr), bf16_tensor(Kr), bf16_tensor(V), bf16_tensor(dO)
    Og, lse = ops.attn_core_forward(cfg, b, q, k, v)
    cfg.out_f32 = 1
    dQ, dK, dV = ops.attn_core_backward(cfg, b, q, k, v, Og, lse, g)
    torch.cuda.synchronize()
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv)
    ref = [np.zeros((T, d)) for _ in range(3)]
    for i in range(len(lengths)):
        a, e = cu[i], cu[i + 1]
        A = O.seq_mask(meta, i, ocfg)
        r = O.attention_core_backward(Qr[a:e].astype(np.float64), Kr[a:e].astype(np.float64),
                                      V[a:e].astype(np.float64), A, dO[a:e].astype(np.float64), H)
        for j in range(3):
            ref[j][a:e] = r[j]
    for name, got, rf in zip(("dQ", "dK", "dV"), (dQ, dK, dV), ref):
        mx, mn, rms = err_stats(to_np(got), rf)
        print(f"core bwd scale {scale} {name}: max {mx:.3e} mean {mn:.3e} rms {rms:.3e}")
        if scale == FLAT:
            assert_close(to_np(got), rf, what=name)
        else:  # P and dS are bf16 MMA operands (as in FlashAttention): the peaky regime is reported and
            # gated at 10x max / 5x mean (R23: bf16 dS rounding alone gives ~2.5e-2 max here)
            assert mx <= 1e-1 and mn <= 5e-3, (name, mx, mn)
        assert (to_np(got)[cu[-1]:] == 0).all()


# ------------------------------------------------------------------ full layer
def layer_case(lengths, d, H, nc=None, seed=0, peaky=False, T_extra=5, stress=True):
    cu, t, s, ncv, T = make_case(lengths, n_cand=nc, seed=seed, stress=stress)
    T = T + T_extra
    t = np.concatenate([t, np.zeros(T_extra, np.int64)])
    s = np.concatenate([s, np.zeros(T_extra, np.int32)])
    X = G.normal_bf16(seed, 1, (T, d))
    X[cu[-1]:] = 0
    W = G.layer_weights(seed, 0, d, peaky=peaky)
    return cu, t, s, ncv, T, X, W


def run_layer_forward(ops, cfg, b, X, W, T, two_pass=False):
    from paper_2602_11410_b200 import _lib as L
    d = cfg.d_model
    Xd = bf16_tensor(X)
    Wd = [bf16_tensor(w) for w in W.as_list()]
    w = L.AttnWeights(*[x.data_ptr() for x in Wd])
    saved = torch.zeros(L.lib().cadet_attn_saved_bytes(C.byref(cfg), T), dtype=torch.uint8, device="cuda")
    extra = L.lib().cadet_attn_bwd_ds_bytes(C.byref(cfg), b.n_seqs, T, b.max_seqlen) if two_pass else 0
    ws = ops.workspace(L.lib().cadet_attn_workspace_bytes(C.byref(cfg), b.n_seqs, T) + extra)
    Y = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    L.check(L.lib().cadet_attn_forward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                       C.c_void_p(Y.data_ptr()), None, C.c_void_p(saved.data_ptr()),
                                       C.c_void_p(ws.data_ptr()), ws.numel(),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return Y, saved, ws, Xd, Wd, w


def saved_views(saved, T, d, H):
    z = ((T * d * 2 + 255) // 256) * 256
    names = ["Zx", "Xt", "Q", "K", "Zq", "Zk", "Qr", "Kr", "V", "O"]
    out = {n: to_np(saved[i * z: i * z + T * d * 2].view(torch.bfloat16).view(T, d)) for i, n in enumerate(names)}
    out["lse"] = saved[10 * z: 10 * z + 4 * H * T].view(torch.float32).view(H, T).cpu().numpy().astype(np.float64)
    return out


LAYER_CASES = [
    ([64, 1, 33, 17], 32, 1, None, False),
    ([200, 77, 300], 128, 2, [0, 7, 30], False),
    ([300, 129, 700], 256, 2, None, True),
    ([513, 257, 1, 300], 352, 4, None, False),
    ([260, 5, 700], 512, 8, None, False),
]


@pytest.mark.parametrize("case", range(len(LAYER_CASES)))
def test_layer_forward_end_to_end(ops, case):
    """Protocol (iv): the bf16 layer output Y from X through the whole fp64 chain of Eqs. 3-7 (gated
    at 1e-2 / 1e-3 in the flat regime, reported in the peaky one).  The per-stage gates (protocol iii,
    on the fp32 accumulators) are in test_gpu_stages.py."""
    lengths, d, H, nc, peaky = LAYER_CASES[case]
    cu, t, s, ncv, T, X, W = layer_case(lengths, d, H, nc, seed=case, peaky=peaky)
    cfg = ops.config(d, H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4, rope_delta_t_max_ms=86_400_000)
    b = to_dev_batch(cu, t, s, ncv, T)
    Y, saved, ws, *_ = run_layer_forward(ops, cfg, b, X, W, T)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv)
    Wl = [w.astype(np.float64) for w in W.as_list()]
    n = cu[-1]
    Yg = to_np(Y)
    Yref, _, _ = O.batch_forward(X.astype(np.float64), Wl, meta, ocfg)
    mx, mn, rms = err_stats(Yg, Yref)
    print(f"[parity] e2e Y (bf16 pipeline): max {mx:.3e} mean {mn:.3e} rms {rms:.3f}")
    if not peaky:
        assert mx <= 1e-2 and mn <= 1e-3
    assert (Yg[n:] == 0).all()


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("case", range(len(LAYER_CASES)))
def test_layer_backward_end_to_end(ops, case, two_pass):
    """two_pass: the workspace holds the dS region, so dQ comes from the dS^T tiles the dK/dV kernel
    stored (attn_bwd_dq2_kernel) instead of the recomputing dQ kernel."""
    from paper_2602_11410_b200 import _lib as L
    lengths, d, H, nc, peaky = LAYER_CASES[case]
    cu, t, s, ncv, T, X, W = layer_case(lengths, d, H, nc, seed=20 + case, peaky=peaky)
    cfg = ops.config(d, H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4, rope_delta_t_max_ms=86_400_000)
    b = to_dev_batch(cu, t, s, ncv, T)
    Y, saved, ws, Xd, Wd, w = run_layer_forward(ops, cfg, b, X, W, T, two_pass=two_pass)
    dY = G.normal_bf16(99, case, (T, d))
    dY[cu[-1]:] = 0
    dYd = bf16_tensor(dY)
    dX = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    gs = [torch.empty(d, d, dtype=torch.float32, device="cuda") for _ in range(7)]
    g = L.AttnGrads(*[x.data_ptr() for x in gs])
    L.check(L.lib().cadet_attn_backward(C.byref(cfg), C.byref(b.struct()), C.byref(w), C.c_void_p(Xd.data_ptr()),
                                        C.c_void_p(saved.data_ptr()), C.c_void_p(dYd.data_ptr()),
                                        C.c_void_p(dX.data_ptr()), None, C.byref(g), C.c_void_p(ws.data_ptr()),
                                        ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ops.poll(ws)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv)
    Wl = [x.astype(np.float64) for x in W.as_list()]
    _, caches, _ = O.batch_forward(X.astype(np.float64), Wl, meta, ocfg)
    dXr, gWr, _ = O.batch_backward(caches, Wl, meta, dY.astype(np.float64), ocfg)
    res = {"dX": err_stats(to_np(dX), dXr)}
    for nm, gg, rr in zip(G.NAMES, gs, gWr):
        res["d" + nm] = err_stats(to_np(gg), rr)
    for k_, (mx, mn, rms) in res.items():
        print(f"e2e {k_}: max {mx:.3e} mean {mn:.3e} rms {rms:.3e}")
    # protocol (iv): bf16 end-to-end gradients are reported; gated at 5x the stage tolerance in
    # the flat regime and 10x in the peaky one (intermediate bf16 storage dominates)
    lim = (1e-1, 1e-2) if peaky else (5e-2, 5e-3)
    for k_, (mx, mn, rms) in res.items():
        assert mx <= lim[0] and mn <= lim[1], (k_, mx, mn)
    assert (to_np(dX)[cu[-1]:] == 0).all()


# ------------------------------------------------------------------ heads
def head_case(n_rows, T, d, K, dh, seed=0):
    rng = np.random.default_rng(seed)
    Hs = G.normal_bf16(seed, 3, (T, d))
    rows = np.sort(rng.choice(T, size=n_rows, replace=False)).astype(np.int32)
    hw = G.head_weights(seed, K, d, dh)
    bucket = rng.integers(0, K, size=n_rows).astype(np.int32)
    label = (rng.random(n_rows) < 0.3).astype(np.float32)
    W1cat = np.concatenate([hw.W1[k] for k in range(K)], axis=1)   # [d, K*dh]
    return Hs, rows, hw, W1cat, bucket, label


@pytest.mark.parametrize("n_rows,T,d,K,dh", [(37, 100, 64, 2, 32), (700, 1500, 256, 2, 128), (2000, 4000, 352, 3, 160),
                                            (999, 2100, 352, 2, 176)])
def test_heads_forward_backward(ops, n_rows, T, d, K, dh):
    from paper_2602_11410_b200 import _lib as L
    Hs, rows, hw, W1cat, bucket, label = head_case(n_rows, T, d, K, dh)
    hc = L.HeadConfig(K, d, dh, 0)
    Hd, W1d = bf16_tensor(Hs), bf16_tensor(W1cat)
    tens = {k: torch.tensor(v, device="cuda") for k, v in dict(
        b1=hw.b1.reshape(-1), w2=hw.w2.reshape(-1), b2=hw.b2, rows=rows, bucket=bucket, label=label).items()}
    hwst = L.HeadWeights(W1d.data_ptr(), tens["b1"].data_ptr(), tens["w2"].data_ptr(), tens["b2"].data_ptr())
    ws = ops.workspace(L.lib().cadet_heads_workspace_bytes(C.byref(hc), n_rows))
    logits = torch.empty(n_rows, K, dtype=torch.float32, device="cuda")
    pre = torch.empty(n_rows, K * dh, dtype=torch.bfloat16, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.check(L.lib().cadet_heads_forward(C.byref(hc), C.byref(hwst), C.c_void_p(Hd.data_ptr()),
                                        C.c_void_p(tens["rows"].data_ptr()), n_rows, C.c_void_p(logits.data_ptr()),
                                        C.c_void_p(pre.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), st))
    loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    dH = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    gr = [torch.empty(d, K * dh, dtype=torch.float32, device="cuda"),
          torch.empty(K * dh, dtype=torch.float32, device="cuda"),
          torch.empty(K * dh, dtype=torch.float32, device="cuda"), torch.empty(K, dtype=torch.float32, device="cuda")]
    hg = L.HeadGrads(*[x.data_ptr() for x in gr])
    L.check(L.lib().cadet_heads_loss_backward(C.byref(hc), C.byref(hwst), C.c_void_p(Hd.data_ptr()),
                                              C.c_void_p(tens["rows"].data_ptr()), n_rows, T,
                                              C.c_void_p(logits.data_ptr()), C.c_void_p(pre.data_ptr()),
                                              C.c_void_p(tens["bucket"].data_ptr()),
                                              C.c_void_p(tens["label"].data_ptr()), C.c_void_p(loss.data_ptr()),
                                              C.c_void_p(dH.data_ptr()), C.byref(hg), C.c_void_p(ws.data_ptr()),
                                              ws.numel(), st))
    torch.cuda.synchronize()
    ops.poll(ws)
    Lr, z, dHr, g = O.heads_loss_backward(Hs.astype(np.float64), rows, hw.W1.astype(np.float64),
                                          hw.b1.astype(np.float64), hw.w2.astype(np.float64),
                                          hw.b2.astype(np.float64), bucket, label.astype(np.float64))
    assert_close(logits.cpu().numpy(), z, what="logits")
    assert abs(loss.item() - Lr) <= 1e-3 * max(1.0, abs(Lr)), (loss.item(), Lr)
    assert_close(to_np(dH), dHr, what="dH")
    dW1r = np.concatenate([g["dW1"][k] for k in range(K)], axis=1)
    assert_close(gr[0].cpu().numpy(), dW1r, what="dW1")
    assert_close(gr[1].cpu().numpy(), g["db1"].reshape(-1), what="db1")
    assert_close(gr[2].cpu().numpy(), g["dw2"].reshape(-1), what="dw2")
    assert_close(gr[3].cpu().numpy(), g["db2"], what="db2")
    # rows_in_ws = 1: the backward reuses the forward's fp16 gathered rows and W1 copy in ws
    # (re-run the forward first: the first backward reused the slots); same results up to the
    # fp32 atomic order of the logits (tower partial dots) and of the split-K dW1
    L.check(L.lib().cadet_heads_forward(C.byref(hc), C.byref(hwst), C.c_void_p(Hd.data_ptr()),
                                        C.c_void_p(tens["rows"].data_ptr()), n_rows, C.c_void_p(logits.data_ptr()),
                                        C.c_void_p(pre.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), st))
    hc1 = L.HeadConfig(K, d, dh, 0, 1)
    dH1 = torch.empty_like(dH)
    gr1 = [torch.empty_like(x) for x in gr]
    hg1 = L.HeadGrads(*[x.data_ptr() for x in gr1])
    L.check(L.lib().cadet_heads_loss_backward(C.byref(hc1), C.byref(hwst), C.c_void_p(Hd.data_ptr()),
                                              C.c_void_p(tens["rows"].data_ptr()), n_rows, T,
                                              C.c_void_p(logits.data_ptr()), C.c_void_p(pre.data_ptr()),
                                              C.c_void_p(tens["bucket"].data_ptr()),
                                              C.c_void_p(tens["label"].data_ptr()), C.c_void_p(loss.data_ptr()),
                                              C.c_void_p(dH1.data_ptr()), C.byref(hg1), C.c_void_p(ws.data_ptr()),
                                              ws.numel(), st))
    torch.cuda.synchronize()
    assert float((dH1.float() - dH.float()).abs().max()) <= 1e-2 * max(1e-3, float(dH.float().abs().max()))
    for a_, b_ in zip(gr1, gr):
        assert float((a_ - b_).abs().max()) <= 1e-5 * max(1.0, float(b_.abs().max()))
