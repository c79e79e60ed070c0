"""NEXT-2 GPU parity: the full loss of PAPER.md Eqs. 10-12 through the C ABI —
tower and auxiliary-head forwards, routed logits, RankNet pairwise term, Eq. 11 logit gradients,
tower / aux backward from the logit gradients — against oracle.full_loss_backward; and the
cross-rank pairwise formulation (each rank's samples against the gathered batch) reproducing the
global Eq. 12 loss and gradient when the shares are summed / concatenated."""
import ctypes as C

import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G
from tests.helpers import assert_close, assert_close_stored, bf16_tensor, to_np

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    from paper_2602_11410_b200 import _lib, build
    build.build()
    return _lib


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _heads(L, hc, Wcat, b1, w2, b2):
    t = {k: torch.tensor(v, device="cuda") for k, v in dict(b1=b1.reshape(-1), w2=w2.reshape(-1), b2=b2).items()}
    Wd = bf16_tensor(Wcat)
    return L.HeadWeights(Wd.data_ptr(), t["b1"].data_ptr(), t["w2"].data_ptr(), t["b2"].data_ptr()), (Wd, t)


@pytest.mark.parametrize("n_rows,T,d,K,dh,J,da", [(700, 1500, 256, 2, 128, 2, 64), (2000, 4000, 352, 2, 176, 2, 96)])
def test_full_loss_matches_oracle(L, n_rows, T, d, K, dh, J, da):
    lib = L.lib()
    rng = np.random.default_rng(n_rows)
    Hs = G.normal_bf16(3, 5, (T, d))
    rows = np.sort(rng.choice(T, size=n_rows, replace=False)).astype(np.int32)
    hw = G.head_weights(1, K, d, dh)
    aw = G.head_weights(2, J, d, da)
    bucket = rng.integers(0, K, size=n_rows).astype(np.int32)
    label = (rng.random(n_rows) < 0.3).astype(np.float32)
    ya = G.aux_labels(4, n_rows)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    Hd = bf16_tensor(Hs)
    rows_d = torch.tensor(rows, device="cuda")
    outs = {}
    for name, w, KK, hid in (("ctx", hw, K, dh), ("aux", aw, J, da)):
        hc = L.HeadConfig(KK, d, hid, 0)
        wst, keep = _heads(L, hc, np.concatenate([w.W1[k] for k in range(KK)], axis=1), w.b1, w.w2, w.b2)
        ws = torch.zeros(lib.cadet_heads_workspace_bytes(C.byref(hc), n_rows), dtype=torch.uint8, device="cuda")
        logits = torch.empty(n_rows, KK, dtype=torch.float32, device="cuda")
        pre = torch.empty(n_rows, KK * hid, dtype=torch.bfloat16, device="cuda")
        L.check(lib.cadet_heads_forward(C.byref(hc), C.byref(wst), _vp(Hd), _vp(rows_d), n_rows, _vp(logits),
                                        _vp(pre), _vp(ws), ws.numel(), st))
        outs[name] = (hc, wst, keep, ws, logits, pre, KK, hid)
    lc = L.LossConfig()
    lib.cadet_default_loss_config(C.byref(lc), J)
    lc.lambda_pair = 0.5  # larger than the default so the pairwise term is visible in the gradients
    bucket_d, label_d = torch.tensor(bucket, device="cuda"), torch.tensor(label, device="cuda")
    ya_d = torch.tensor(ya, device="cuda")
    zr = torch.empty(n_rows, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_routed_logits(_vp(outs["ctx"][4]), K, _vp(bucket_d), n_rows, _vp(zr), st))
    pws = torch.zeros(lib.cadet_pairwise_workspace_bytes(n_rows, n_rows), dtype=torch.uint8, device="cuda")
    share = torch.zeros(1, dtype=torch.float32, device="cuda")
    dzp = torch.empty(n_rows, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_pairwise_loss(_vp(zr), _vp(label_d), n_rows, _vp(zr), _vp(label_d), n_rows, _vp(share), _vp(dzp),
                                    _vp(pws), pws.numel(), st))
    losses = torch.empty(J + 3, dtype=torch.float32, device="cuda")
    dz_ctx = torch.empty(n_rows, K, dtype=torch.float32, device="cuda")
    dz_aux = torch.empty(n_rows, J, dtype=torch.float32, device="cuda")
    L.check(lib.cadet_full_loss_grads(C.byref(lc), _vp(outs["ctx"][4]), K, _vp(bucket_d), _vp(label_d), _vp(dzp),
                                      _vp(share), _vp(outs["aux"][4]), _vp(ya_d), n_rows, _vp(losses), _vp(dz_ctx),
                                      _vp(dz_aux), st))
    dHs = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    grads = {}
    for name, dz, acc in (("ctx", dz_ctx, 0), ("aux", dz_aux, 1)):
        hc, wst, keep, ws, logits, pre, KK, hid = outs[name]
        gr = [torch.empty(d, KK * hid, dtype=torch.float32, device="cuda"),
              torch.empty(KK * hid, dtype=torch.float32, device="cuda"),
              torch.empty(KK * hid, dtype=torch.float32, device="cuda"), torch.empty(KK, dtype=torch.float32, device="cuda")]
        hg = L.HeadGrads(*[x.data_ptr() for x in gr])
        L.check(lib.cadet_heads_backward(C.byref(hc), C.byref(wst), _vp(Hd), _vp(rows_d), n_rows, T, _vp(pre), _vp(dz),
                                         acc, _vp(dHs), C.byref(hg), _vp(ws), ws.numel(), st))
        grads[name] = gr
    torch.cuda.synchronize()
    f64 = lambda w: (w.W1.astype(np.float64), w.b1.astype(np.float64), w.w2.astype(np.float64), w.b2.astype(np.float64))
    lam = (1.0, tuple(lc.lambda_aux[j] for j in range(J)), 0.5)
    terms, dHr, gc, ga = O.full_loss_backward(Hs.astype(np.float64), rows, f64(hw), f64(aw), bucket,
                                              label.astype(np.float64), ya.astype(np.float64), lam)
    lg = losses.cpu().numpy().astype(np.float64)
    assert lg[0] == pytest.approx(terms["ctx"], rel=1e-3)
    for j in range(J):
        assert lg[1 + j] == pytest.approx(terms["aux"][j], rel=1e-3)
    assert lg[J + 1] == pytest.approx(terms["pair"], rel=1e-4)
    assert lg[J + 2] == pytest.approx(terms["total"], rel=1e-3)
    # the pairwise gradient itself (fp32 sums of fp32 logits) against the oracle's adjoint of the GPU logits
    zg = zr.cpu().numpy().astype(np.float64)
    gp, gn = O.pairwise_grad(zg[label > 0.5], zg[label <= 0.5])
    dzp_ref = np.zeros(n_rows)
    dzp_ref[label > 0.5], dzp_ref[label <= 0.5] = gp, gn
    assert np.abs(dzp.cpu().numpy() - dzp_ref).max() <= 1e-4 * np.abs(dzp_ref).max()
    assert_close_stored(to_np(dHs), dHr, what="dH (towers + aux)")
    for name, g, ref in (("ctx", grads["ctx"], gc), ("aux", grads["aux"], ga)):
        KK = K if name == "ctx" else J
        assert_close(g[0].cpu().numpy(), np.concatenate([ref["dW1"][k] for k in range(KK)], axis=1), what=f"{name} dW1")
        assert_close(g[1].cpu().numpy(), ref["db1"].reshape(-1), what=f"{name} db1")
        assert_close(g[2].cpu().numpy(), ref["dw2"].reshape(-1), what=f"{name} dw2")
        assert_close(g[3].cpu().numpy(), ref["db2"], what=f"{name} db2")


def test_pairwise_cross_rank_shares_reproduce_the_global_loss(L):
    """R29 data-parallel form: each 'rank' (slices of one batch) pairs its samples against the gathered
    batch; the shares sum to Eq. 12 and the concatenated dz equals the global adjoint."""
    lib = L.lib()
    rng = np.random.default_rng(11)
    n = 5000
    z = rng.normal(size=n).astype(np.float32) * 2
    y = (rng.random(n) < 0.25).astype(np.float32)
    zd, yd = torch.tensor(z, device="cuda"), torch.tensor(y, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    cuts = [0, 1234, 3000, n]
    shares, dzs = [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        m = b - a
        ws = torch.zeros(lib.cadet_pairwise_workspace_bytes(m, n), dtype=torch.uint8, device="cuda")
        sh = torch.zeros(1, dtype=torch.float32, device="cuda")
        dz = torch.empty(m, dtype=torch.float32, device="cuda")
        L.check(lib.cadet_pairwise_loss(_vp(zd[a:b]), _vp(yd[a:b]), m, _vp(zd), _vp(yd), n, _vp(sh), _vp(dz), _vp(ws),
                                        ws.numel(), st))
        shares.append(sh)
        dzs.append(dz)
    torch.cuda.synchronize()
    zf = z.astype(np.float64)
    ref = O.pairwise_loss(zf[y > 0.5], zf[y <= 0.5])
    assert sum(float(s.item()) for s in shares) == pytest.approx(ref, rel=1e-5)
    gp, gn = O.pairwise_grad(zf[y > 0.5], zf[y <= 0.5])
    g = np.zeros(n)
    g[y > 0.5], g[y <= 0.5] = gp, gn
    got = torch.cat(dzs).cpu().numpy()
    assert np.abs(got - g).max() <= 1e-5 * np.abs(g).max()
