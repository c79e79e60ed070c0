"""GPU parity: tcgen05 GEMM, mask plan (bit-exact), chunk/pack (bit-exact), attention core
forward/backward vs the fp64 oracle.  Every call goes through the libcadet C ABI."""
import dataclasses
import math

import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G
from tests.helpers import (assert_close, bf16_tensor, err_stats, make_case, to_dev_batch, to_np)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ops():
    from paper_2602_11410_b200 import build, ops as _ops
    build.build()
    return _ops


def oracle_cfg(cfg):
    return O.AttnConfig(d_model=cfg.d_model, n_heads=cfg.n_heads, mask_flags=cfg.mask_flags,
                        delta_delay_ms=cfg.delta_delay_ms, delta_cand_ms=cfg.delta_cand_ms,
                        rope_dt_max_ms=cfg.rope_delta_t_max_ms, rope_phi_min=cfg.rope_phi_min,
                        rope_base=cfg.rope_base, use_rope=bool(cfg.use_rope), use_rep_gate=bool(cfg.use_rep_gate),
                        use_int_gate=bool(cfg.use_int_gate), use_out_proj=bool(cfg.use_out_proj))


def meta_of(cu, t, s, nc, n_static=None, flags=None):
    return O.SeqMeta(cu=cu.astype(np.int64), t_ms=t, n_cand=nc, session_ids=s, n_static=n_static,
                     pair_flags=flags)


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (304, 192, 200), (512, 512, 1024), (776, 768, 320),
                                   (512, 352, 352), (4352, 352, 352)])  # ragged N on the 128-wide CTA-pair tiles
def test_gemm_majors(ops, a_mn, b_mn, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    Ad = bf16_tensor(A.T.copy() if a_mn else A)
    Bd = bf16_tensor(B if b_mn else B.T.copy())
    Cg = ops.gemm(Ad, Bd, a_mn=bool(a_mn), b_mn=bool(b_mn), out_f32=True)
    torch.cuda.synchronize()
    ref = G.bf16_round(A).astype(np.float64) @ G.bf16_round(B).astype(np.float64)
    got = to_np(Cg)
    assert np.abs(got - ref).max() / max(1.0, np.abs(ref).max()) < 1e-4


def test_gemm_resid_bf16_out(ops):
    rng = np.random.default_rng(5)
    M, N, K = 256, 256, 128
    A = bf16_tensor(rng.standard_normal((M, K)))
    B = bf16_tensor(rng.standard_normal((N, K)))
    R = bf16_tensor(rng.standard_normal((M, N)))
    Cg = ops.gemm(A, B, out_f32=False, resid=R)
    ref = to_np(A) @ to_np(B).T + to_np(R)
    assert np.abs(to_np(Cg) - ref).max() < 0.02 * max(1, np.abs(ref).max())


# ------------------------------------------------------------------ mask plan (bit-exact)
PLAN_CASES = [
    # (lengths, n_cand, flags, delta, deltac, T extra)
    ([64, 1, 33, 17], None, 1, 120_000, 0, 13),
    ([64, 1, 33, 17], [0, 0, 8, 4], 1, 120_000, 0, 0),
    ([300, 129, 128, 127, 700], [0, 5, 0, 127, 64], 1, 60_000, 30_000, 100),
    ([300, 129, 700], None, 1 | 2, 60_000, 0, 5),
    ([513, 257, 1], [0, 0, 0], 1 | 4, 600_000, 0, 0),
]


@pytest.mark.parametrize("case", range(len(PLAN_CASES)))
def test_mask_plan_bit_exact(ops, case):
    lengths, nc, flags, dl, dc, extra = PLAN_CASES[case]
    cu, t, s, ncv, T = make_case(lengths, n_cand=nc)
    T = T + extra
    t = np.concatenate([t, np.zeros(extra, np.int64)]) if extra else t
    s = np.concatenate([s, np.zeros(extra, np.int32)]) if extra else s
    pf = (np.arange(T) % 2 == 1).astype(np.uint8) if flags & 4 else None
    cfg = ops.config(32, 1, mask_flags=flags, delta_delay_ms=dl, delta_cand_ms=dc)
    b = to_dev_batch(cu, t, s, ncv, T, flags=pf)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    cap = int(sum(((l + 127) // 128) ** 2 for l in lengths))
    kv_end, tc, pairs = ops.mask_export(cfg, b, ws, cap)
    ops.poll(ws)
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv, flags=pf)
    kv_ref, tc_ref, pairs_ref = O.mask_artifacts(meta, ocfg, T)
    assert (kv_end.cpu().numpy() == kv_ref).all()
    assert (tc.cpu().numpy() == tc_ref).all()
    assert int(pairs.item()) == pairs_ref


# (lengths, n_cand, flags, delta, n_static): static prefixes across a tile edge, pair flags on every
# odd row and on rows 128 k (the flagged i-1 cell in the previous tile), all three rules at once
PLAN_CASES_STATIC = [
    ([300, 129, 700], None, 1, 60_000, [130, 0, 5]),
    ([513, 257, 1], [0, 40, 0], 1 | 4, 600_000, [2, 129, 1]),
    ([400, 300, 129], [0, 50, 0], 1 | 2 | 4, 120_000, [0, 200, 128]),
    ([256, 256], None, 2, 0, [255, 1]),
]


@pytest.mark.parametrize("case", range(len(PLAN_CASES_STATIC)))
def test_mask_plan_static_prefix_and_tile_edge_pairs_bit_exact(ops, case):
    """n_static (R13) and PAIR_PREV (R12) with flagged rows at 128-row tile edges."""
    lengths, nc, flags, dl, nst = PLAN_CASES_STATIC[case]
    cu, t, s, ncv, T = make_case(lengths, n_cand=nc)
    pf = np.zeros(T, np.uint8)
    for a, e in zip(cu[:-1], cu[1:]):
        loc = np.arange(e - a)
        pf[a:e] = ((loc % 2 == 1) | ((loc % 128 == 0) & (loc > 0))).astype(np.uint8)
    nstv = np.asarray(nst, np.int32)
    cfg = ops.config(32, 1, mask_flags=flags, delta_delay_ms=dl)
    b = to_dev_batch(cu, t, s, ncv, T, n_static=nstv, flags=pf)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    cap = int(sum(((l + 127) // 128) ** 2 for l in lengths))
    kv_end, tc, pairs = ops.mask_export(cfg, b, ws, cap)
    ops.poll(ws)
    kv_ref, tc_ref, pairs_ref = O.mask_artifacts(meta_of(cu, t, s, ncv, n_static=nstv, flags=pf), oracle_cfg(cfg), T)
    assert (kv_end.cpu().numpy() == kv_ref).all()
    assert (tc.cpu().numpy() == tc_ref).all()
    assert int(pairs.item()) == pairs_ref


def test_mask_plan_fig3_and_tile_vector(ops):
    # Fig. 3 with one token per time unit and delay width 2
    cfg = ops.config(32, 1, delta_delay_ms=2)
    cu = np.array([0, 6], np.int32)
    t = np.array([0, 1, 2, 3, 5, 5], np.int64)
    b = to_dev_batch(cu, t, np.zeros(6, np.int32), np.array([2], np.int32), 6)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    kv, tc, pairs = ops.mask_export(cfg, b, ws, 1)
    # rows of Fig. 3: prefix ends 0,0,1,2,4,4 ; pairs = 1+1+2+3+5+5 = 17
    assert list(kv.cpu().numpy()) == [0, 0, 1, 2, 4, 4]
    assert int(pairs.item()) == 17
    # 256 context + 128 candidates, Delta = 0: SKIP (0,1),(0,2),(1,2); FULL (1,0),(2,0),(2,1)
    L_, N_ = 256, 128
    t = np.concatenate([np.repeat(np.arange(L_ // 2), 2), np.full(N_, 10_000)]).astype(np.int64)
    cfg = ops.config(32, 1, delta_delay_ms=0)
    b = to_dev_batch(np.array([0, 384], np.int32), t, np.zeros(384, np.int32), np.array([128], np.int32), 384)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    kv, tc, pairs = ops.mask_export(cfg, b, ws, 9)
    assert list(tc.cpu().numpy()) == [1, 0, 0, 2, 1, 0, 2, 2, 1]
    assert int(pairs.item()) == 65792


def test_mask_plan_detects_order_error(ops):
    from paper_2602_11410_b200 import _lib
    cfg = ops.config(32, 1)
    t = np.array([5, 4, 6], np.int64)
    b = to_dev_batch(np.array([0, 3], np.int32), t, np.zeros(3, np.int32), np.zeros(1, np.int32), 3)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    with pytest.raises(_lib.CadetError) as e:
        ops.poll(ws)
    assert e.value.status == 3


# ------------------------------------------------------------------ chunk / pack (bit-exact)
def test_chunk_bit_exact(ops):
    rng = np.random.default_rng(3)
    lens = np.concatenate([[10, 8, 4096, 1, 2049], rng.integers(1, 9000, size=200)])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ref = O.chunk_offsets(cu, 2048)
    cu_d = torch.tensor(cu, device="cuda")
    out, n, ws = ops.chunk(cu_d, 2048, len(ref) + 5)
    ops.poll(ws)
    assert int(n.item()) == len(ref) - 1
    assert (out[: len(ref)].cpu().numpy() == ref).all()
    out, n, ws = ops.chunk(torch.tensor([0, 10], dtype=torch.int32, device="cuda"), 4, 8)
    assert list(out[:4].cpu().numpy()) == [0, 2, 6, 10]


def test_pack_bit_exact(ops):
    rng = np.random.default_rng(4)
    for lens, budget in (([5, 3, 6], 16), ([10, 10], 16), ([7, 1, 9, 3, 4], 20)):
        B, Lmax, d = len(lens), max(lens), 64
        X = rng.standard_normal((B, Lmax, d)).astype(np.float32)
        tp = rng.integers(0, 10**12, size=(B, Lmax)).astype(np.int64)
        src_row = torch.arange(B, dtype=torch.int64, device="cuda") * Lmax
        packed, t_out, s_out, cu, n_packed, ws = ops.pack(bf16_tensor(X.reshape(B * Lmax, d)),
                                                          torch.tensor(lens, dtype=torch.int32, device="cuda"),
                                                          budget, src_row=src_row, t_src=torch.tensor(tp, device="cuda"))
        ops.poll(ws)
        cu_ref, nref, pad = O.pack_greedy(lens, budget)
        k = int(n_packed.item())
        assert k == nref and list(cu.cpu().numpy()[: k + 1]) == list(cu_ref)
        P = to_np(packed)
        Xb = G.bf16_round(X)
        for s_ in range(k):
            assert (P[cu_ref[s_]:cu_ref[s_ + 1]] == Xb[s_, : lens[s_]]).all()
            assert (t_out.cpu().numpy()[cu_ref[s_]:cu_ref[s_ + 1]] == tp[s_, : lens[s_]]).all()
        assert (P[cu_ref[-1]:] == 0).all() and budget - cu_ref[-1] == pad
    # contiguous histories (src_row = NULL): packed rows are the source rows
    lens = [5, 3, 6, 4]
    X = rng.standard_normal((18, 32)).astype(np.float32)
    packed, *_rest, n_packed, ws = ops.pack(bf16_tensor(X), torch.tensor(lens, dtype=torch.int32, device="cuda"), 16)
    assert int(n_packed.item()) == 3
    assert (to_np(packed)[:14] == G.bf16_round(X[:14])).all() and (to_np(packed)[14:] == 0).all()


def test_pack_split_modes_match_the_full_pack(ops):
    """cadet_pack with src = packed = NULL (offsets + timestamps / sessions only, one thread per row)
    and with t / s NULL (offsets + rows only) together reproduce the full call bit for bit — the
    split CadetStack uses to move the rows on a side stream."""
    import ctypes as C
    from paper_2602_11410_b200 import _lib as L
    rng = np.random.default_rng(9)
    lens = [513, 1, 77, 300, 129, 1000]
    R, d, budget = sum(lens), 64, 1500
    X = bf16_tensor(rng.standard_normal((R, d)).astype(np.float32))
    tp = torch.tensor(rng.integers(0, 10**12, size=R), dtype=torch.int64, device="cuda")
    sp = torch.tensor(rng.integers(0, 50, size=R), dtype=torch.int32, device="cuda")
    ln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    full = ops.pack(X, ln, budget, t_src=tp, s_src=sp)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    ws = ops.workspace(L.lib().cadet_pack_workspace_bytes(len(lens)))
    t_out = torch.full((budget,), -1, dtype=torch.int64, device="cuda")
    s_out = torch.full((budget,), -1, dtype=torch.int32, device="cuda")
    cu1 = torch.empty(len(lens) + 1, dtype=torch.int32, device="cuda")
    n1 = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.check(L.lib().cadet_pack(None, None, vp(ln), len(lens), d, budget, vp(tp), vp(sp), None, vp(t_out), vp(s_out),
                               vp(cu1), vp(n1), vp(ws), ws.numel(), st))
    rows = torch.full((budget, d), 7.0, dtype=torch.bfloat16, device="cuda")
    cu2 = torch.empty(len(lens) + 1, dtype=torch.int32, device="cuda")
    n2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.check(L.lib().cadet_pack(vp(X), None, vp(ln), len(lens), d, budget, None, None, vp(rows), None, None, vp(cu2),
                               vp(n2), vp(ws), ws.numel(), st))
    ops.poll(ws)
    packed, t_full, s_full, cu, n_packed, _ = full
    assert torch.equal(n1, n_packed) and torch.equal(n2, n_packed)
    k = int(n_packed.item())
    assert torch.equal(cu1[: k + 1], cu[: k + 1]) and torch.equal(cu2[: k + 1], cu[: k + 1])
    assert torch.equal(t_out, t_full) and torch.equal(s_out, s_full)
    assert torch.equal(rows, packed)
    # one of src / packed alone is an argument error
    with pytest.raises(L.CadetError):
        L.check(L.lib().cadet_pack(vp(X), None, vp(ln), len(lens), d, budget, vp(tp), vp(sp), None, vp(t_out),
                                   vp(s_out), vp(cu1), vp(n1), vp(ws), ws.numel(), st))


# ------------------------------------------------------------------ attention core forward
def core_case(lengths, d, H, nc=None, scale=1.0, seed=0, flags=1, dl=120_000, T_extra=7):
    cu, t, s, ncv, T = make_case(lengths, n_cand=nc, seed=seed)
    T = T + T_extra
    t = np.concatenate([t, np.zeros(T_extra, np.int64)])
    s = np.concatenate([s, np.zeros(T_extra, np.int32)])
    rng = np.random.default_rng(seed + 100)
    Qr = G.bf16_round(rng.standard_normal((T, d)).astype(np.float32) * scale)
    Kr = G.bf16_round(rng.standard_normal((T, d)).astype(np.float32) * scale)
    V = G.bf16_round(rng.standard_normal((T, d)).astype(np.float32))
    return cu, t, s, ncv, T, Qr, Kr, V


CORE_CASES = [
    # lengths, d, H, n_cand, scale
    ([64, 1, 33, 17], 32, 1, None, 1.0),
    ([64, 1, 33, 17], 32, 1, [0, 0, 8, 4], 1.0),
    ([300, 129, 128, 127, 700], 128, 2, [0, 5, 0, 127, 64], 1.0),
    ([300, 129, 700], 256, 2, None, 2.0),
    ([513, 257, 1, 900], 352, 4, None, 1.0),
    ([400, 1000], 384, 4, [0, 100], 1.5),
    ([260, 5, 700], 512, 8, None, 1.0),
]


@pytest.mark.parametrize("paired", [False, True], ids=["one_tile_per_cta", "paired_persistent"])
@pytest.mark.parametrize("case", range(len(CORE_CASES)))
def test_attn_core_forward(ops, case, paired, monkeypatch):
    # paired: the opt-in persistent kernel (two q-tiles of a sequence share one K / V stream), read per launch
    if paired:
        monkeypatch.setenv("CADET_FWD_PAIRED", "1")
    lengths, d, H, nc, scale = CORE_CASES[case]
    cu, t, s, ncv, T, Qr, Kr, V = core_case(lengths, d, H, nc, scale, seed=case)
    cfg = ops.config(d, H, delta_delay_ms=120_000, out_f32=1)
    b = to_dev_batch(cu, t, s, ncv, T)
    Og, lseg = ops.attn_core_forward(cfg, b, bf16_tensor(Qr), bf16_tensor(Kr), bf16_tensor(V))
    torch.cuda.synchronize()
    ocfg = oracle_cfg(cfg)
    meta = meta_of(cu, t, s, ncv)
    Oref = np.zeros((T, d))
    lref = np.zeros((H, T))
    for k in range(len(lengths)):
        a, e = cu[k], cu[k + 1]
        A = O.seq_mask(meta, k, ocfg)
        o, l, _ = O.attention_core_forward(Qr[a:e].astype(np.float64), Kr[a:e].astype(np.float64),
                                           V[a:e].astype(np.float64), A, H)
        Oref[a:e] = o
        lref[:, a:e] = l
    assert_close(to_np(Og), Oref, what="O")
    assert_close(to_np(lseg), lref, what="LSE")
    assert (to_np(Og)[cu[-1]:] == 0).all()


# ------------------------------------------------------------------ device-latched input errors (cadet.h)
@pytest.mark.parametrize("kind", ["offsets_start", "offsets_decreasing", "offsets_past_T", "too_long", "cand"])
def test_mask_plan_device_latches(ops, kind):
    """Each device-detected input error of cadet_mask_plan latches its bit and cadet_poll returns it
    (then clears it): OFFSETS, TOO_LONG, CAND."""
    from paper_2602_11410_b200 import _lib
    T = 300
    cu = np.array([0, 100, 250], np.int32)
    nc = np.zeros(2, np.int32)
    maxlen = 256
    want = {"offsets_start": 2, "offsets_decreasing": 2, "offsets_past_T": 2, "too_long": 4, "cand": 5}[kind]
    if kind == "offsets_start":
        cu = np.array([1, 100, 250], np.int32)
    elif kind == "offsets_decreasing":
        cu = np.array([0, 100, 90], np.int32)
    elif kind == "offsets_past_T":
        cu = np.array([0, 100, 301], np.int32)
    elif kind == "too_long":
        maxlen = 120
    elif kind == "cand":
        nc = np.array([0, 151], np.int32)
    t = np.arange(T, dtype=np.int64) * 1000
    cfg = ops.config(32, 1)
    b = to_dev_batch(cu, t, np.zeros(T, np.int32), nc, T, max_seqlen=maxlen)
    ws = ops.plan_workspace(b)
    ops.mask_plan(cfg, b, ws)
    with pytest.raises(_lib.CadetError) as e:
        ops.poll(ws)
    assert e.value.status == want
    ops.poll(ws)  # the word was cleared


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("kind", ["bucket", "nonfinite"])
def test_heads_device_latches(ops, kind, dtype):
    """Routed BCE (Eq. 9): a bucket outside [0, K) latches BUCKET ("routing error"); a non-finite
    loss latches NONFINITE (fail-fast numerics).  bf16 and fp32 towers."""
    import ctypes as C
    from paper_2602_11410_b200 import _lib as L
    n, T, d, K, dh = 40, 64, 64, 2, 32
    rng = np.random.default_rng(1)
    el = torch.float32 if dtype else torch.bfloat16
    Hs = torch.tensor(rng.standard_normal((T, d)), dtype=torch.float32, device="cuda").to(el)
    W1 = torch.tensor(rng.standard_normal((d, K * dh)) * 0.1, dtype=torch.float32, device="cuda").to(el)
    b1, w2 = (torch.zeros(K * dh, device="cuda") for _ in range(2))
    b2 = torch.zeros(K, device="cuda")
    rows = torch.arange(n, dtype=torch.int32, device="cuda")
    bucket = torch.zeros(n, dtype=torch.int32, device="cuda")
    label = torch.zeros(n, device="cuda")
    logits = torch.zeros(n, K, device="cuda")
    if kind == "bucket":
        bucket[7] = K
    else:
        logits[3, 0] = float("nan")
    hc = L.HeadConfig(K, d, dh, dtype)
    hw = L.HeadWeights(W1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr())
    ws = ops.workspace(L.lib().cadet_heads_workspace_bytes(C.byref(hc), n))
    ws.zero_()
    pre = torch.zeros(n, K * dh, dtype=el, device="cuda")
    loss = torch.zeros(1, device="cuda")
    dH = torch.empty(T, d, dtype=el, device="cuda")
    gr = [torch.empty(d, K * dh, device="cuda"), torch.empty(K * dh, device="cuda"), torch.empty(K * dh, device="cuda"),
          torch.empty(K, device="cuda")]
    hg = L.HeadGrads(*[x.data_ptr() for x in gr])
    L.check(L.lib().cadet_heads_loss_backward(C.byref(hc), C.byref(hw), C.c_void_p(Hs.data_ptr()),
                                              C.c_void_p(rows.data_ptr()), n, T, C.c_void_p(logits.data_ptr()),
                                              C.c_void_p(pre.data_ptr()), C.c_void_p(bucket.data_ptr()),
                                              C.c_void_p(label.data_ptr()), C.c_void_p(loss.data_ptr()),
                                              C.c_void_p(dH.data_ptr()), C.byref(hg), C.c_void_p(ws.data_ptr()),
                                              ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    with pytest.raises(L.CadetError) as e:
        ops.poll(ws)
    assert e.value.status == (6 if kind == "bucket" else 7)


@pytest.mark.parametrize("bnd", [(4,), (1, 4), (2, 3, 7, 20), tuple(range(1, 33))])
def test_bucketize_bit_exact(ops, bnd):
    """cadet_bucketize vs oracle.bucketize: bit-exact; a position < 1 latches
    CADET_E_BUCKET."""
    import ctypes as C
    from paper_2602_11410_b200 import _lib as L
    rng = np.random.default_rng(len(bnd))
    pos = rng.integers(1, 40, size=10_007).astype(np.int32)
    pd = torch.tensor(pos, device="cuda")
    out = torch.full((pos.size,), -1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    arr = (C.c_int32 * len(bnd))(*bnd)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.check(L.lib().cadet_bucketize(C.c_void_p(pd.data_ptr()), pos.size, arr, len(bnd), C.c_void_p(out.data_ptr()),
                                    C.c_void_p(ws.data_ptr()), st))
    ops.poll(ws)
    assert (out.cpu().numpy() == O.bucketize(pos, bnd)).all()
    pd[5] = 0
    L.check(L.lib().cadet_bucketize(C.c_void_p(pd.data_ptr()), pos.size, arr, len(bnd), C.c_void_p(out.data_ptr()),
                                    C.c_void_p(ws.data_ptr()), st))
    with pytest.raises(L.CadetError) as e:
        ops.poll(ws)
    assert e.value.status == 6
