"""Pins for the fp64 CPU oracle (runs without a GPU: -m "not gpu").

Each test pins the oracle to something other than itself: values printed in
PAPER.md/SPEC.md (golden fixtures under tests/golden/), closed forms, special
cases that reduce to a library routine (torch SDPA), an independent per-element
loop, and central finite differences.  Citations: P:n = PAPER.md line,
S:n = SPEC.md line.
"""
import dataclasses
import math
import os

import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_bits(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line)
    return rows


# ---------------------------------------------------------------- mask pins
def test_fig3_mask_bit_exact():
    """Fig. 3: 4 train tokens + 2 val/candidate tokens, delay width 2 (in
    timestamp units with one token per time unit)."""
    want = np.array([[c == "1" for c in r] for r in _read_bits("fig3_mask.txt")])
    t = np.array([0, 1, 2, 3, 5, 5], dtype=np.int64)
    cfg = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=2, delta_cand_ms=0)
    A = O.mask_dense(t, 2, cfg)
    assert (A == want).all()


def test_fig3_striped_cells_are_the_delta_difference():
    """Striped cells: allowed causally (Delta=0) but masked in training."""
    want = {tuple(map(int, r.split())) for r in _read_bits("fig3_striped.txt")}
    t = np.array([0, 1, 2, 3, 5, 5], dtype=np.int64)
    cfg2 = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=2)
    cfg0 = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=0)
    A2, A0 = O.mask_dense(t, 2, cfg2), O.mask_dense(t, 2, cfg0)
    got = {(i, j) for i in range(4) for j in range(4) if A0[i, j] and not A2[i, j]}
    assert got == want


def test_eq6_substitution_examples():
    """t_i=7.2e6, t_j=3.5e6, Delta=3.6e6 -> allowed; t_j=3.7e6 -> masked."""
    cfg = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=3_600_000)
    A = O.mask_dense(np.array([3_500_000, 7_200_000]), 0, cfg)
    assert A[1, 0]
    A = O.mask_dense(np.array([3_700_000, 7_200_000]), 0, cfg)
    assert not A[1, 0]
    # tie t_j = t_i - Delta is allowed (R9)
    A = O.mask_dense(np.array([3_600_000, 7_200_000]), 0, cfg)
    assert A[1, 0]


def test_candidate_pattern_example():
    """L=3, N=2 -> query 4 sees {1,2,3,4}, query 5 sees {1,2,3,5} (1-indexed)."""
    cfg = O.AttnConfig(d_model=2, n_heads=1, mask_flags=O.MASK_TIME, delta_delay_ms=0)
    A = O.mask_dense(np.array([0, 1, 2, 10, 10]), 2, cfg)
    assert set(np.nonzero(A[3])[0] + 1) == {1, 2, 3, 4}
    assert set(np.nonzero(A[4])[0] + 1) == {1, 2, 3, 5}
    # context rows are causal (Delta=0)
    assert (A[:3, :3] == np.tril(np.ones((3, 3), bool))).all()


def _fixture(name):
    """Golden mask fixture: 'key v v ...' header lines, then 0/1 rows (hand-worked, cited inside)."""
    meta, rows = {}, []
    for line in _read_bits(name):
        parts = line.split()
        if parts[0][0].isalpha():
            meta[parts[0]] = [int(v) for v in parts[1:]]
        else:
            rows.append(line)
    return meta, np.array([[c == "1" for c in r] for r in rows])


def test_session_mask_hand_worked():
    """R10 reading of P:288-290 (same-session information hidden): SESSION-only rule, by hand."""
    meta, want = _fixture("session_mask.txt")
    m = len(meta["sessions"])
    cfg = O.AttnConfig(d_model=2, n_heads=1, mask_flags=O.MASK_SESSION)
    A = O.mask_dense(np.zeros(m, np.int64), 0, cfg, session_ids=np.array(meta["sessions"]))
    assert (A == want).all()


def test_session_and_time_rules_combine_by_and():
    """Both flags = AND of Eq. 6 and the session rule (R10), by hand."""
    meta, want = _fixture("session_time_and.txt")
    cfg = O.AttnConfig(d_model=2, n_heads=1, mask_flags=O.MASK_TIME | O.MASK_SESSION,
                       delta_delay_ms=meta["delta"][0])
    A = O.mask_dense(np.array(meta["times"]), 0, cfg, session_ids=np.array(meta["sessions"]))
    assert (A == want).all()
    # each rule alone is a superset of the combination
    At = O.mask_dense(np.array(meta["times"]), 0, dataclasses.replace(cfg, mask_flags=O.MASK_TIME))
    As = O.mask_dense(np.array(meta["times"]), 0, dataclasses.replace(cfg, mask_flags=O.MASK_SESSION),
                      session_ids=np.array(meta["sessions"]))
    assert (A == (At & As)).all() and not (A == At).all() and not (A == As).all()


def test_pair_prev_exception_hand_worked():
    """S:310 (action token sees its own impression; reading R12), by hand; without the flag the
    paper-literal rule hides exactly the flagged i-1 cells."""
    meta, want = _fixture("pair_prev_mask.txt")
    t, fl = np.array(meta["times"]), np.array(meta["flags"], np.uint8)
    cfg = O.AttnConfig(d_model=2, n_heads=1, mask_flags=O.MASK_TIME | O.MASK_PAIR_PREV,
                       delta_delay_ms=meta["delta"][0])
    A = O.mask_dense(t, 0, cfg, pair_flags=fl)
    assert (A == want).all()
    Alit = O.mask_dense(t, 0, dataclasses.replace(cfg, mask_flags=O.MASK_TIME))
    diff = {(i, j) for i in range(len(t)) for j in range(len(t)) if A[i, j] != Alit[i, j]}
    assert diff == {(1, 0), (3, 2), (5, 4)}
    # canonical kv_end (R24) is taken from the mask WITHOUT the exception: the prefix ends
    assert list(O.kv_end_local(Alit)) == [0, 0, 2, 2, 2, 2]


def test_static_prefix_always_visible_hand_worked():
    """S:319 / R13: the static prefix M (Eq. 1) is visible to every context query."""
    meta, want = _fixture("static_prefix_mask.txt")
    cfg = O.AttnConfig(d_model=2, n_heads=1, mask_flags=O.MASK_TIME, delta_delay_ms=meta["delta"][0])
    A = O.mask_dense(np.array(meta["times"]), 0, cfg, n_static=meta["n_static"][0])
    assert (A == want).all()
    # n_static = 0 leaves only the diagonal (all timestamps equal, Delta > 0)
    A0 = O.mask_dense(np.array(meta["times"]), 0, cfg, n_static=0)
    assert (A0 == np.eye(len(meta["times"]), dtype=bool)).all()


@pytest.mark.parametrize("L,N", [(0, 1), (1, 0), (3, 2), (7, 5), (16, 9), (40, 0), (33, 17)])
def test_pair_count_closed_form(L, N):
    """allowed pairs of the inference pattern = L(L+1)/2 + N(L+1) (brute count)."""
    cfg = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=0)
    t = np.concatenate([np.arange(L), np.full(N, L + 5)]).astype(np.int64)
    A = O.mask_dense(t, N, cfg)
    assert int(A.sum()) == O.count_pairs_inference(L, N)


def test_pair_count_paper_scale():
    """L=4096, N=512 -> 10,488,320 (paper's L^2/2+LN = 10,485,760 within 0.1%)."""
    assert O.count_pairs_inference(4096, 512) == 10_488_320
    assert abs(O.count_pairs_inference(4096, 512) - (4096 ** 2 // 2 + 4096 * 512)) / 10_488_320 < 1e-3


def test_delta_zero_is_causal():
    """Delta=0 degrades to the causal mask."""
    cfg = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=0)
    b = G.fixed_lengths_batch([37])
    A = O.mask_dense(b.timestamps, 0, cfg)
    assert (A == np.tril(np.ones((37, 37), bool))).all()


def test_tile_vector_256_128():
    rows = _read_bits("tile_vector_256_128.txt")
    want = np.array([list(map(int, r.split())) for r in rows[:3]], dtype=np.int8)
    pairs = int(rows[3].split()[1])
    L, N = 256, 128
    t = np.concatenate([np.repeat(np.arange(L // 2), 2), np.full(N, 10_000)]).astype(np.int64)
    cfg = O.AttnConfig(d_model=2, n_heads=1, delta_delay_ms=0)
    A = O.mask_dense(t, N, cfg)
    assert (O.tile_classes(A, 128) == want).all()
    assert int(A.sum()) == pairs == O.count_pairs_inference(L, N)


def test_mask_artifacts_structure_on_generator_batch():
    b = G.fixed_lengths_batch([64, 1, 33, 17], cfg=G.stress_config())
    cu = np.concatenate([[0], np.cumsum(b.lengths)])
    meta = O.SeqMeta(cu=cu, t_ms=b.timestamps, n_cand=np.array([0, 0, 8, 4]))
    cfg = O.AttnConfig(d_model=32, n_heads=1, delta_delay_ms=120_000)
    kv_end, tiles, pairs = O.mask_artifacts(meta, cfg, 128)
    assert kv_end.shape == (128,) and (kv_end[cu[-1]:] == np.arange(cu[-1], 128)).all()
    assert (kv_end[: cu[-1]] <= np.arange(cu[-1])).all()
    assert tiles.shape == (4,)
    assert pairs >= cu[-1]


# ---------------------------------------------------------------- batching pins
def test_pack_example():
    """S:527 / Fig. 4: lengths [5,3,6], budget 16 -> offsets [0,5,8,14], pad 2."""
    cu, n, pad = O.pack_greedy([5, 3, 6], 16)
    assert list(cu) == [0, 5, 8, 14] and n == 3 and pad == 2
    cu, n, pad = O.pack_greedy([10, 10], 16)      # S:528 greedy split
    assert list(cu) == [0, 10] and n == 1 and pad == 6
    cu, n, pad = O.pack_greedy([], 16)
    assert list(cu) == [0] and n == 0 and pad == 16


def test_chunk_examples():
    """L=10, Lc=4 -> [6,10), [2,6), [0,2); L=8 -> 2 full chunks."""
    assert list(O.chunk_offsets(np.array([0, 10]), 4)) == [0, 2, 6, 10]
    assert list(O.chunk_offsets(np.array([0, 8]), 4)) == [0, 4, 8]
    out = O.chunk_offsets(np.array([0, 10, 13, 4109]), 2048)
    assert list(out) == [0, 10, 13, 2061, 4109]
    # count = ceil(L / Lc) per sequence; round trip covers every token once
    rng = np.random.default_rng(0)
    lens = rng.integers(1, 50, size=20)
    cu = np.concatenate([[0], np.cumsum(lens)])
    out = O.chunk_offsets(cu, 7)
    assert len(out) - 1 == int(sum(-(-l // 7) for l in lens))
    assert set(cu).issubset(set(out)) and (np.diff(out) > 0).all() and (np.diff(out) <= 7).all()


# ---------------------------------------------------------------- RoPE pins
def test_rope_theta0_paper_constants():
    """theta_0 = 1e-4 / 31,536,000,000 = 3.17098e-15 rad/ms; theta_0 * dt_max = phi_min."""
    for hd in (32, 64, 88, 128):
        th = O.rope_theta(hd, 1e-4, 600000.0, 31_536_000_000)
        assert abs(th[0] - 3.17098e-15) < 1e-19
        assert th[0] * 31_536_000_000 == pytest.approx(1e-4, rel=1e-15)
        assert (np.diff(th) > 0).all()
    # fastest channel at hd 128 is ~1.55e-9 rad/ms
    assert O.rope_theta(128, 1e-4, 600000.0, 31_536_000_000)[-1] == pytest.approx(1.55e-9, rel=0.01)


def test_rope_rotation_closed_form():
    """S:219 sign pin ((1,0) by pi/2 -> (0,1)) and adjacent pairing / frequency order (R4):
    hd=4, phi_min=pi/2, dt_max=1, base=4 -> theta = (pi/2, pi): e0 -> e1, e2 -> -e2, e3 -> -e3."""
    th = O.rope_theta(4, math.pi / 2, 4.0, 1)
    assert th == pytest.approx([math.pi / 2, math.pi])
    x = np.eye(4)
    r = O.rope_rotate(x, np.ones(4, dtype=np.int64), th)
    assert r[0] == pytest.approx([0, 1, 0, 0], abs=1e-12)
    assert r[1] == pytest.approx([-1, 0, 0, 0], abs=1e-12)
    assert r[2] == pytest.approx([0, 0, -1, 0], abs=1e-12)
    assert r[3] == pytest.approx([0, 0, 0, -1], abs=1e-12)
    # t = 0 -> identity; norm preserved; R(-a) inverts R(a)
    v = np.random.default_rng(1).standard_normal((5, 8))
    tt = np.array([0, 1, 5, 99, 12345], dtype=np.int64)
    th8 = O.rope_theta(8, 0.3, 50.0, 1000)
    assert O.rope_rotate(v[:1], np.zeros(1, np.int64), th8) == pytest.approx(v[:1])
    rv = O.rope_rotate(v, tt, th8)
    assert np.linalg.norm(rv, axis=1) == pytest.approx(np.linalg.norm(v, axis=1), rel=1e-12)
    assert O.rope_rotate(rv, tt, th8, -1.0) == pytest.approx(v, abs=1e-12)


def test_rotated_dot_depends_on_time_difference_only():
    """shift both timestamps by +1e9 ms -> dot unchanged (+-1e-9)."""
    rng = np.random.default_rng(2)
    q, k = rng.standard_normal((1, 64)), rng.standard_normal((1, 64))
    th = O.rope_theta(64, 1e-4, 600000.0, 31_536_000_000)
    tq, tk = np.array([1_735_000_123_456]), np.array([1_734_000_000_000])
    d0 = (O.rope_rotate(q, tq, th) * O.rope_rotate(k, tk, th)).sum()
    d1 = (O.rope_rotate(q, tq + 10**9, th) * O.rope_rotate(k, tk + 10**9, th)).sum()
    assert abs(d0 - d1) < 1e-9
    dsame = (O.rope_rotate(q, tq, th) * O.rope_rotate(k, tq, th)).sum()
    assert dsame == pytest.approx((q * k).sum(), abs=1e-9)


# ---------------------------------------------------------------- gates / softmax pins
def test_sigmoid_and_gate_examples():
    """S:53 sigma(2)=0.8807970779778823; S:157 d=1,x=2,W=1 -> 1.7615942; S:156 W=0 -> x/2."""
    assert O.sigmoid(np.array([2.0]))[0] == pytest.approx(0.8807970779778823, abs=1e-15)
    assert O.sigmoid(np.array([-1000.0]))[0] == 0.0
    cfg = O.AttnConfig(d_model=1, n_heads=1, use_rope=False, use_int_gate=False)
    W = [np.array([[1.0]])] + [np.array([[1.0]])] * 6
    _, c = O.layer_forward_seq(np.array([[2.0]]), W, np.array([0]), np.ones((1, 1), bool), cfg)
    assert c["Xt"][0, 0] == pytest.approx(1.7615942, abs=1e-7)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((6, 8))
    W = [np.zeros((8, 8))] + [rng.standard_normal((8, 8)) for _ in range(6)]
    cfg = O.AttnConfig(d_model=8, n_heads=2)
    _, c = O.layer_forward_seq(X, W, np.arange(6), np.tril(np.ones((6, 6), bool)), cfg)
    assert (c["Xt"] == X / 2).all()
    assert (np.abs(c["Xt"]) <= np.abs(X)).all()
    assert (np.abs(c["Qt"]) <= np.abs(c["Q"]) + 1e-15).all()


def test_softmax_examples_and_masked_zero():
    """[1,2,3] -> [0.09003,0.24473,0.66524]; [5,-inf,-inf] -> [1,0,0]; masked weight exactly 0."""
    Q = np.array([[0.0], [0.0], [0.0]])
    # with hd=1, S = q k / 1: use q=1 on row 2 and k = [1,2,3]
    Qr = np.array([[1.0], [1.0], [1.0]])
    Kr = np.array([[1.0], [2.0], [3.0]])
    V = np.eye(3)
    O3, _, Ps = O.attention_core_forward(Qr, Kr, np.eye(3)[:, :1], np.ones((3, 3), bool), 1)
    assert Ps[0][2] == pytest.approx([0.09003, 0.24473, 0.66524], abs=1e-5)
    A = np.array([[True, False, False]] * 3)
    _, _, Ps = O.attention_core_forward(Qr, Kr * 5, np.eye(3)[:, :1], A, 1)
    assert (Ps[0][:, 1:] == 0.0).all() and (Ps[0][:, 0] == 1.0).all()
    del Q, V, O3


def test_equal_scores_uniform_weights():
    """all scores equal over m allowed keys -> weights 1/m."""
    m = 9
    Qr = np.zeros((m, 4))
    Kr = np.random.default_rng(4).standard_normal((m, 4))
    _, _, Ps = O.attention_core_forward(Qr, Kr, Kr, np.tril(np.ones((m, m), bool)), 1)
    for i in range(m):
        assert Ps[0][i, : i + 1] == pytest.approx(np.full(i + 1, 1.0 / (i + 1)))


def test_single_token_output_is_v_wo():
    """S:173 / S:362: one token -> attention weight 1 on self -> Y = v W_O."""
    rng = np.random.default_rng(5)
    d = 8
    X = rng.standard_normal((1, d))
    W = [rng.standard_normal((d, d)) for _ in range(7)]
    cfg = O.AttnConfig(d_model=d, n_heads=2)
    Y, c = O.layer_forward_seq(X, W, np.array([123]), np.ones((1, 1), bool), cfg)
    assert Y == pytest.approx(c["V"] @ W[6], abs=1e-12)


# ---------------------------------------------------------------- the four self-checks
def _small_case(lengths=(13, 1, 9, 6), d=8, H=2, seed=0, stress=True, n_cand=None, scale=1.0):
    cfgg = G.stress_config() if stress else G.GenConfig()
    b = G.fixed_lengths_batch(list(lengths), seed=seed, cfg=cfgg, n_cand=n_cand)
    rng = np.random.default_rng(seed + 11)
    T = b.n_tokens + 3
    X = rng.standard_normal((T, d))
    X[b.n_tokens:] = 0
    W = [rng.standard_normal((d, d)) * scale / math.sqrt(d) for _ in range(7)]
    cu = np.concatenate([[0], np.cumsum(b.lengths)])
    t = np.concatenate([b.timestamps, np.zeros(3, np.int64)])
    nc = np.zeros(len(lengths), np.int64) if n_cand is None else np.asarray(n_cand)
    meta = O.SeqMeta(cu=cu, t_ms=t, n_cand=nc, session_ids=np.concatenate([b.session_ids, np.zeros(3, np.int32)]))
    return X, W, meta, T


def _stress_cfg(d, H, **kw):
    base = dict(d_model=d, n_heads=H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4,
                rope_dt_max_ms=86_400_000)
    base.update(kw)
    return O.AttnConfig(**base)


@pytest.mark.parametrize("flags", [O.MASK_TIME, O.MASK_TIME | O.MASK_SESSION])
def test_check1_dense_equals_per_element_loop(flags):
    """Check 1: the dense-matrix oracle equals an independent per-pair loop."""
    X, W, meta, T = _small_case(lengths=(7, 1, 5), d=4, H=2, n_cand=[0, 0, 2])
    cfg = _stress_cfg(4, 2, mask_flags=flags)
    Y, _, _ = O.batch_forward(X, W, meta, cfg)
    for s in range(len(meta.cu) - 1):
        a, e = int(meta.cu[s]), int(meta.cu[s + 1])
        Yl = O.layer_forward_loop(X[a:e], W, meta.t_ms[a:e], int(meta.n_cand[s]), cfg,
                                  meta.session_ids[a:e])
        assert Y[a:e] == pytest.approx(Yl, abs=1e-12)


def test_check2_packed_equals_unpacked():
    """Check 2: one T x T block-diagonal mask over the packed buffer == per-sequence."""
    X, W, meta, T = _small_case(n_cand=[0, 0, 3, 1])
    cfg = _stress_cfg(8, 2)
    Y, _, _ = O.batch_forward(X, W, meta, cfg)
    Yp = O.packed_forward_blockdiag(X, W, meta, cfg, T)
    assert Y == pytest.approx(Yp, abs=1e-12)
    assert (Y[int(meta.cu[-1]):] == 0).all()


@pytest.mark.parametrize("stress", [True, False])
def test_check3_timestamp_shift_invariance(stress):
    """Check 3: shifting every timestamp leaves outputs unchanged."""
    X, W, meta, T = _small_case(stress=stress)
    cfg = _stress_cfg(8, 2) if stress else O.AttnConfig(d_model=8, n_heads=2)
    Y0, _, _ = O.batch_forward(X, W, meta, cfg)
    meta2 = dataclasses.replace(meta, t_ms=meta.t_ms + 123_456_789)
    Y1, _, _ = O.batch_forward(X, W, meta2, cfg)
    assert np.abs(Y0 - Y1).max() < 1e-9
    # ... and RoPE is actually active: different relative times change the output
    meta3 = dataclasses.replace(meta, t_ms=meta.t_ms * 2)
    Y2, _, _ = O.batch_forward(X, W, meta3, _stress_cfg(8, 2, delta_delay_ms=0))
    Y3, _, _ = O.batch_forward(X, W, meta, _stress_cfg(8, 2, delta_delay_ms=0))
    if stress:
        assert np.abs(Y2 - Y3).max() > 1e-3


def test_check4_no_gates_no_rope_equals_torch_sdpa():
    """Check 4: gates off + RoPE off -> textbook masked attention (torch SDPA, fp64, bool mask)."""
    torch = pytest.importorskip("torch")
    X, W, meta, T = _small_case(lengths=(17, 5, 11), d=8, H=2, n_cand=[0, 2, 3])
    cfg = _stress_cfg(8, 2, use_rope=False, use_rep_gate=False, use_int_gate=False)
    Y, caches, _ = O.batch_forward(X, W, meta, cfg)
    for (a, e, A, c) in caches:
        Xs = torch.tensor(X[a:e], dtype=torch.float64)
        Wt = [torch.tensor(w, dtype=torch.float64) for w in W]
        q, k, v = Xs @ Wt[1], Xs @ Wt[2], Xs @ Wt[3]
        sh = lambda z: z.view(e - a, 2, 4).transpose(0, 1)
        o = torch.nn.functional.scaled_dot_product_attention(sh(q), sh(k), sh(v),
                                                             attn_mask=torch.tensor(A))
        yt = o.transpose(0, 1).reshape(e - a, 8) @ Wt[6]
        assert Y[a:e] == pytest.approx(yt.numpy(), abs=1e-12)


# ---------------------------------------------------------------- gradients vs finite differences
def _fd_check(f, x, g, idxs, eps=1e-5):
    worst = 0.0
    for ix in idxs:
        old = x[ix]
        x[ix] = old + eps
        fp = f()
        x[ix] = old - eps
        fm = f()
        x[ix] = old
        num = (fp - fm) / (2 * eps)
        worst = max(worst, abs(num - g[ix]) / max(abs(num), abs(g[ix]), 1e-8))
    return worst


@pytest.mark.parametrize("flags,ncand", [(O.MASK_TIME, None), (O.MASK_TIME | O.MASK_SESSION, [0, 0, 3, 1])])
def test_layer_backward_finite_differences(flags, ncand):
    """analytic fp64 gradients == central differences (rel err < 1e-5)."""
    X, W, meta, T = _small_case(n_cand=ncand, scale=2.0)
    cfg = _stress_cfg(8, 2, mask_flags=flags)
    R = np.random.default_rng(9).standard_normal(X.shape)

    def loss():
        Y, _, _ = O.batch_forward(X, W, meta, cfg)
        return float((Y * R).sum())

    Y, caches, _ = O.batch_forward(X, W, meta, cfg)
    dX, gW, _ = O.batch_backward(caches, W, meta, R, cfg)
    rng = np.random.default_rng(10)
    n = int(meta.cu[-1])
    idx = [(int(rng.integers(0, n)), int(rng.integers(0, 8))) for _ in range(25)]
    assert _fd_check(loss, X, dX, idx) < 1e-5
    for k in range(7):
        idx = [(int(rng.integers(0, 8)), int(rng.integers(0, 8))) for _ in range(10)]
        assert _fd_check(loss, W[k], gW[k], idx) < 1e-5, O.AttnConfig.__name__ + str(k)
    # pad rows get zero gradient (R17)
    assert (dX[n:] == 0).all()


def test_core_backward_finite_differences():
    rng = np.random.default_rng(12)
    m, d, H = 10, 8, 2
    Qr, Kr, V = (rng.standard_normal((m, d)) for _ in range(3))
    A = np.tril(np.ones((m, m), bool))
    A[5, 2:5] = False
    R = rng.standard_normal((m, d))

    def loss():
        return float((O.attention_core_forward(Qr, Kr, V, A, H)[0] * R).sum())

    dQ, dK, dV = O.attention_core_backward(Qr, Kr, V, A, R, H)
    idx = [(int(rng.integers(0, m)), int(rng.integers(0, d))) for _ in range(20)]
    for x, g in ((Qr, dQ), (Kr, dK), (V, dV)):
        assert _fd_check(loss, x, g, idx) < 1e-5


# ---------------------------------------------------------------- heads
def test_bucketize_paper_and_spec_examples():
    """S:145-150 (1-based k): position 1, [4] -> 1; position 5, [4] -> 2; position 4, [1, 4] -> 2;
    P:624 K = 2 "positions 1--4, and 5+"; P:393 example k = 1 for position 1, k = 2 for 2--4, k = 3 for 5+."""
    assert O.bucketize([1], [4])[0] + 1 == 1
    assert O.bucketize([5], [4])[0] + 1 == 2
    assert O.bucketize([4], [1, 4])[0] + 1 == 2
    pos = np.arange(1, 13)
    assert list(O.bucketize(pos, [4])) == [0, 0, 0, 0] + [1] * 8
    assert list(O.bucketize(pos, [1, 4])) == [0, 1, 1, 1] + [2] * 8
    # equals the library routine: #{b : pos > b} = searchsorted(b, pos, side="left")
    rng = np.random.default_rng(0)
    bnd = np.sort(rng.choice(np.arange(1, 50), size=5, replace=False))
    p = rng.integers(1, 60, size=1000)
    assert (O.bucketize(p, bnd) == np.searchsorted(bnd, p, side="left")).all()


def test_head_loss_examples():
    """logit 0, y=1 -> ln 2; logit 2, y=1 -> 0.126928."""
    assert O.heads_loss(np.array([[0.0, 5.0]]), np.array([0]), np.array([1.0])) == pytest.approx(math.log(2))
    assert O.heads_loss(np.array([[9.0, 2.0]]), np.array([1]), np.array([1.0])) == pytest.approx(0.126928, abs=1e-6)


def test_heads_zero_weights_and_identical_towers():
    """zero weights -> logits 0; identical MLP_1 == MLP_2 -> identical logits."""
    rng = np.random.default_rng(13)
    H = rng.standard_normal((10, 6))
    z, _, _ = O.heads_forward(H, np.arange(10), np.zeros((2, 6, 3)), np.zeros((2, 3)), np.zeros((2, 3)), np.zeros(2))
    assert (z == 0).all()
    W1 = np.repeat(rng.standard_normal((1, 6, 3)), 2, axis=0)
    b1, w2 = np.repeat(rng.standard_normal((1, 3)), 2, 0), np.repeat(rng.standard_normal((1, 3)), 2, 0)
    z, _, _ = O.heads_forward(H, np.arange(10), W1, b1, w2, np.array([0.3, 0.3]))
    assert (z[:, 0] == z[:, 1]).all()


def test_heads_backward_finite_differences_and_routing():
    """Routed BCE gradients vs central differences; unrealized head gets zero grad."""
    rng = np.random.default_rng(14)
    n, d, dh, K = 12, 6, 4, 2
    Hm = rng.standard_normal((20, d))
    rows = rng.choice(20, size=n, replace=False)
    W1, b1, w2, b2 = rng.standard_normal((K, d, dh)), rng.standard_normal((K, dh)), rng.standard_normal((K, dh)), rng.standard_normal(K)
    bucket = rng.integers(0, K, size=n)
    label = (rng.random(n) < 0.4).astype(float)

    def loss():
        z, _, _ = O.heads_forward(Hm, rows, W1, b1, w2, b2)
        return O.heads_loss(z, bucket, label)

    L, z, dH, g = O.heads_loss_backward(Hm, rows, W1, b1, w2, b2, bucket, label)
    idx = [(int(rng.integers(0, 20)), int(rng.integers(0, d))) for _ in range(15)]
    assert _fd_check(loss, Hm, dH, idx) < 1e-5
    idx = [(int(rng.integers(0, K)), int(rng.integers(0, d)), int(rng.integers(0, dh))) for _ in range(15)]
    assert _fd_check(loss, W1, g["dW1"], idx) < 1e-5
    for arr, gg in ((b1, g["db1"]), (w2, g["dw2"])):
        idx = [(int(rng.integers(0, K)), int(rng.integers(0, dh))) for _ in range(8)]
        assert _fd_check(loss, arr, gg, idx) < 1e-5
    assert _fd_check(loss, b2, g["db2"], [(0,), (1,)]) < 1e-5
    # routing isolation: all impressions in bucket 0 -> head 1 gets exactly zero gradient
    L, z, dH, g = O.heads_loss_backward(Hm, rows, W1, b1, w2, b2, np.zeros(n, int), label)
    assert (g["dW1"][1] == 0).all() and g["db2"][1] == 0 and (g["dw2"][1] == 0).all()


# ------------------------------------------------------------------ NEXT-2: full loss (Eqs. 10-12)
def test_pairwise_unit_values_and_translation_invariance():
    """S:745 loss unit values: RankNet z+ = z- -> ln 2; z+ = 2, z- = 0 -> 0.126928 (+-1e-6); a common
    logit shift leaves Eq. 12 unchanged; an empty side gives 0."""
    assert O.pairwise_loss([0.3], [0.3]) == pytest.approx(math.log(2.0), abs=1e-12)
    assert O.pairwise_loss([2.0], [0.0]) == pytest.approx(0.126928, abs=1e-6)
    rng = np.random.default_rng(3)
    zp, zn = rng.normal(size=7), rng.normal(size=5)
    assert O.pairwise_loss(zp + 3.7, zn + 3.7) == pytest.approx(O.pairwise_loss(zp, zn), abs=1e-12)
    assert O.pairwise_loss([], zn) == 0.0 and O.pairwise_loss(zp, []) == 0.0


def test_pairwise_brute_force_and_gradient():
    """Eq. 12 as a pure-Python double loop of -log(1 / (1 + exp(-(a - b)))) / (N+ N-), and the
    analytic adjoint against central differences."""
    rng = np.random.default_rng(4)
    zp, zn = rng.normal(size=4), rng.normal(size=6)
    bf = 0.0
    for a in zp:
        for b in zn:
            bf -= math.log(1.0 / (1.0 + math.exp(-(a - b))))
    assert O.pairwise_loss(zp, zn) == pytest.approx(bf / (len(zp) * len(zn)), abs=1e-13)
    gp, gn = O.pairwise_grad(zp, zn)
    eps = 1e-6
    for i in range(len(zp)):
        e = np.zeros_like(zp)
        e[i] = eps
        fd = (O.pairwise_loss(zp + e, zn) - O.pairwise_loss(zp - e, zn)) / (2 * eps)
        assert gp[i] == pytest.approx(fd, abs=1e-8)
    for j in range(len(zn)):
        e = np.zeros_like(zn)
        e[j] = eps
        fd = (O.pairwise_loss(zp, zn + e) - O.pairwise_loss(zp, zn - e)) / (2 * eps)
        assert gn[j] == pytest.approx(fd, abs=1e-8)


def test_aux_losses_closed_form_and_gradient():
    """R31: BCE with logits (softplus(z) - y z) and squared error (z - y)^2, summed; dz by FD."""
    za = np.array([[0.0, 1.5], [2.0, -0.5], [-1.0, 3.0]])
    ya = np.array([[1.0, 1.0], [0.0, 0.0], [1.0, 2.5]])
    l = O.aux_losses(za, ya)
    # rows: (z 0, y 1) -> ln 2; (z 2, y 0) -> log1p(e^2); (z -1, y 1) -> log1p(e^-1) + 1
    assert l[0] == pytest.approx(math.log(2) + math.log1p(math.exp(2.0)) + math.log1p(math.exp(-1.0)) + 1.0, abs=1e-12)
    assert l[1] == pytest.approx(0.25 + 0.25 + 0.25, abs=1e-12)
    dz = O.aux_dz(za, ya)
    eps = 1e-6
    for i in range(3):
        for j in range(2):
            e = np.zeros_like(za)
            e[i, j] = eps
            fd = (O.aux_losses(za + e, ya)[j] - O.aux_losses(za - e, ya)[j]) / (2 * eps)
            assert dz[i, j] == pytest.approx(fd, abs=1e-7)


def _full_case(seed=5, n_rows=9, T=14, d=8, K=2, dh=6, da=4):
    rng = np.random.default_rng(seed)
    H = rng.normal(size=(T, d))
    rows = np.sort(rng.choice(T, size=n_rows, replace=False))
    ctx = (rng.normal(size=(K, d, dh)) / 3, rng.normal(size=(K, dh)) / 3, rng.normal(size=(K, dh)), rng.normal(size=K))
    aux = (rng.normal(size=(2, d, da)) / 3, rng.normal(size=(2, da)) / 3, rng.normal(size=(2, da)), rng.normal(size=2))
    bucket = rng.integers(0, K, size=n_rows)
    label = (rng.random(n_rows) < 0.4).astype(np.float64)
    label[0], label[1] = 1.0, 0.0
    ya = np.stack([(rng.random(n_rows) < 0.3).astype(np.float64), rng.exponential(size=n_rows)], axis=1)
    return H, rows, ctx, aux, bucket, label, ya


def test_full_loss_gradient_by_finite_differences():
    """Eq. 11 total: the analytic dH (through the towers, the aux heads and RankNet on the routed
    logits) and a tower / aux weight gradient against central differences of the total."""
    H, rows, ctx, aux, bucket, label, ya = _full_case()
    lam = (1.0, (0.3, 0.2), 0.7)
    terms, dH, gc, ga = O.full_loss_backward(H, rows, ctx, aux, bucket, label, ya, lam)
    f = lambda H_, ctx_=ctx, aux_=aux: O.full_loss_backward(H_, rows, ctx_, aux_, bucket, label, ya, lam)[0]["total"]
    eps = 1e-6
    for (r, c) in [(rows[0], 1), (rows[3], 5), (rows[-1], 0)]:
        e = np.zeros_like(H)
        e[r, c] = eps
        assert dH[r, c] == pytest.approx((f(H + e) - f(H - e)) / (2 * eps), abs=1e-6)
    for name, g, params, which in (("dW1", gc, ctx, 0), ("dW1", ga, aux, 1)):
        W1 = params[0]
        e = np.zeros_like(W1)
        e[1, 2, 3] = eps
        p_plus = (W1 + e,) + tuple(params[1:])
        p_minus = (W1 - e,) + tuple(params[1:])
        if which == 0:
            fd = (f(H, p_plus, aux) - f(H, p_minus, aux)) / (2 * eps)
        else:
            fd = (f(H, ctx, p_plus) - f(H, ctx, p_minus)) / (2 * eps)
        assert g[name][1, 2, 3] == pytest.approx(fd, abs=1e-6)


def test_full_loss_reductions():
    """lam_pair = 0 gives exactly the context + aux gradient (S:472 linearity); aux heads do not touch
    the towers' gradients and vice versa (isolation); lam = (1, 0, 0) reduces to Eq. 9's routed BCE."""
    H, rows, ctx, aux, bucket, label, ya = _full_case(seed=6)
    t0, dH0, gc0, ga0 = O.full_loss_backward(H, rows, ctx, aux, bucket, label, ya, (1.0, (0.3, 0.2), 0.0))
    t1, dH1, gc1, ga1 = O.full_loss_backward(H, rows, ctx, aux, bucket, label, ya, (1.0, (0.3, 0.2), 0.5))
    assert np.array_equal(ga0["dW1"], ga1["dW1"])        # RankNet acts on the towers only
    L, z, dHc, gcc = O.heads_loss_backward(H, rows, *ctx, bucket, label)
    t2, dH2, gc2, ga2 = O.full_loss_backward(H, rows, ctx, aux, bucket, label, ya, (1.0, (0.0, 0.0), 0.0))
    assert t2["total"] == pytest.approx(L, abs=1e-12)
    assert np.allclose(dH2, dHc, atol=1e-14) and np.allclose(gc2["dW1"], gcc["dW1"], atol=1e-14)
    assert np.all(ga2["dW1"] == 0)
    # pairwise-only part of the tower gradient is linear in lam_pair
    t3, dH3, gc3, ga3 = O.full_loss_backward(H, rows, ctx, aux, bucket, label, ya, (1.0, (0.3, 0.2), 1.0))
    assert np.allclose(gc3["db2"] - gc0["db2"], 2.0 * (gc1["db2"] - gc0["db2"]), atol=1e-13)


# ------------------------------------------------------------------ NEXT-3: the full block
def test_rmsnorm_unit_rms_scale_invariance_and_gradient():
    rng = np.random.default_rng(21)
    x = rng.normal(size=(4, 16)) * 3
    y, _ = O.rmsnorm(x, np.ones(16), eps=0.0)
    assert np.allclose(np.sqrt((y ** 2).mean(-1)), 1.0, atol=1e-14)
    g = rng.normal(size=16)
    assert np.allclose(O.rmsnorm(7.5 * x, g, eps=0.0)[0], O.rmsnorm(x, g, eps=0.0)[0], atol=1e-13)
    dy = rng.normal(size=(4, 16))
    dx, dg = O.rmsnorm_backward(x, g, dy)
    f = lambda x_, g_: float(np.sum(O.rmsnorm(x_, g_)[0] * dy))
    eps = 1e-6
    for (i, j) in [(0, 0), (2, 7), (3, 15)]:
        e = np.zeros_like(x)
        e[i, j] = eps
        assert dx[i, j] == pytest.approx((f(x + e, g) - f(x - e, g)) / (2 * eps), abs=1e-7)
    e = np.zeros(16)
    e[5] = eps
    assert dg[5] == pytest.approx((f(x, g + e) - f(x, g - e)) / (2 * eps), abs=1e-7)


def test_gelu_values_and_ffn_gradient():
    """Exact GELU u Phi(u): Phi(1) = 0.8413447460685429 (normal CDF), GELU(0) = 0, odd-part identity
    GELU(u) - GELU(-u) = u; FFN adjoint by finite differences."""
    assert O.gelu(0.0) == 0.0
    assert O.gelu(1.0) == pytest.approx(0.8413447460685429, abs=1e-15)
    assert O.gelu(-1.0) == pytest.approx(-0.15865525393145707, abs=1e-15)
    u = np.linspace(-4, 4, 17)
    assert np.allclose(O.gelu(u) - O.gelu(-u), u, atol=1e-14)
    eps = 1e-6
    assert np.allclose(O.gelu_grad(u), (O.gelu(u + eps) - O.gelu(u - eps)) / (2 * eps), atol=1e-8)
    rng = np.random.default_rng(22)
    x = rng.normal(size=(5, 8))
    W1, W2 = rng.normal(size=(8, 32)) / 3, rng.normal(size=(32, 8)) / 5
    y, uu = O.ffn_forward(x, W1, W2)
    dy = rng.normal(size=y.shape)
    dx, dW1, dW2 = O.ffn_backward(x, W1, W2, uu, dy)
    f = lambda x_, a, b: float(np.sum(O.ffn_forward(x_, a, b)[0] * dy))
    for (M, grad, k) in ((x, dx, 0), (W1, dW1, 1), (W2, dW2, 2)):
        e = np.zeros_like(M)
        e[1, 2] = eps
        args_p = [x, W1, W2]
        args_m = [x, W1, W2]
        args_p[k] = M + e
        args_m[k] = M - e
        assert grad[1, 2] == pytest.approx((f(*args_p) - f(*args_m)) / (2 * eps), abs=1e-7)


def test_block_backward_by_finite_differences_and_zero_ffn_reduction():
    """Pre-norm block through attention: dX and one weight of each part against central
    differences; W2 = 0 reduces the block to X + Attn(RMSNorm_1(X))."""
    b = G.fixed_lengths_batch([7], seed=3, cfg=G.stress_config())
    d, H = 8, 2
    cfg = O.AttnConfig(d_model=d, n_heads=H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4,
                       rope_dt_max_ms=86_400_000)
    meta = O.SeqMeta(cu=np.array([0, 7]), t_ms=b.timestamps, n_cand=np.zeros(1, np.int64))
    A = O.seq_mask(meta, 0, cfg)
    rng = np.random.default_rng(23)
    X = rng.normal(size=(7, d))
    W = [rng.normal(size=(d, d)) / np.sqrt(d) for _ in range(7)]
    ffn = (rng.normal(size=(d, 4 * d)) / 3, rng.normal(size=(4 * d, d)) / 6)
    gam = (1.0 + 0.1 * rng.normal(size=d), 1.0 + 0.1 * rng.normal(size=d))
    Y, c = O.block_forward_seq(X, W, ffn, gam, b.timestamps, A, cfg)
    dY = rng.normal(size=Y.shape)
    dX, g = O.block_backward_seq(c, W, ffn, gam, b.timestamps, A, dY, cfg)
    f = lambda X_=X, W_=W, ffn_=ffn, gam_=gam: float(np.sum(O.block_forward_seq(X_, W_, ffn_, gam_, b.timestamps, A,
                                                                                   cfg)[0] * dY))
    eps = 1e-6
    e = np.zeros_like(X)
    e[3, 4] = eps
    assert dX[3, 4] == pytest.approx((f(X_=X + e) - f(X_=X - e)) / (2 * eps), abs=1e-6)
    e = np.zeros_like(ffn[0])
    e[2, 9] = eps
    assert g["dW1f"][2, 9] == pytest.approx((f(ffn_=(ffn[0] + e, ffn[1])) - f(ffn_=(ffn[0] - e, ffn[1]))) / (2 * eps),
                                            abs=1e-6)
    e = np.zeros(d)
    e[1] = eps
    assert g["dg1"][1] == pytest.approx((f(gam_=(gam[0] + e, gam[1])) - f(gam_=(gam[0] - e, gam[1]))) / (2 * eps),
                                        abs=1e-6)
    ew = np.zeros_like(W[1])
    ew[0, 3] = eps
    Wp = [w.copy() for w in W]
    Wm = [w.copy() for w in W]
    Wp[1] = W[1] + ew
    Wm[1] = W[1] - ew
    assert g["gW"][1][0, 3] == pytest.approx((f(W_=Wp) - f(W_=Wm)) / (2 * eps), abs=1e-6)
    Y0, _ = O.block_forward_seq(X, W, (ffn[0], np.zeros_like(ffn[1])), gam, b.timestamps, A, cfg)
    Ya, _ = O.layer_forward_seq(O.rmsnorm(X, gam[0])[0], W, b.timestamps, A, cfg)
    assert np.allclose(Y0, X + Ya, atol=1e-13)


# ------------------------------------------------------------------ NEXT-4: AdamW (R35)
def test_embeddings_onehot_matmul_loop_and_adjoint():
    """NEXT-3 embeddings (Eq. 1): the gather-sum equals the one-hot matmul sum_f onehot_f E_f (a
    library routine) and a per-token loop; the backward equals onehot_f^T dX and satisfies the adjoint
    identity <embed(E), dX> = sum_f <E_f, dE_f>."""
    rng = np.random.default_rng(3)
    vocab, d, T = (2, 50, 5, 3), 16, 200
    ids = np.stack([rng.integers(-1, V, size=T) for V in vocab], axis=1)
    tables = [rng.standard_normal((V, d)) for V in vocab]
    X = O.embed_forward(ids, tables)
    onehot = [np.eye(V)[np.where(ids[:, f] >= 0, ids[:, f], 0)] * (ids[:, f] >= 0)[:, None] for f, V in enumerate(vocab)]
    assert np.allclose(X, sum(oh @ E for oh, E in zip(onehot, tables)), atol=1e-12)
    loop = np.zeros((T, d))
    for t in range(T):
        for f in range(len(vocab)):
            if ids[t, f] >= 0:
                loop[t] += tables[f][ids[t, f]]
    assert np.array_equal(X, loop)
    dX = rng.standard_normal((T, d))
    dE = O.embed_backward(ids, dX, vocab)
    for oh, g in zip(onehot, dE):
        assert np.allclose(g, oh.T @ dX, atol=1e-12)
    lhs = float((X * dX).sum())
    rhs = sum(float((E * g).sum()) for E, g in zip(tables, dE))
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))


def test_adamw_first_step_constant_gradient_and_decay_closed_forms():
    """Pins of O.adamw_step against closed forms of Adam's algebra (Kingma & Ba, Alg. 1; decoupled
    decay, Loshchilov & Hutter): (i) step 1: m_hat = g, v_hat = g^2, so the update is
    -lr g / (|g| + eps) (= -lr sign(g) for |g| >> eps); (ii) a constant gradient keeps m_hat = g and
    v_hat = g^2 at every step (the bias corrections are exact), so k steps move theta by
    -k lr g / (|g| + eps); (iii) with g = 0 only the decay acts: theta_k = theta_0 (1 - lr wd)^k;
    (iv) a hand-computed two-step example with beta1 = 0.5, beta2 = 0.75."""
    rng = np.random.default_rng(3)
    th = rng.normal(size=257)
    g = rng.normal(size=257) * np.logspace(-6, 2, 257)
    z = np.zeros(257)
    lr = 1e-3
    t1, m1, v1 = O.adamw_step(th, z, z, g, 1, lr=lr)
    assert np.allclose(t1, th - lr * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
    assert np.allclose(m1, 0.1 * g) and np.allclose(v1, 0.001 * g * g)
    t, m, v = th, z, z
    for k in range(1, 8):
        t, m, v = O.adamw_step(t, m, v, g, k, lr=lr)
    assert np.allclose(t, th - 7 * lr * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-12)
    t, m, v = th, z, z
    for k in range(1, 6):
        t, m, v = O.adamw_step(t, m, v, z, k, lr=lr, weight_decay=0.1)
    assert np.allclose(t, th * (1 - lr * 0.1) ** 5, rtol=1e-14)
    # (iv) theta 1, g = 2 then -1, lr 0.1, beta1 0.5, beta2 0.75, eps 0:
    # step 1: m = 1, v = 1, m_hat = 2, v_hat = 4 -> theta = 1 - 0.1 * 2 / 2 = 0.9
    # step 2: m = 0.5 - 0.5 = 0, v = 0.75 + 0.25 = 1 -> m_hat = 0, theta stays 0.9
    t, m, v = O.adamw_step(np.array([1.0]), np.zeros(1), np.zeros(1), np.array([2.0]), 1, lr=0.1, beta1=0.5,
                           beta2=0.75, eps=0.0)
    assert t[0] == pytest.approx(0.9) and m[0] == pytest.approx(1.0) and v[0] == pytest.approx(1.0)
    t, m, v = O.adamw_step(t, m, v, np.array([-1.0]), 2, lr=0.1, beta1=0.5, beta2=0.75, eps=0.0)
    assert t[0] == pytest.approx(0.9) and m[0] == pytest.approx(0.0) and v[0] == pytest.approx(1.0)
