"""CADET hot-path ORACLE — plain, slow, fp64 CPU reference.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this module.
It shares no code with the CUDA path (paper_2602_11410_b200/) and never
imports it.  Every function follows PAPER.md (P:n) / SPEC.md (S:n) as cited,
with the readings R1..R35 listed in DESIGN.md §3 (R29-R31: the NEXT-2 full loss; R32-R33: the
NEXT-3 block; R35: the NEXT-4 optimizer).

Conventions: row-vector projections y = x.W, W[d_in][d_out] (R1); all math in
float64 on bf16-valued inputs (R20); heads are per-head slices of width hd of
the d-wide rows; RoPE pairs are adjacent (2i, 2i+1) (R4), per head (R5).
Parity status: every function below is pinned by a `-m "not gpu"` test in
tests/test_oracle_pins.py (no "parity unpinned" functions).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
import numpy as np

MASK_TIME = 1
MASK_SESSION = 2
MASK_PAIR_PREV = 4


# ------------------------------------------------------------------ config
@dataclass
class AttnConfig:
    d_model: int
    n_heads: int
    mask_flags: int = MASK_TIME
    delta_delay_ms: int = 3_600_000          # P:561 "Delta_delay of one hour"
    delta_cand_ms: int = 0                    # R11: candidates see all context
    rope_dt_max_ms: int = 31_536_000_000      # P:627, R6
    rope_phi_min: float = 1e-4
    rope_base: float = 600000.0
    use_rope: bool = True
    use_rep_gate: bool = True
    use_int_gate: bool = True
    use_out_proj: bool = True

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


# ------------------------------------------------------------------ numerics
def sigmoid(x):
    """sigma(x) = 1/(1+exp(-x)); evaluated without overflow."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def softplus(x):
    return np.logaddexp(0.0, np.asarray(x, dtype=np.float64))


# ------------------------------------------------------------------ RoPE
def rope_theta(head_dim: int, phi_min: float, base: float, dt_max_ms: int) -> np.ndarray:
    """theta_i = (phi_min / dt_max) * base^(2i/d), i in [0, d/2)  (R5: d = head dim)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    return (phi_min / float(dt_max_ms)) * np.power(float(base), 2.0 * i / head_dim)


def rope_rotate(x: np.ndarray, t_ms: np.ndarray, theta: np.ndarray, sign: float = 1.0) -> np.ndarray:
    """Rotate adjacent pairs (x_2i, x_2i+1) of each row by alpha_i = t * theta_i.

    x: [m, hd]; t_ms: int64 [m] absolute Unix ms, used as fp64 (R21).
    sign=-1 applies R(-alpha) (the transpose), used by the backward.
    """
    alpha = sign * t_ms.astype(np.float64)[:, None] * theta[None, :]
    c, s = np.cos(alpha), np.sin(alpha)
    x0, x1 = x[:, 0::2], x[:, 1::2]
    out = np.empty_like(x, dtype=np.float64)
    out[:, 0::2] = x0 * c - x1 * s
    out[:, 1::2] = x0 * s + x1 * c
    return out


# ------------------------------------------------------------------ mask (Fig. 3)
def mask_dense(t_ms, n_cand: int, cfg: AttnConfig, session_ids=None, n_static: int = 0,
               pair_flags=None) -> np.ndarray:
    """Dense boolean mask A[i, j] (True = may attend) for ONE sequence (local indices).

    - j == i always allowed (preserved diagonal, Fig. 3 caption P:383; R8).
    - context query i < L (L = m - n_cand): j < i and
        (TIME    => t_j <= t_i - Delta_delay)   (Eq. 6; tie allowed, R9)
        (SESSION => sess_j < sess_i)            (R10, opt-in)
      plus j < min(i, n_static) always (R13), plus j == i-1 if PAIR_PREV and flag_i (R12).
    - candidate query i >= L: j < L and t_j <= t_i - Delta_cand (R11), never
      another candidate.
    """
    t = np.asarray(t_ms, dtype=np.int64)
    m = t.shape[0]
    L = m - int(n_cand)
    i = np.arange(m)[:, None]
    j = np.arange(m)[None, :]
    ctx_ok = j < i
    if cfg.mask_flags & MASK_TIME:
        ctx_ok = ctx_ok & (t[None, :] <= t[:, None] - np.int64(cfg.delta_delay_ms))
    if cfg.mask_flags & MASK_SESSION:
        s = np.asarray(session_ids, dtype=np.int64)
        ctx_ok = ctx_ok & (s[None, :] < s[:, None])
    if n_static:
        ctx_ok = ctx_ok | (j < np.minimum(i, n_static))
    if (cfg.mask_flags & MASK_PAIR_PREV) and pair_flags is not None:
        pf = np.asarray(pair_flags).astype(bool)
        ctx_ok = ctx_ok | ((j == i - 1) & pf[:, None])
    cand_ok = (j < L) & (t[None, :] <= t[:, None] - np.int64(cfg.delta_cand_ms))
    A = np.where(i < L, ctx_ok, cand_ok)
    A = A | (i == j)
    return A


def kv_end_local(A: np.ndarray) -> np.ndarray:
    """Exclusive end of the visible off-diagonal prefix of each row.

    A must be built WITHOUT the PAIR_PREV exception (the canonical kv_end ignores
    it).  Asserts every row is a prefix U {i}, which holds when timestamps and
    session ids are non-decreasing within the sequence.
    """
    m = A.shape[0]
    e = np.zeros(m, dtype=np.int64)
    for i in range(m):
        row = A[i, :i]
        nz = np.nonzero(row)[0]
        ei = 0 if nz.size == 0 else int(nz[-1]) + 1
        assert row[:ei].all(), "mask row is not a prefix"
        assert not A[i, i + 1:].any(), "mask row sees the future"
        e[i] = ei
    return e


def tile_classes(A: np.ndarray, tile: int = 128) -> np.ndarray:
    """Per (q-tile, k-tile), anchored at the sequence start, in-bounds cells only:
    0 = SKIP (none allowed), 1 = PARTIAL, 2 = FULL (all allowed)."""
    m = A.shape[0]
    nq = (m + tile - 1) // tile
    out = np.zeros((nq, nq), dtype=np.int8)
    for a in range(nq):
        for b in range(nq):
            blk = A[a * tile:(a + 1) * tile, b * tile:(b + 1) * tile]
            out[a, b] = 0 if not blk.any() else (2 if blk.all() else 1)
    return out


def count_pairs_inference(L: int, N: int) -> int:
    """Closed form of the allowed-pair count for the candidate pattern: L(L+1)/2 + N(L+1)."""
    return L * (L + 1) // 2 + N * (L + 1)


# ------------------------------------------------------------------ batching
def chunk_offsets(cu: np.ndarray, L_chunk: int) -> np.ndarray:
    """Split each [a, e) at e - L_chunk, e - 2 L_chunk, ... (newest chunk full);
    chunks emitted in buffer (time) order so they stay contiguous."""
    out = [0]
    for s in range(len(cu) - 1):
        a, e = int(cu[s]), int(cu[s + 1])
        bounds = []
        k = 1
        while True:
            lo = max(a, e - k * L_chunk)
            bounds.append(lo)
            if lo == a:
                break
            k += 1
        for b in reversed(bounds[:-1]):
            out.append(b)
        out.append(e)
    return np.asarray(out, dtype=np.int64)


def pack_greedy(lengths, budget: int):
    """Greedy arrival-order packing into ONE fixed-budget buffer.
    Returns (cu_seqlens, n_packed, pad)."""
    cu = [0]
    for m in lengths:
        if cu[-1] + int(m) > budget:
            break
        cu.append(cu[-1] + int(m))
    return np.asarray(cu, dtype=np.int64), len(cu) - 1, budget - cu[-1]


# ------------------------------------------------------------------ attention core (Eq. 7)
def attention_core_forward(Qr, Kr, V, A, n_heads: int):
    """Per head: S = Q K^T / sqrt(hd); S[~A] = -inf; P = softmax_rows(S); O = P V.
    Returns O [m, H*hd], LSE [H, m] (natural log of the masked row sum of exp(S)), P list."""
    m, d = Qr.shape
    hd = d // n_heads
    O = np.zeros((m, d))
    lse = np.zeros((n_heads, m))
    Ps = []
    for h in range(n_heads):
        sl = slice(h * hd, (h + 1) * hd)
        S = Qr[:, sl] @ Kr[:, sl].T / math.sqrt(hd)
        S = np.where(A, S, -np.inf)
        mx = S.max(axis=1, keepdims=True)
        E = np.where(A, np.exp(S - mx), 0.0)
        Z = E.sum(axis=1, keepdims=True)
        P = E / Z
        O[:, sl] = P @ V[:, sl]
        lse[h] = (mx + np.log(Z))[:, 0]
        Ps.append(P)
    return O, lse, Ps


def attention_core_backward(Qr, Kr, V, A, dO, n_heads: int):
    """Adjoint of attention_core_forward (row A10): dV = P^T dO; dP = dO V^T;
    dS = P * (dP - rowsum(dO*O)); dQ = dS K / sqrt(hd); dK = dS^T Q / sqrt(hd)."""
    m, d = Qr.shape
    hd = d // n_heads
    O, _, Ps = attention_core_forward(Qr, Kr, V, A, n_heads)
    dQ = np.zeros_like(Qr, dtype=np.float64)
    dK = np.zeros_like(Kr, dtype=np.float64)
    dV = np.zeros_like(V, dtype=np.float64)
    for h in range(n_heads):
        sl = slice(h * hd, (h + 1) * hd)
        P = Ps[h]
        dV[:, sl] = P.T @ dO[:, sl]
        dP = dO[:, sl] @ V[:, sl].T
        D = (dO[:, sl] * O[:, sl]).sum(axis=1, keepdims=True)
        dS = P * (dP - D)
        dQ[:, sl] = dS @ Kr[:, sl] / math.sqrt(hd)
        dK[:, sl] = dS.T @ Qr[:, sl] / math.sqrt(hd)
    return dQ, dK, dV


# ------------------------------------------------------------------ full gated layer (Eqs. 3-7)
def rope_heads(X, t_ms, cfg: AttnConfig, sign: float = 1.0):
    hd = cfg.head_dim
    th = rope_theta(hd, cfg.rope_phi_min, cfg.rope_base, cfg.rope_dt_max_ms)
    out = np.empty_like(X, dtype=np.float64)
    for h in range(cfg.n_heads):
        sl = slice(h * hd, (h + 1) * hd)
        out[:, sl] = rope_rotate(X[:, sl], t_ms, th, sign)
    return out


def layer_forward_seq(X, W, t_ms, A, cfg: AttnConfig):
    """One sequence through the self-gated attention layer.

    Gx = sigma(X W_xg), Xt = X * Gx                 (Eq. 4; R1)
    Q, K, V = Xt W_q, Xt W_k, Xt W_v                (Eq. 3; R2)
    Qt = Q * sigma(Q W_qg), Kt = K * sigma(K W_kg)  (Eq. 5)
    Qr, Kr = RoPE_t(Qt), RoPE_t(Kt) per head        (R3-R5)
    O = softmax(Qr Kr^T / sqrt(hd) + M) V           (Eq. 7; R16)
    Y = O W_o                                       (R14)
    """
    X = np.asarray(X, dtype=np.float64)
    Wxg, Wq, Wk, Wv, Wqg, Wkg, Wo = [np.asarray(w, dtype=np.float64) for w in W]
    c = {}
    c["X"] = X
    if cfg.use_rep_gate:
        c["Zx"] = X @ Wxg
        c["Gx"] = sigmoid(c["Zx"])
        Xt = X * c["Gx"]
    else:
        Xt = X
    c["Xt"] = Xt
    Q, K, V = Xt @ Wq, Xt @ Wk, Xt @ Wv
    c["Q"], c["K"], c["V"] = Q, K, V
    if cfg.use_int_gate:
        c["Zq"], c["Zk"] = Q @ Wqg, K @ Wkg
        c["Gq"], c["Gk"] = sigmoid(c["Zq"]), sigmoid(c["Zk"])
        Qt, Kt = Q * c["Gq"], K * c["Gk"]
    else:
        Qt, Kt = Q, K
    c["Qt"], c["Kt"] = Qt, Kt
    if cfg.use_rope:
        Qr, Kr = rope_heads(Qt, t_ms, cfg), rope_heads(Kt, t_ms, cfg)
    else:
        Qr, Kr = Qt, Kt
    c["Qr"], c["Kr"] = Qr, Kr
    O, lse, _ = attention_core_forward(Qr, Kr, V, A, cfg.n_heads)
    c["O"], c["lse"] = O, lse
    Y = O @ Wo if cfg.use_out_proj else O
    c["Y"] = Y
    return Y, c


def layer_backward_seq(c, W, t_ms, A, dY, cfg: AttnConfig):
    """Hand-derived adjoint of layer_forward_seq (rows A9, A10, A11, A12).
    Returns dX and the list of 7 weight gradients in NAMES order."""
    Wxg, Wq, Wk, Wv, Wqg, Wkg, Wo = [np.asarray(w, dtype=np.float64) for w in W]
    dY = np.asarray(dY, dtype=np.float64)
    d = Wq.shape[0]
    g = {n: np.zeros((d, d)) for n in ["W_xg", "W_q", "W_k", "W_v", "W_qg", "W_kg", "W_o"]}
    if cfg.use_out_proj:
        dO = dY @ Wo.T
        g["W_o"] = c["O"].T @ dY
    else:
        dO = dY
    dQr, dKr, dV = attention_core_backward(c["Qr"], c["Kr"], c["V"], A, dO, cfg.n_heads)
    if cfg.use_rope:
        dQt, dKt = rope_heads(dQr, t_ms, cfg, -1.0), rope_heads(dKr, t_ms, cfg, -1.0)
    else:
        dQt, dKt = dQr, dKr
    if cfg.use_int_gate:
        uq = dQt * c["Q"] * c["Gq"] * (1.0 - c["Gq"])
        uk = dKt * c["K"] * c["Gk"] * (1.0 - c["Gk"])
        dQ = dQt * c["Gq"] + uq @ Wqg.T
        dK = dKt * c["Gk"] + uk @ Wkg.T
        g["W_qg"] = c["Q"].T @ uq
        g["W_kg"] = c["K"].T @ uk
    else:
        dQ, dK = dQt, dKt
    Xt = c["Xt"]
    g["W_q"], g["W_k"], g["W_v"] = Xt.T @ dQ, Xt.T @ dK, Xt.T @ dV
    dXt = dQ @ Wq.T + dK @ Wk.T + dV @ Wv.T
    if cfg.use_rep_gate:
        ux = dXt * c["X"] * c["Gx"] * (1.0 - c["Gx"])
        dX = dXt * c["Gx"] + ux @ Wxg.T
        g["W_xg"] = c["X"].T @ ux
    else:
        dX = dXt
    inter = dict(dO=dO, dQr=dQr, dKr=dKr, dV=dV, dQt=dQt, dKt=dKt, dQ=dQ, dK=dK, dXt=dXt)
    return dX, [g[n] for n in ["W_xg", "W_q", "W_k", "W_v", "W_qg", "W_kg", "W_o"]], inter


# ------------------------------------------------------------------ packed batch drivers
@dataclass
class SeqMeta:
    cu: np.ndarray             # [n+1] offsets into the packed buffer
    t_ms: np.ndarray           # [T] int64
    n_cand: np.ndarray         # [n]
    session_ids: np.ndarray = None
    n_static: np.ndarray = None
    pair_flags: np.ndarray = None


def seq_mask(meta: SeqMeta, s: int, cfg: AttnConfig) -> np.ndarray:
    a, e = int(meta.cu[s]), int(meta.cu[s + 1])
    return mask_dense(meta.t_ms[a:e], int(meta.n_cand[s]), cfg,
                      None if meta.session_ids is None else meta.session_ids[a:e],
                      0 if meta.n_static is None else int(meta.n_static[s]),
                      None if meta.pair_flags is None else meta.pair_flags[a:e])


def mask_artifacts(meta: SeqMeta, cfg: AttnConfig, T: int, tile: int = 128):
    """Bit-exact targets: global kv_end [T], concatenated tile classes, pair count.

    kv_end comes from the mask without the PAIR_PREV exception; the full mask
    is asserted to equal prefix U {i} U {i-1 if flagged}."""
    import dataclasses
    cfg_nopp = dataclasses.replace(cfg, mask_flags=cfg.mask_flags & ~MASK_PAIR_PREV)
    kv_end = np.arange(T, dtype=np.int64)          # pad rows: kv_end = i
    tiles = []
    pairs = 0
    for s in range(len(meta.cu) - 1):
        a, e = int(meta.cu[s]), int(meta.cu[s + 1])
        A = seq_mask(meta, s, cfg)
        e_loc = kv_end_local(seq_mask(meta, s, cfg_nopp))
        m = e - a
        L = m - int(meta.n_cand[s])
        # structural assertion: A == prefix U diag U pair
        R = np.arange(m)[None, :] < e_loc[:, None]
        R |= np.eye(m, dtype=bool)
        if (cfg.mask_flags & MASK_PAIR_PREV) and meta.pair_flags is not None:
            pf = np.asarray(meta.pair_flags[a:e]).astype(bool)
            for i in range(1, min(m, L)):
                if pf[i]:
                    R[i, i - 1] = True
        assert (R == A).all(), "mask is not prefix U diag U pair"
        kv_end[a:e] = a + e_loc
        tiles.append(tile_classes(A, tile).reshape(-1))
        pairs += int(A.sum())
    tiles = np.concatenate(tiles) if tiles else np.zeros(0, np.int8)
    return kv_end, tiles, pairs


def batch_forward(X, W, meta: SeqMeta, cfg: AttnConfig):
    """Unpacked per-sequence forward over a packed buffer; pad rows give 0 (R17)."""
    T, d = X.shape
    Y = np.zeros((T, d))
    caches = []
    lse = np.zeros((cfg.n_heads, T))
    for s in range(len(meta.cu) - 1):
        a, e = int(meta.cu[s]), int(meta.cu[s + 1])
        A = seq_mask(meta, s, cfg)
        Ys, c = layer_forward_seq(X[a:e], W, meta.t_ms[a:e], A, cfg)
        Y[a:e] = Ys
        lse[:, a:e] = c["lse"]
        caches.append((a, e, A, c))
    return Y, caches, lse


def batch_backward(caches, W, meta: SeqMeta, dY, cfg: AttnConfig):
    T, d = dY.shape
    dX = np.zeros((T, d))
    gs = [np.zeros((d, d)) for _ in range(7)]
    inters = []
    for (a, e, A, c) in caches:
        dXs, g, inter = layer_backward_seq(c, W, meta.t_ms[a:e], A, dY[a:e], cfg)
        dX[a:e] = dXs
        for k in range(7):
            gs[k] += g[k]
        inters.append((a, e, inter))
    return dX, gs, inters


def packed_forward_blockdiag(X, W, meta: SeqMeta, cfg: AttnConfig, T: int):
    """The SAME layer over the whole packed buffer with one T x T block-diagonal mask
    (check 2: packed == unpacked).  Pad rows see only themselves."""
    A = np.zeros((T, T), dtype=bool)
    for s in range(len(meta.cu) - 1):
        a, e = int(meta.cu[s]), int(meta.cu[s + 1])
        A[a:e, a:e] = seq_mask(meta, s, cfg)
    n_real = int(meta.cu[-1])
    for i in range(n_real, T):
        A[i, i] = True
    Y, c = layer_forward_seq(X, W, meta.t_ms, A, cfg)
    Y[n_real:] = 0.0
    return Y


# ------------------------------------------------------------------ heads (Eqs. 8-9)
def bucketize(raw_position, boundaries):
    """Context bucket of a raw feed position ("partition the context space into K discrete
    buckets"; deployed K = 2, "positions 1--4, and 5+"): the plain definition
    k = #{b in boundaries : position > b}, 0-based (SPEC's 1-based k minus one)."""
    pos = np.asarray(raw_position, dtype=np.int64)
    k = np.zeros(pos.shape, dtype=np.int64)
    for b in boundaries:
        k += (pos > int(b)).astype(np.int64)
    return k


def heads_forward(H, rows, W1, b1, w2, b2):
    """z_k = w2_k . ReLU(H_r W1_k + b1_k) + b2_k for all k in one pass (R14)."""
    Hr = np.asarray(H, dtype=np.float64)[rows]
    K = W1.shape[0]
    pre = np.stack([Hr @ W1[k] + b1[k] for k in range(K)])          # [K, n, dh]
    hid = np.maximum(pre, 0.0)
    z = np.stack([hid[k] @ w2[k] + b2[k] for k in range(K)], axis=1)  # [n, K]
    return z, pre, hid


def heads_loss(z, bucket, label):
    """L_ctx = sum_t CE(y_hat_{k_t}, y_t) with logits (Eq. 9; R15 sum)."""
    zk = z[np.arange(z.shape[0]), bucket]
    return float(np.sum(softplus(zk) - label * zk))


def heads_loss_backward(H, rows, W1, b1, w2, b2, bucket, label, relu_active=None):
    """Routed BCE adjoint: dz_{k_t} = sigma(z_{k_t}) - y_t, 0 for other heads.

    relu_active (optional, [K][n, dh] bool): the ReLU derivative's 0/1 decision taken from the
    implementation under test, for pre-activations at the kink (|pre| ~ rounding) where the two
    sides may round to opposite signs; default pre > 0."""
    z, pre, hid = heads_forward(H, rows, W1, b1, w2, b2)
    n, K = z.shape
    dz = np.zeros_like(z)
    dz[np.arange(n), bucket] = sigmoid(z[np.arange(n), bucket]) - label
    Hr = np.asarray(H, dtype=np.float64)[rows]
    dW1 = np.zeros_like(W1, dtype=np.float64)
    db1 = np.zeros_like(b1, dtype=np.float64)
    dw2 = np.zeros_like(w2, dtype=np.float64)
    db2 = dz.sum(axis=0)
    dHr = np.zeros_like(Hr)
    for k in range(K):
        act = (pre[k] > 0) if relu_active is None else np.asarray(relu_active[k], dtype=bool)
        dhid = dz[:, k:k + 1] * w2[k][None, :] * act
        dW1[k] = Hr.T @ dhid
        db1[k] = dhid.sum(axis=0)
        dw2[k] = hid[k].T @ dz[:, k]
        dHr += dhid @ np.asarray(W1[k], dtype=np.float64).T
    dH = np.zeros_like(np.asarray(H, dtype=np.float64))
    np.add.at(dH, rows, dHr)
    return heads_loss(z, bucket, label), z, dH, dict(dW1=dW1, db1=db1, dw2=dw2, db2=db2)


# ------------------------------------------------------------------ NEXT-3: input embeddings (Eq. 1)
def embed_forward(ids, tables):
    """x_t = sum_f E_f[id_{t,f}] over the fields present for the token (id >= 0): the input sequence
    x = [M; I_1, (C_1, A_1); ...] of Eq. 1 as summed id + token-type embeddings (
    reading R37)."""
    ids = np.asarray(ids, dtype=np.int64)
    X = np.zeros((ids.shape[0], tables[0].shape[1]))
    for f, E in enumerate(tables):
        m = ids[:, f] >= 0
        X[m] += np.asarray(E, dtype=np.float64)[ids[m, f]]
    return X


def embed_backward(ids, dX, vocab):
    """Adjoint of embed_forward: dE_f[v] = sum of dX over the tokens whose field f has id v."""
    ids = np.asarray(ids, dtype=np.int64)
    dX = np.asarray(dX, dtype=np.float64)
    out = []
    for f, V in enumerate(vocab):
        g = np.zeros((V, dX.shape[1]))
        m = ids[:, f] >= 0
        np.add.at(g, ids[m, f], dX[m])
        out.append(g)
    return out


# ------------------------------------------------------------------ NEXT-2: full loss (Eqs. 10-12)
AUX_KINDS = ("bce", "se")  # R30: S:492 desk-scale tasks: long-dwell indicator (CE), impression duration (SE)


def aux_heads_forward(H, rows, W1a, b1a, w2a, b2a):
    """y^aux_j = MLP_j(h_t) (Eq. 10): J independent two-layer ReLU MLPs d -> da -> 1 on the
    impression rows (R30); no routing (not context-conditioned)."""
    return heads_forward(H, rows, W1a, b1a, w2a, b2a)


def aux_losses(za, ya, kinds=AUX_KINDS):
    """L_j^aux summed over impressions (R31): 'bce' = softplus(z) - y z (logits), 'se' = (z - y)^2."""
    out = []
    for j, kd in enumerate(kinds):
        z, y = za[:, j], ya[:, j]
        out.append(float(np.sum(softplus(z) - y * z)) if kd == "bce" else float(np.sum((z - y) ** 2)))
    return out


def aux_dz(za, ya, kinds=AUX_KINDS):
    """dL_j^aux / dz: sigma(z) - y (bce), 2 (z - y) (se)."""
    dz = np.zeros_like(np.asarray(za, dtype=np.float64))
    for j, kd in enumerate(kinds):
        dz[:, j] = (sigmoid(za[:, j]) - ya[:, j]) if kd == "bce" else 2.0 * (za[:, j] - ya[:, j])
    return dz


def pairwise_loss(z_pos, z_neg):
    """RankNet over the batch (Eq. 12): -1/(N+ N-) sum_i sum_j log sigma(z+_i - z-_j);
    0 when either set is empty (Eq. 12 undefined: S:459)."""
    z_pos, z_neg = np.asarray(z_pos, np.float64), np.asarray(z_neg, np.float64)
    if z_pos.size == 0 or z_neg.size == 0:
        return 0.0
    return float(np.sum(softplus(-(z_pos[:, None] - z_neg[None, :]))) / (z_pos.size * z_neg.size))


def pairwise_grad(z_pos, z_neg):
    """Adjoint of Eq. 12: dL/dz+_i = -1/(N+N-) sum_j sigma(z-_j - z+_i), dL/dz-_j = +1/(N+N-) sum_i
    sigma(z-_j - z+_i)."""
    z_pos, z_neg = np.asarray(z_pos, np.float64), np.asarray(z_neg, np.float64)
    if z_pos.size == 0 or z_neg.size == 0:
        return np.zeros_like(z_pos), np.zeros_like(z_neg)
    s = sigmoid(z_neg[None, :] - z_pos[:, None])
    c = 1.0 / (z_pos.size * z_neg.size)
    return -c * s.sum(axis=1), c * s.sum(axis=0)


def heads_backward_dz(H, rows, W1, b1, w2, b2, dz):
    """Tower backward from given logit gradients dz [n, K] (every tower, no routing)."""
    z, pre, hid = heads_forward(H, rows, W1, b1, w2, b2)
    Hr = np.asarray(H, dtype=np.float64)[rows]
    K = W1.shape[0]
    g = dict(dW1=np.zeros_like(W1, dtype=np.float64), db1=np.zeros_like(b1, dtype=np.float64),
             dw2=np.zeros_like(w2, dtype=np.float64), db2=dz.sum(axis=0))
    dHr = np.zeros_like(Hr)
    for k in range(K):
        dhid = dz[:, k:k + 1] * w2[k][None, :] * (pre[k] > 0)
        g["dW1"][k] = Hr.T @ dhid
        g["db1"][k] = dhid.sum(axis=0)
        g["dw2"][k] = hid[k].T @ dz[:, k]
        dHr += dhid @ np.asarray(W1[k], dtype=np.float64).T
    dH = np.zeros_like(np.asarray(H, dtype=np.float64))
    np.add.at(dH, rows, dHr)
    return dH, g


def full_loss_backward(H, rows, ctx, aux, bucket, label, ya, lam=(1.0, (0.1, 0.1), 0.1), kinds=AUX_KINDS):
    """Total loss (Eq. 11): L = lam_ctx L_ctx + sum_j lam_j L_j^aux + lam_pair L_pair, with
    L_ctx the routed BCE (Eq. 9) and L_pair RankNet over the routed context logits z_{k_t} of the
    batch (positives y = 1, negatives y = 0: R29).  ctx / aux = (W1, b1, w2, b2) of the towers and
    the auxiliary heads.  Returns (loss terms dict, dH, ctx grads, aux grads)."""
    lam_ctx, lam_aux, lam_pair = lam
    z, _, _ = heads_forward(H, rows, *ctx)
    za, _, _ = aux_heads_forward(H, rows, *aux)
    n = z.shape[0]
    zr = z[np.arange(n), bucket]
    pos, neg = label > 0.5, label <= 0.5
    terms = dict(ctx=heads_loss(z, bucket, label), aux=aux_losses(za, ya, kinds),
                 pair=pairwise_loss(zr[pos], zr[neg]))
    terms["total"] = lam_ctx * terms["ctx"] + sum(l * a for l, a in zip(lam_aux, terms["aux"])) + lam_pair * terms["pair"]
    dz = np.zeros_like(z)
    dz[np.arange(n), bucket] = lam_ctx * (sigmoid(zr) - label)
    gp, gn = pairwise_grad(zr[pos], zr[neg])
    dzr = np.zeros(n)
    dzr[pos], dzr[neg] = gp, gn
    dz[np.arange(n), bucket] += lam_pair * dzr
    dza = aux_dz(za, ya, kinds) * np.asarray(lam_aux, np.float64)[None, :]
    dH1, gc = heads_backward_dz(H, rows, *ctx, dz)
    dH2, ga = heads_backward_dz(H, rows, *aux, dza)
    return terms, dH1 + dH2, gc, ga


# ------------------------------------------------------------------ NEXT-3: the full CADET block
RMS_EPS = 1e-6


def rmsnorm(x, gamma, eps=RMS_EPS):
    """R32: y = x / sqrt(mean(x^2) + eps) * gamma per row (pre-norm, S:644 'two normalization layers')."""
    x = np.asarray(x, np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * np.asarray(gamma, np.float64)[None, :], r


def rmsnorm_backward(x, gamma, dy, eps=RMS_EPS):
    """Adjoint of rmsnorm: dx = r (g dy) - x r^3 mean(x g dy); dgamma = sum_rows dy x r."""
    x, dy, g = np.asarray(x, np.float64), np.asarray(dy, np.float64), np.asarray(gamma, np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    gd = dy * g[None, :]
    dx = r * gd - x * r ** 3 * np.mean(x * gd, axis=-1, keepdims=True)
    return dx, np.sum(dy * x * r, axis=0)


def gelu(u):
    """R33: exact GELU u Phi(u) ('smooth nonlinearity')."""
    u = np.asarray(u, np.float64)
    return 0.5 * u * (1.0 + np.vectorize(math.erf)(u / math.sqrt(2.0)))


def gelu_grad(u):
    u = np.asarray(u, np.float64)
    return 0.5 * (1.0 + np.vectorize(math.erf)(u / math.sqrt(2.0))) + u * np.exp(-0.5 * u * u) / math.sqrt(2 * math.pi)


def ffn_forward(x, W1, W2):
    """FFN(x) = GELU(x W1) W2, W1 [d, m d], W2 [m d, d], no biases (R33; multiplier m = 4)."""
    u = np.asarray(x, np.float64) @ W1
    return gelu(u) @ W2, u


def ffn_backward(x, W1, W2, u, dy):
    g = gelu(u)
    dg = dy @ W2.T
    du = dg * gelu_grad(u)
    return du @ W1.T, x.T @ du, g.T @ dy


def block_forward_seq(X, W, ffn, gammas, t_ms, A, cfg: AttnConfig):
    """Pre-norm CADET block: H = X + Attn(RMSNorm_1(X)); Y = H + FFN(RMSNorm_2(H))."""
    Xn, _ = rmsnorm(X, gammas[0])
    Ya, ca = layer_forward_seq(Xn, W, t_ms, A, cfg)
    H = np.asarray(X, np.float64) + Ya
    Hn, _ = rmsnorm(H, gammas[1])
    Yf, u = ffn_forward(Hn, *ffn)
    return H + Yf, dict(X=np.asarray(X, np.float64), Xn=Xn, ca=ca, H=H, Hn=Hn, u=u)


def block_backward_seq(c, W, ffn, gammas, t_ms, A, dY, cfg: AttnConfig):
    dHn, dW1f, dW2f = ffn_backward(c["Hn"], *ffn, c["u"], dY)
    dH_norm, dg2 = rmsnorm_backward(c["H"], gammas[1], dHn)
    dH = dY + dH_norm
    dXn, gW, _ = layer_backward_seq(c["ca"], W, t_ms, A, dH, cfg)
    dX_norm, dg1 = rmsnorm_backward(c["X"], gammas[0], dXn)
    return dH + dX_norm, dict(gW=gW, dW1f=dW1f, dW2f=dW2f, dg1=dg1, dg2=dg2)


# ------------------------------------------------------------------ NEXT-4: the optimizer of the HSDP step
def adamw_step(theta, m, v, g, step, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    """R35: AdamW (decoupled weight decay), bias-corrected, eps outside the square root — the update
    every rank applies to its shard of the fp32 master parameters (HSDP shards parameters, gradients
    and optimizer state within a node; the update is elementwise, so sharding does not change
    it).  Returns (theta', m', v'); step counts from 1."""
    theta, m, v, g = (np.asarray(a, np.float64) for a in (theta, m, v, g))
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** step)
    v_hat = v / (1.0 - beta2 ** step)
    theta = theta * (1.0 - lr * weight_decay) - lr * m_hat / (np.sqrt(v_hat) + eps)
    return theta, m, v


# ------------------------------------------------------------------ per-element loop (check 1)
def layer_forward_loop(X, W, t_ms, n_cand, cfg: AttnConfig, session_ids=None):
    """Independent evaluation for tiny inputs: pure-Python loops over (i, j) with
    the mask predicate evaluated per pair (no dense mask, no matmul for attention)."""
    X = np.asarray(X, dtype=np.float64)
    Wxg, Wq, Wk, Wv, Wqg, Wkg, Wo = [np.asarray(w, dtype=np.float64) for w in W]
    m, d = X.shape
    H, hd = cfg.n_heads, cfg.head_dim
    L = m - n_cand

    def sig(v):
        return 1.0 / (1.0 + math.exp(-v))

    def allowed(i, j):
        if i == j:
            return True
        if i < L:
            ok = j < i
            if cfg.mask_flags & MASK_TIME:
                ok = ok and t_ms[j] <= t_ms[i] - cfg.delta_delay_ms
            if cfg.mask_flags & MASK_SESSION:
                ok = ok and session_ids[j] < session_ids[i]
            return ok
        return j < L and t_ms[j] <= t_ms[i] - cfg.delta_cand_ms

    def vecmat(v, Wm):
        return [sum(v[a] * Wm[a][b] for a in range(d)) for b in range(d)]

    Xt, Qr, Kr, Vv = [], [], [], []
    for i in range(m):
        x = list(X[i])
        if cfg.use_rep_gate:
            z = vecmat(x, Wxg)
            x = [x[a] * sig(z[a]) for a in range(d)]
        q, k, v = vecmat(x, Wq), vecmat(x, Wk), vecmat(x, Wv)
        if cfg.use_int_gate:
            zq, zk = vecmat(q, Wqg), vecmat(k, Wkg)
            q = [q[a] * sig(zq[a]) for a in range(d)]
            k = [k[a] * sig(zk[a]) for a in range(d)]
        if cfg.use_rope:
            for h in range(H):
                for p in range(hd // 2):
                    th = (cfg.rope_phi_min / cfg.rope_dt_max_ms) * cfg.rope_base ** (2.0 * p / hd)
                    al = float(t_ms[i]) * th
                    for vec in (q, k):
                        a0, a1 = vec[h * hd + 2 * p], vec[h * hd + 2 * p + 1]
                        vec[h * hd + 2 * p] = a0 * math.cos(al) - a1 * math.sin(al)
                        vec[h * hd + 2 * p + 1] = a0 * math.sin(al) + a1 * math.cos(al)
        Qr.append(q); Kr.append(k); Vv.append(v)
    Y = np.zeros((m, d))
    for i in range(m):
        o = [0.0] * d
        for h in range(H):
            js = [j for j in range(m) if allowed(i, j)]
            sc = [sum(Qr[i][h * hd + a] * Kr[j][h * hd + a] for a in range(hd)) / math.sqrt(hd) for j in js]
            mx = max(sc)
            ex = [math.exp(s - mx) for s in sc]
            Z = sum(ex)
            for w, j in zip(ex, js):
                for a in range(hd):
                    o[h * hd + a] += (w / Z) * Vv[j][h * hd + a]
        Y[i] = vecmat(o, Wo) if cfg.use_out_proj else o
    return Y
