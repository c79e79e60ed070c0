"""Seeded synthetic workload generator.

This module produces *inputs only*: user histories (lengths, int64 Unix-ms
timestamps, session ids, labels, raw feed positions) and dense random tensors
(features X, weights, upstream gradients) rounded to bf16.  It holds none of
the method's arithmetic (no masking, RoPE, gating, attention, chunking or
packing): both the CUDA path and the CPU oracle consume what it returns.

Recipe (mirrors PAPER.md P:460):
  1. impressions n ~ round(LogNormal(ln 96, 1.5)), clipped to [1, max_tokens/2];
     each impression is 2 tokens (I_t, then (C_t, A_t)) sharing one timestamp.
  2. impressions per session ~ Geometric(1/3) on {1,2,...}; last session trimmed.
  3. user span ~ U(0.25, 1) * dt_max; inter-session gaps Exp(1) normalised to the
     span then floored at `session_gap_floor_ms` (1 h; 1 min in stress mode);
     intra-session gaps Exp(60 s), cumulative from the session start.
  4. events older than dt_max before the newest one are dropped (lookback).
  5. timestamps start at `t0_ms` (1,735,000,000,000; 0 in stress mode);
     session ids are per-user running counters.
  6. labels y ~ Bernoulli(0.03), feed position p ~ U{1..8} per impression (the raw context signal
     of P:624; bucketing it is the method's step, not the generator's).
  7. serving shape (C2): context of U{448..576}-64 tokens from the same session
     process; 64 candidates share one request time = last context time + Exp(10 min).
Per-user RNG streams are keyed by (seed, user).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

MS_PER_YEAR = 365 * 24 * 3600 * 1000          # R6: 31,536,000,000 ms
MS_PER_DAY = 24 * 3600 * 1000
T0_UNIX_MS = 1_735_000_000_000


@dataclass
class UserHistory:
    timestamps: np.ndarray      # int64 [m], non-decreasing
    session_ids: np.ndarray     # int32 [m], non-decreasing
    labels: np.ndarray          # float32 [m] (meaningful on impression rows)
    positions: np.ndarray       # int32 [m] raw feed position >= 1 (meaningful on impression rows)
    impression_rows: np.ndarray  # int32 local positions of impression tokens
    n_candidates: int = 0

    @property
    def length(self) -> int:
        return int(self.timestamps.shape[0])


@dataclass
class GenConfig:
    median_impressions: float = 96.0
    sigma: float = 1.5
    max_tokens: int = 8192
    dt_max_ms: int = MS_PER_YEAR
    session_gap_floor_ms: int = 3600 * 1000
    intra_gap_mean_ms: float = 60_000.0
    t0_ms: int = T0_UNIX_MS
    ctr: float = 0.03
    max_position: int = 8


def stress_config(**kw) -> GenConfig:
    """R7 stress mode: dt_max = 1 day, timestamps from 0, 1-minute session-gap floor."""
    base = dict(dt_max_ms=MS_PER_DAY, session_gap_floor_ms=60_000, t0_ms=0)
    base.update(kw)
    return GenConfig(**base)


def _session_times(rng: np.random.Generator, n_imp: int, cfg: GenConfig) -> tuple[np.ndarray, np.ndarray]:
    """Impression timestamps + session ids for one user (steps 2-5)."""
    sizes = []
    left = n_imp
    while left > 0:
        s = int(rng.geometric(1.0 / 3.0))
        s = min(s, left)
        sizes.append(s)
        left -= s
    n_sess = len(sizes)
    span = rng.uniform(0.25, 1.0) * cfg.dt_max_ms
    if n_sess > 1:
        gaps = rng.exponential(1.0, size=n_sess - 1)
        gaps = gaps / gaps.sum() * span
        gaps = np.maximum(gaps, cfg.session_gap_floor_ms)
    else:
        gaps = np.zeros(0)
    starts = np.concatenate([[0.0], np.cumsum(gaps)])
    ts, sid = [], []
    for s_idx, (st, sz) in enumerate(zip(starts, sizes)):
        intra = np.cumsum(rng.exponential(cfg.intra_gap_mean_ms, size=sz)) - 0.0
        intra[0] = 0.0 if sz > 0 else 0.0
        ts.append(st + intra)
        sid.append(np.full(sz, s_idx, dtype=np.int32))
    t = np.concatenate(ts)
    t = np.floor(t).astype(np.int64) + np.int64(cfg.t0_ms)
    t = np.maximum.accumulate(t)             # guard: non-decreasing after flooring
    s = np.concatenate(sid)
    # step 4: lookback window relative to the newest event
    keep = t >= t[-1] - cfg.dt_max_ms
    return t[keep], s[keep]


def gen_user(seed: int, user: int, cfg: GenConfig) -> UserHistory:
    """One fully-labelled user history (steps 1-6): 2 tokens per impression."""
    rng = np.random.default_rng([seed, user])
    n = int(round(rng.lognormal(np.log(cfg.median_impressions), cfg.sigma)))
    n = int(np.clip(n, 1, cfg.max_tokens // 2))
    t_imp, s_imp = _session_times(rng, n, cfg)
    n = t_imp.shape[0]
    t = np.repeat(t_imp, 2)
    s = np.repeat(s_imp, 2)
    y = np.zeros(2 * n, dtype=np.float32)
    k = np.zeros(2 * n, dtype=np.int32)
    y[0::2] = (rng.random(n) < cfg.ctr).astype(np.float32)
    k[0::2] = rng.integers(1, cfg.max_position + 1, size=n).astype(np.int32)
    rows = np.arange(0, 2 * n, 2, dtype=np.int32)
    return UserHistory(t, s.astype(np.int32), y, k, rows, 0)


def gen_serving_user(seed: int, user: int, cfg: GenConfig, lo: int = 448, hi: int = 576,
                     n_cand: int = 64) -> UserHistory:
    """C2 serving shape (step 7): context + n_cand candidates sharing one request time."""
    rng = np.random.default_rng([seed, user])
    m = int(rng.integers(lo, hi + 1))
    L = m - n_cand
    n_imp = (L + 1) // 2
    t_imp, s_imp = _session_times(rng, n_imp, cfg)
    while 2 * t_imp.shape[0] < L:          # lookback dropped events: pad with more at the end
        t_imp = np.concatenate([t_imp, t_imp[-1:]])
        s_imp = np.concatenate([s_imp, s_imp[-1:]])
    t_ctx = np.repeat(t_imp, 2)[:L]
    s_ctx = np.repeat(s_imp, 2)[:L]
    t_req = t_ctx[-1] + np.int64(np.floor(rng.exponential(600_000.0)))
    t = np.concatenate([t_ctx, np.full(n_cand, t_req, dtype=np.int64)])
    s = np.concatenate([s_ctx, np.full(n_cand, s_ctx[-1] + 1, dtype=np.int32)])
    y = (rng.random(m) < cfg.ctr).astype(np.float32)
    k = rng.integers(1, cfg.max_position + 1, size=m).astype(np.int32)
    rows = np.arange(L, m, dtype=np.int32)
    return UserHistory(t, s.astype(np.int32), y, k, rows, n_cand)


def gen_users_for_budget(seed: int, budget: int, cfg: GenConfig, first_user: int = 0) -> list[UserHistory]:
    """Draw users in arrival order until the next one would overflow `budget` tokens.

    This is the data-loader side of P:462 ("aggregates user sequences until the
    packed length approaches a configured budget"); the pack step itself
    (offsets, padding to exactly `budget`) belongs to the method.
    """
    users, total, u = [], 0, first_user
    while True:
        h = gen_user(seed, u, cfg)
        if total + h.length > budget:
            break
        users.append(h)
        total += h.length
        u += 1
    return users


# ---------------------------------------------------------------- dense tensors
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bf16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    b = (b + 0x7FFF + lsb) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of bf16-rounded values (for handing to the device)."""
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def normal_bf16(seed: int, stream: int, shape, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng([seed, 7919, stream])
    return bf16_round(rng.standard_normal(size=shape, dtype=np.float32) * np.float32(scale))


@dataclass
class LayerWeights:
    """Seven d x d matrices, y = x.W with W[d_in][d_out], bf16-valued float32."""
    W_xg: np.ndarray
    W_q: np.ndarray
    W_k: np.ndarray
    W_v: np.ndarray
    W_qg: np.ndarray
    W_kg: np.ndarray
    W_o: np.ndarray

    def as_list(self):
        return [self.W_xg, self.W_q, self.W_k, self.W_v, self.W_qg, self.W_kg, self.W_o]


NAMES = ["W_xg", "W_q", "W_k", "W_v", "W_qg", "W_kg", "W_o"]


def layer_weights(seed: int, layer: int, d: int, peaky: bool = False) -> LayerWeights:
    """N(0, 1/d) weights; W_q, W_k x4 in the 'peaky' regime."""
    s = 1.0 / np.sqrt(d)
    ws = {}
    for i, n in enumerate(NAMES):
        scale = s * (4.0 if (peaky and n in ("W_q", "W_k")) else 1.0)
        ws[n] = normal_bf16(seed, 1000 * (layer + 1) + i, (d, d), scale)
    return LayerWeights(**ws)


@dataclass
class HeadWeights:
    W1: np.ndarray   # [K, d, dh]
    b1: np.ndarray   # [K, dh]
    w2: np.ndarray   # [K, dh]
    b2: np.ndarray   # [K]


def head_weights(seed: int, K: int, d: int, dh: int) -> HeadWeights:
    return HeadWeights(
        W1=normal_bf16(seed, 90001, (K, d, dh), 1.0 / np.sqrt(d)),
        b1=normal_bf16(seed, 90002, (K, dh), 0.1),
        w2=normal_bf16(seed, 90003, (K, dh), 1.0 / np.sqrt(dh)),
        b2=normal_bf16(seed, 90004, (K,), 0.1),
    )


@dataclass
class Batch:
    """A list of sequences laid out back to back (arrival order) plus per-token data."""
    users: list
    lengths: np.ndarray
    timestamps: np.ndarray
    session_ids: np.ndarray
    n_candidates: np.ndarray
    token_flags: np.ndarray = field(default=None)

    @property
    def n_tokens(self) -> int:
        return int(self.lengths.sum())


def concat_users(users: list[UserHistory]) -> Batch:
    lengths = np.array([u.length for u in users], dtype=np.int32)
    ts = np.concatenate([u.timestamps for u in users]) if users else np.zeros(0, np.int64)
    ss = np.concatenate([u.session_ids for u in users]) if users else np.zeros(0, np.int32)
    nc = np.array([u.n_candidates for u in users], dtype=np.int32)
    return Batch(users, lengths, ts.astype(np.int64), ss.astype(np.int32), nc)


def fixed_lengths_batch(lengths, seed: int = 0, cfg: GenConfig | None = None, n_cand=None) -> Batch:
    """Sequences of given lengths with generator timestamps (C1 and tests)."""
    cfg = cfg or GenConfig()
    users = []
    for u, m in enumerate(lengths):
        rng = np.random.default_rng([seed, 5003, u])
        n_imp = max(1, (m + 1) // 2)
        t_imp, s_imp = _session_times(rng, n_imp, cfg)
        while 2 * t_imp.shape[0] < m:
            t_imp = np.concatenate([t_imp, t_imp[-1:]])
            s_imp = np.concatenate([s_imp, s_imp[-1:]])
        t = np.repeat(t_imp, 2)[:m]
        s = np.repeat(s_imp, 2)[:m]
        y = (rng.random(m) < 0.3).astype(np.float32)
        k = rng.integers(1, cfg.max_position + 1, size=m).astype(np.int32)
        nc = 0 if n_cand is None else int(n_cand[u])
        users.append(UserHistory(t, s.astype(np.int32), y, k, np.arange(0, m, 2, dtype=np.int32), nc))
    return concat_users(users)


EMBED_VOCAB = (2, 16384, 8, 4)   # token type (impression / action), ad id, request feature, action id


def token_ids(seed: int, users, vocab=EMBED_VOCAB) -> np.ndarray:
    """Per-token integer ids of the embedded input fields (Eq. 1), int32 [R, 4] for the
    users' tokens back to back, -1 = field absent for the token kind (R37):
      column 0  token type: 0 = impression I_t (even local rows), 1 = action token (C_t, A_t)
      column 1  ad id of the impression, Zipf(1.2) over vocab[1] (impressions only)
      column 2  request feature (e.g. device type) ~ U{0 .. vocab[2]-1} (impressions only)
      column 3  action id ~ U{0 .. vocab[3]-1} (action tokens only)
    Raw categorical inputs only: looking the rows up and summing them is the method's step."""
    out = []
    for u, usr in enumerate(users):
        rng = np.random.default_rng([seed, 7919, u])
        m = usr.length
        ids = np.full((m, 4), -1, dtype=np.int32)
        imp = (np.arange(m) % 2) == 0
        ids[:, 0] = np.where(imp, 0, 1)
        n_i, n_a = int(imp.sum()), int((~imp).sum())
        ids[imp, 1] = (rng.zipf(1.2, size=n_i) - 1) % vocab[1]
        ids[imp, 2] = rng.integers(0, vocab[2], size=n_i)
        ids[~imp, 3] = rng.integers(0, vocab[3], size=n_a)
        out.append(ids)
    return np.concatenate(out) if out else np.zeros((0, 4), np.int32)


def embed_tables(seed: int, d: int, vocab=EMBED_VOCAB) -> list:
    """Embedding tables E_f ~ N(0, 1/len(vocab)) rounded to bf16 (the summed row has unit variance)."""
    return [normal_bf16(seed, 8000 + f, (V, d), scale=1.0 / np.sqrt(len(vocab))) for f, V in enumerate(vocab)]


def aux_labels(seed: int, n: int) -> np.ndarray:
    """Auxiliary-task targets per impression (NEXT-2): column 0 a long-dwell indicator
    (Bernoulli 0.2), column 1 an impression duration in minutes (log-normal, median 0.5).
    float32 [n, 2]."""
    rng = np.random.default_rng([seed, 17])
    out = np.empty((n, 2), np.float32)
    out[:, 0] = (rng.random(n) < 0.2).astype(np.float32)
    out[:, 1] = np.exp(rng.normal(np.log(0.5), 0.8, size=n)).astype(np.float32)
    return out



@dataclass
class BlockWeights:
    """NEXT-3 (R32, R33): the pre-norm block's RMSNorm scales and FFN weights."""
    gamma1: np.ndarray  # [d] fp32 (bf16-valued)
    gamma2: np.ndarray  # [d]
    W1: np.ndarray      # [d, m d]
    W2: np.ndarray      # [m d, d]


def block_weights(seed: int, layer: int, d: int, m: int = 4) -> BlockWeights:
    """gamma = 1 + N(0, 0.1^2); W1 ~ N(0, 1/d), W2 ~ N(0, 1/(m d)) (unit-variance activations)."""
    base = 5000 * (layer + 1)
    return BlockWeights(
        gamma1=1.0 + normal_bf16(seed, base + 1, (d,), 0.1),
        gamma2=1.0 + normal_bf16(seed, base + 2, (d,), 0.1),
        W1=normal_bf16(seed, base + 3, (d, m * d), 1.0 / np.sqrt(d)),
        W2=normal_bf16(seed, base + 4, (m * d, d), 1.0 / np.sqrt(m * d)),
    )
