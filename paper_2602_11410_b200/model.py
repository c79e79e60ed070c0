"""CADET hot-path training step over the libcadet C ABI (one process per GPU).

A step (in order):
  A13 pack   contiguous user histories -> fixed budget T (cadet_pack)
  A0  chunk  refine offsets so no sequence exceeds L_chunk (cadet_chunk)
  A1-A6      L residual layers of self-gated attention forward (cadet_attn_forward; plan inside)
  A7-A8      context-conditioned towers + routed BCE + tower backward (cadet_heads_*)
  A9-A12     layers backward (cadet_attn_backward), weight gradients into one flat fp32 buffer
  DP         SURVEY 8(e), NCCL through torch.distributed when world > 1: per-layer gradient buckets
             all-reduced (SUM) asynchronously as soon as each layer's backward is enqueued, loss and
             impression count all-reduced, logits + labels all-gathered (dp_gather_scores); whole
             users are assigned to ranks by LPT on estimated cost (partition_lpt)
  NEXT-2..4  optional: the full Eq. 11 loss (full_loss), the pre-norm block (block), gradient
             checkpointing (recompute), and the AdamW step with HSDP sharding within the node
             (optimizer="adamw": reduce-scatter, shard update, bf16 all-gather)
Every computation is a libcadet kernel; PyTorch only allocates memory, provides the stream and
runs the NCCL collective.
"""
from __future__ import annotations

import ctypes as C
import math
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
    boundaries: tuple = (4,)     # context buckets from raw positions: K = 2 "positions 1--4, and 5+"
    d_hidden: int = 0            # 0 -> d_model // 2
    delta_delay_ms: int = 3_600_000
    mask_flags: int = L.CADET_MASK_TIME
    full_loss: bool = False      # NEXT-2: Eq. 11 = ctx + aux heads (Eq. 10) + RankNet (Eq. 12)
    recompute: bool = False      # gradient checkpointing: one `saved` buffer, layers re-run fwd in bwd
    J: int = 2                   # auxiliary tasks (long-dwell BCE, duration SE)
    block: bool = False          # NEXT-3: pre-norm CADET block (RMSNorm, attention, RMSNorm, FFN, R32/R33)
    ffn_mult: int = 4            # FFN width multiplier m
    optimizer: str = "none"      # NEXT-4: "adamw" appends the optimizer step (R35) to every training step
    shard: bool = True           # NEXT-4 with a process group: HSDP within the node (reduce-scatter grads, AdamW on
                                 # this rank's shard of master params + moments, all-gather bf16 params)
    lr: float = 1e-4
    weight_decay: float = 0.0
    embed: bool = False          # NEXT-3 input embeddings (Eq. 1): H[0] = sum of id + type embedding rows
    vocab: tuple = (2, 16384, 8, 4)  # token type, ad id, request feature, action id (synth.generator.EMBED_VOCAB)
    taps: bool = False           # parity taps (cfg.out_f32 = 1 on the layer calls): fp32 stage values in the
                                 # workspace, read with cadet_attn_stage_views (tests only; ~2x the layer time)

    @property
    def dh(self) -> int:
        return self.d_hidden or self.d_model // 2

    @property
    def da(self) -> int:
        """Aux head width (R30): d / 4 rounded up so that J * da is a multiple of 32."""
        q = 32 // math.gcd(32, self.J)
        return -(-(self.d_model // 4) // q) * q


@dataclass
class StepInputs:
    """Device (or pinned host) tensors of one step plus host-side counts known to the loader."""
    X_hist: torch.Tensor     # [R, d] bf16, histories back to back (arrival order)
    t_hist: torch.Tensor     # [R] int64 Unix ms
    s_hist: torch.Tensor     # [R] int32 session ids
    lens: torch.Tensor       # [B] int32 history lengths
    rows: torch.Tensor       # [n_imp] int32 packed rows of impression tokens
    position: torch.Tensor   # [n_imp] int32 raw feed position (>= 1) of impression t: the context signal
    label: torch.Tensor      # [n_imp] fp32 click label y_t
    n_hist: int
    n_chunks: int
    tokens: int              # real tokens T_r
    aux_label: torch.Tensor | None = None  # [n_imp, J] fp32 (NEXT-2 full loss)
    ids: torch.Tensor | None = None        # [R, F] int32 embedded field ids (NEXT-3 embeddings; X_hist is None)

    def to(self, device, non_blocking=True) -> "StepInputs":
        f = lambda t: t.to(device, non_blocking=non_blocking) if t is not None else None
        return StepInputs(f(self.X_hist), f(self.t_hist), f(self.s_hist), f(self.lens), f(self.rows),
                          f(self.position), f(self.label), self.n_hist, self.n_chunks, self.tokens, f(self.aux_label),
                          f(self.ids))

    FIELDS = ("X_hist", "t_hist", "s_hist", "lens", "rows", "position", "label", "aux_label", "ids")

    def copy_(self, src: "StepInputs"):
        for a in self.FIELDS:
            if getattr(self, a) is not None:
                getattr(self, a).copy_(getattr(src, a), non_blocking=True)

    def nbytes(self) -> int:
        return sum(getattr(self, a).numel() * getattr(self, a).element_size() for a in self.FIELDS
                   if getattr(self, a) is not None)


def make_inputs(users, d: int, L_chunk: int, seed: int, pin: bool = False, J: int = 0, vocab=None) -> StepInputs:
    """Host-side data loader output for one batch of generator users (synth/ Appendix B).  With `vocab`
    (NEXT-3 embeddings) the tokens carry their field ids instead of dense feature rows."""
    from synth import generator as G
    lens = np.array([u.length for u in users], dtype=np.int32)
    R = int(lens.sum())
    X = G.normal_bf16(seed, 11, (R, d)) if vocab is None else None
    t = np.concatenate([u.timestamps for u in users]).astype(np.int64)
    s = np.concatenate([u.session_ids for u in users]).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    rows = np.concatenate([st + u.impression_rows for st, u in zip(starts, users)]).astype(np.int32)
    position = np.concatenate([u.positions[u.impression_rows] for u in users]).astype(np.int32)
    label = np.concatenate([u.labels[u.impression_rows] for u in users]).astype(np.float32)
    n_chunks = int(sum(-(-int(m) // L_chunk) for m in lens))
    mk = lambda a, dt: (torch.from_numpy(np.ascontiguousarray(a)).to(dt))
    Xt = torch.from_numpy(X).to(torch.bfloat16) if X is not None else None
    aux = mk(G.aux_labels(seed, len(rows))[:, :J], torch.float32) if J > 0 else None
    ids = mk(G.token_ids(seed, users, vocab), torch.int32) if vocab is not None else None
    inp = StepInputs(Xt, mk(t, torch.int64), mk(s, torch.int32), mk(lens, torch.int32), mk(rows, torch.int32),
                     mk(position, torch.int32), mk(label, torch.float32), len(users), n_chunks, R, aux, ids)
    if pin:
        pinned = [x.pin_memory() if x is not None else None for x in (inp.X_hist, inp.t_hist, inp.s_hist, inp.lens,
                                                                       inp.rows, inp.position, inp.label, inp.aux_label,
                                                                       inp.ids)]
        inp = StepInputs(*pinned[:7], inp.n_hist, inp.n_chunks, inp.tokens, pinned[7], pinned[8])
    return inp


def dp_reduce(grads: torch.Tensor, loss: torch.Tensor, group=None):
    """the routed loss is a SUM over impressions (Eq. 9, R15), so summing the ranks'
    flat fp32 gradient buffers (one NCCL all-reduce bucket) gives exactly the union-batch gradient."""
    if group is None:
        return grads, loss
    torch.distributed.all_reduce(grads, group=group)
    torch.distributed.all_reduce(loss, group=group)
    return grads, loss


class GradBuckets:
    """gradient buckets all-reduced (SUM) as soon as their producer is enqueued.

    `launch(i)` starts an async all_reduce of bucket i (NCCL orders it after the work already on
    the current stream, so it overlaps the backward of earlier layers); `wait()` joins them all.
    Summation is exact for the union batch because the loss is a sum (Eq. 9, R15)."""

    def __init__(self, buckets, group=None):
        self.buckets = list(buckets)
        self.group = group
        self.handles = []

    def launch(self, i: int):
        if self.group is not None:
            self.handles.append(torch.distributed.all_reduce(self.buckets[i], group=self.group, async_op=True))

    def wait(self):
        for h in self.handles:
            h.wait()
        self.handles = []


def dp_reduce_stats(loss: torch.Tensor, n_imp: int, group=None):
    """global loss sum and impression count (one all_reduce of a 2-vector)."""
    v = torch.stack([loss.reshape(-1)[0].to(torch.float64), torch.tensor(float(n_imp), dtype=torch.float64,
                                                                        device=loss.device)])
    if group is not None:
        torch.distributed.all_reduce(v, group=group)
    return float(v[0].item()), int(round(float(v[1].item())))


def dp_gather_scores(logits: torch.Tensor, labels: torch.Tensor, group=None):
    """all_gather of the ranks' logits [n_r, K] and labels [n_r] (evaluation and
    the cross-user pairwise loss of NEXT-2).  n_r differs per rank: gather the counts first, pad to
    the maximum, gather, then drop the padding.  Returns rank-ordered concatenations."""
    if group is None:
        return logits, labels
    world = torch.distributed.get_world_size(group)
    n = torch.tensor([logits.shape[0]], dtype=torch.int64, device=logits.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    torch.distributed.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    lp = torch.zeros((m,) + tuple(logits.shape[1:]), dtype=logits.dtype, device=logits.device)
    yp = torch.zeros((m,), dtype=labels.dtype, device=labels.device)
    lp[: logits.shape[0]] = logits
    yp[: labels.shape[0]] = labels
    gl = [torch.empty_like(lp) for _ in range(world)]
    gy = [torch.empty_like(yp) for _ in range(world)]
    torch.distributed.all_gather(gl, lp, group=group)
    torch.distributed.all_gather(gy, yp, group=group)
    return (torch.cat([g[:c] for g, c in zip(gl, counts)]), torch.cat([g[:c] for g, c in zip(gy, counts)]))


def chunk_lengths(length: int, L_chunk: int):
    """A0 split of one history (newest chunk full, oldest may be short)."""
    n = -(-int(length) // L_chunk)
    return [int(length) - (n - 1) * L_chunk] + [L_chunk] * (n - 1) if n > 0 else []


def user_cost(length: int, L_chunk: int, d_model: int) -> float:
    """Estimated step cost of one user: per chunk c1 len + c2 len^2 with c1 = 7 d, c2 = 1, i.e. the
    42 d^2 projection flops per token against ~6 d len attention flops per token (len / 2 visible
    keys, 12 d flops per pair fwd + bwd), in units of 6 d flops."""
    return float(sum(7.0 * d_model * c + float(c) * c for c in chunk_lengths(length, L_chunk)))


def partition_lpt(lens, world: int, budget: int, L_chunk: int, d_model: int):
    """SURVEY 8(e) partitioning: whole users (their chunks stay together, chunking runs on device)
    to ranks by longest-processing-time-first on user_cost, each rank under its token budget.
    Deterministic (ties by user index, then rank).  Returns per-rank sorted user-index arrays
    (arrival order is kept inside a rank).  Raises if a user cannot be placed."""
    lens = [int(x) for x in lens]
    cost = [user_cost(m, L_chunk, d_model) for m in lens]
    order = sorted(range(len(lens)), key=lambda i: (-cost[i], i))
    load = [0.0] * world
    tokens = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        best = None
        for r in range(world):
            if tokens[r] + lens[i] <= budget and (best is None or load[r] < load[best]):
                best = r
        if best is None:
            raise ValueError(f"user {i} ({lens[i]} tokens) fits no rank under budget {budget}")
        out[best].append(i)
        load[best] += cost[i]
        tokens[best] += lens[i]
    return [np.array(sorted(o), dtype=np.int64) for o in out]


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def shard_range(n: int, world: int, rank: int):
    """NEXT-4: [lo, hi) of rank's equal shard of a flat buffer of n elements (n % (64 world) == 0, so
    every shard is 256-byte aligned; reduce_scatter_tensor / all_gather_into_tensor split the same way)."""
    if n % (64 * world):
        raise ValueError(f"flat buffer of {n} elements does not split into {world} aligned shards")
    s = n // world
    return rank * s, (rank + 1) * s


class CadetStack:
    """Weights, activations and workspaces for L layers + towers on one GPU."""

    def __init__(self, cfg: StackConfig, seed: int = 0, device="cuda", peaky: bool = False):
        from synth import generator as G
        self.cfg = cfg
        self.dev = torch.device(device)
        d, T, nl = cfg.d_model, cfg.budget, cfg.n_layers
        assert cfg.K == len(cfg.boundaries) + 1, "K towers need K - 1 bucket boundaries"
        self.acfg = ops.config(d, cfg.n_heads, delta_delay_ms=cfg.delta_delay_ms, mask_flags=cfg.mask_flags,
                               out_f32=1 if cfg.taps else 0)
        # ONE flat layout for gradients and parameters: 7 d^2 per layer (+ the block's FFN and RMSNorm
        # scales, NEXT-3), the towers (+ the aux heads, NEXT-2); every slice starts on a 256-byte
        # boundary (the split-K weight-gradient epilogue adds float4 atomics) and the total is padded to
        # a multiple of 8 x 64 elements so it splits into equal, aligned shards for 1/2/4/8 ranks (NEXT-4)
        N = cfg.K * cfg.dh
        Na = cfg.J * cfg.da if cfg.full_loss else 0
        md = cfg.ffn_mult * d
        pad = lambda x: -(-x // 64) * 64
        per_layer = [d * d] * 7 + ([d * md, md * d, d, d] if cfg.block else [])
        kind_layer = ["m"] * 7 + (["m", "m", "v", "v"] if cfg.block else [])
        npl = len(per_layer)
        sizes = per_layer * nl + [d * N, N, N, cfg.K] + ([d * Na, Na, Na, cfg.J] if cfg.full_loss else [])
        kinds = kind_layer * nl + ["m", "v", "v", "v"] + (["m", "v", "v", "v"] if cfg.full_loss else [])
        n_before_embed = len(sizes)
        if cfg.embed:  # NEXT-3 embedding tables (bf16 compute copies, fp32 gradients) after everything else
            sizes += [V * d for V in cfg.vocab]
            kinds += ["m"] * len(cfg.vocab)
        self.n_grad = -(-sum(pad(x) for x in sizes) // 512) * 512
        self.grads = torch.zeros(self.n_grad, dtype=torch.float32, device=self.dev)
        # parameters: bf16 compute copies (matrices are consumed as bf16) and fp32 compute copies (vectors:
        # biases, w2, RMSNorm scales are consumed as fp32), both in the flat layout
        self.wbf = torch.zeros(self.n_grad, dtype=torch.bfloat16, device=self.dev)
        self.wf32 = torch.zeros(self.n_grad, dtype=torch.float32, device=self.dev)
        views, pviews, offs, off = [], [], [], 0
        for x, k in zip(sizes, kinds):
            views.append(self.grads[off:off + x])
            pviews.append(self.wbf[off:off + x] if k == "m" else self.wf32[off:off + x])
            offs.append(off)
            off += pad(x)
        self._slices = list(zip(offs, sizes, kinds))

        def put(i, a, shape=None):  # initial value of parameter slice i
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32).reshape(-1)).to(self.dev)
            pviews[i].copy_(t)
            self.wbf[offs[i]:offs[i] + sizes[i]].copy_(t)  # bf16 copy of every slice (the all-gathered copy)
            return pviews[i].view(*shape) if shape else pviews[i]
        self.W = [[put(npl * l + i, w, (d, d)) for i, w in enumerate(G.layer_weights(seed, l, d, peaky).as_list())]
                  for l in range(nl)]
        if cfg.block:  # NEXT-3: FFN weights (bf16) and RMSNorm scales (fp32) per layer
            bw = [G.block_weights(seed, l, d, cfg.ffn_mult) for l in range(nl)]
            self.F = [(put(npl * l + 7, w.W1, (d, md)), put(npl * l + 8, w.W2, (md, d))) for l, w in enumerate(bw)]
            self.gam = [(put(npl * l + 10, w.gamma1), put(npl * l + 9, w.gamma2)) for l, w in enumerate(bw)]
            self.gF = [views[npl * l + 7:npl * l + 11] for l in range(nl)]  # dW1f, dW2f, dgamma2, dgamma1
        t0 = npl * nl
        hw = G.head_weights(seed, cfg.K, d, cfg.dh)
        self.W1 = put(t0, np.concatenate([hw.W1[k] for k in range(cfg.K)], axis=1), (d, N))
        self.b1, self.w2, self.b2 = put(t0 + 1, hw.b1), put(t0 + 2, hw.w2), put(t0 + 3, hw.b2)
        self.gW = [views[npl * l:npl * l + 7] for l in range(nl)]
        # DP all-reduce groups per layer, in the order their gradients complete in the backward
        rng_ = lambda a, b: self.grads[offs[a]:offs[b - 1] + pad(sizes[b - 1])]
        self._groups = [dict(attn=(rng_(npl * l + 6, npl * l + 7), rng_(npl * l + 4, npl * l + 6),
                                   rng_(npl * l + 1, npl * l + 4), rng_(npl * l, npl * l + 1)),
                             ffn=rng_(npl * l + 7, npl * l + 10) if cfg.block else None,
                             g1=rng_(npl * l + 10, npl * l + 11) if cfg.block else None) for l in range(nl)]
        self.gW1, self.gb1, self.gw2, self.gb2 = views[t0:t0 + 4]
        self._tower_off = offs[t0]  # towers (and aux heads) follow the layers
        self._embed_off = offs[n_before_embed] if cfg.embed else self.n_grad  # then the embedding tables
        if cfg.embed:
            et = G.embed_tables(seed, d, cfg.vocab)
            self.E = [put(n_before_embed + f, et[f], (V, d)) for f, V in enumerate(cfg.vocab)]
            self.dE = [views[n_before_embed + f].view(V, d) for f, V in enumerate(cfg.vocab)]
            self.ecfg = L.EmbedConfig(len(cfg.vocab), d, (C.c_int32 * 8)(*cfg.vocab))
            self._ews = ops.workspace(L.lib().cadet_embed_workspace_bytes(C.byref(self.ecfg)), self.dev)
        if cfg.full_loss:  # NEXT-2 auxiliary heads (Eq. 10): J towers of width da, never routed
            aw = G.head_weights(seed + 1, cfg.J, d, cfg.da)
            self.aW1 = put(t0 + 4, np.concatenate([aw.W1[k] for k in range(cfg.J)], axis=1), (d, Na))
            self.ab1, self.aw2, self.ab2 = put(t0 + 5, aw.b1), put(t0 + 6, aw.w2), put(t0 + 7, aw.b2)
            self.agW1, self.agb1, self.agw2, self.agb2 = views[t0 + 4:t0 + 8]
            self.lcfg = L.LossConfig()
            L.lib().cadet_default_loss_config(C.byref(self.lcfg), cfg.J)
            self.losses = torch.zeros(cfg.J + 3, dtype=torch.float32, device=self.dev)
        self._opt = None           # NEXT-4 optimizer state, built at the first optimizer step
        lib = L.lib()
        self.saved_bytes = lib.cadet_attn_saved_bytes(C.byref(self.acfg), T)
        # gradient checkpointing keeps only the layer inputs Hs[l] and ONE saved-activation buffer,
        # refilled by re-running layer l's forward right before its backward
        n_saved = 1 if cfg.recompute else nl
        self.saved = [torch.empty(self.saved_bytes, dtype=torch.uint8, device=self.dev) for _ in range(n_saved)]
        self._rec_y = torch.empty(T, d, dtype=torch.bfloat16, device=self.dev) if cfg.recompute else None
        self.Hs = [torch.empty(T, d, dtype=torch.bfloat16, device=self.dev) for _ in range(nl + 1)]
        if cfg.block:  # per (saved) layer: Xn, H (after attention), Hn, rstd1, rstd2, U, G; backward scratch
            bt = lambda n: torch.empty(T, n, dtype=torch.bfloat16, device=self.dev)
            ft = lambda: torch.empty(T, dtype=torch.float32, device=self.dev)
            self.blk = [dict(Xn=bt(d), H=bt(d), Hn=bt(d), r1=ft(), r2=ft(), U=bt(md), G=bt(md)) for _ in range(n_saved)]
            self._dA, self._dB = bt(d), bt(d)
            self._fws = ops.workspace(lib.cadet_ffn_workspace_bytes(T, d, cfg.ffn_mult), self.dev)
        self.dHs = [torch.empty(T, d, dtype=torch.bfloat16, device=self.dev) for _ in range(nl + 1)]
        self.t_p = torch.empty(T, dtype=torch.int64, device=self.dev)
        self.s_p = torch.empty(T, dtype=torch.int32, device=self.dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.small_ws = ops.workspace(4096, self.dev)
        self._ws = None
        self._hws = None
        self._bufs_for = None
        self._side = None          # DP: stream on which per-group gradient all-reduces are issued
        self._pack_stream = None   # side stream of the A13 row move
        self._pack_done = None
        self._grad_events = None   # DP: [layer][4] events recorded by cadet_attn_backward_ev

    # -------------------------------------------------------------- buffers sized per batch
    def _ensure(self, n_chunks: int, n_imp: int, n_hist: int):
        key = (n_chunks, n_imp, n_hist)
        if self._bufs_for == key:
            return
        lib = L.lib()
        cfg = self.cfg
        # + the dS region of the two-pass attention backward (cadet_attn_bwd_ds_bytes)
        wsb = lib.cadet_attn_workspace_bytes(C.byref(self.acfg), n_chunks, cfg.budget) + \
            lib.cadet_attn_bwd_ds_bytes(C.byref(self.acfg), n_chunks, cfg.budget, cfg.L_chunk)
        if self._ws is None or self._ws.numel() < wsb:
            self._ws = ops.workspace(wsb, self.dev)
        hc = L.HeadConfig(cfg.K, cfg.d_model, cfg.dh, 0)
        hwb = lib.cadet_heads_workspace_bytes(C.byref(hc), n_imp)
        if self._hws is None or self._hws.numel() < hwb:
            self._hws = ops.workspace(hwb, self.dev)
        self.logits = torch.empty(n_imp, cfg.K, dtype=torch.float32, device=self.dev)
        self.bucket = torch.empty(n_imp, dtype=torch.int32, device=self.dev)  # cadet_bucketize of the positions
        self.pre = torch.empty(n_imp, cfg.K * cfg.dh, dtype=torch.bfloat16, device=self.dev)
        self.cu_hist = torch.empty(n_hist + 1, dtype=torch.int32, device=self.dev)
        self.cu = torch.empty(n_chunks + 8, dtype=torch.int32, device=self.dev)
        self.n_out = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.n_packed = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.cu_hist2 = torch.empty(n_hist + 1, dtype=torch.int32, device=self.dev)  # the row-move pack's copy
        self.n_packed2 = torch.zeros(1, dtype=torch.int32, device=self.dev)
        if cfg.full_loss:
            ahc = L.HeadConfig(cfg.J, cfg.d_model, cfg.da, 0)
            awb = lib.cadet_heads_workspace_bytes(C.byref(ahc), n_imp)
            self._aws = ops.workspace(awb, self.dev)
            self.za = torch.empty(n_imp, cfg.J, dtype=torch.float32, device=self.dev)
            self.apre = torch.empty(n_imp, cfg.J * cfg.da, dtype=torch.bfloat16, device=self.dev)
            self.zr = torch.empty(n_imp, dtype=torch.float32, device=self.dev)
            self.dz_pair = torch.empty(n_imp, dtype=torch.float32, device=self.dev)
            self.dz_ctx = torch.empty(n_imp, cfg.K, dtype=torch.float32, device=self.dev)
            self.dz_aux = torch.empty(n_imp, cfg.J, dtype=torch.float32, device=self.dev)
            self.pair_share = torch.zeros(1, dtype=torch.float32, device=self.dev)
            self._pws = None
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
        # A13 pack (contiguous histories, src_row = NULL) and A0 chunk.  The row move (HBM-bound) runs
        # on a side stream while this stream packs the timestamps / sessions, chunks, plans and builds
        # the RoPE table (latency-bound); the first layer waits for the rows.
        cur = torch.cuda.current_stream()
        if self._pack_stream is None:
            self._pack_stream = torch.cuda.Stream(self.dev)
            self._pack_done = torch.cuda.Event()
        self._pack_stream.wait_stream(cur)
        if not cfg.embed:
            with torch.cuda.stream(self._pack_stream):
                chk(lib.cadet_pack(_vp(inp.X_hist), None, _vp(inp.lens), inp.n_hist, d, T, None, None,
                                   _vp(self.Hs[0]), None, None, _vp(self.cu_hist2), _vp(self.n_packed2),
                                   C.c_void_p(self.small_ws.data_ptr() + 512), 256,
                                   C.c_void_p(self._pack_stream.cuda_stream)))
        self._pack_done.record(self._pack_stream)
        chk(lib.cadet_pack(None, None, _vp(inp.lens), inp.n_hist, d, T, _vp(inp.t_hist), _vp(inp.s_hist), None,
                           _vp(self.t_p), _vp(self.s_p), _vp(self.cu_hist), _vp(self.n_packed), _vp(self.small_ws),
                           256, st))
        chk(lib.cadet_chunk(_vp(self.cu_hist), inp.n_hist, cfg.L_chunk, _vp(self.cu), inp.n_chunks + 8,
                            _vp(self.n_out), C.c_void_p(self.small_ws.data_ptr() + 256), st))
        if cfg.embed:  # NEXT-3: H[0] = summed embeddings of the packed tokens (contiguous histories: the packed
            # rows are the first cu_hist[n_hist] history rows; the rest of the budget is padding)
            tabs = (C.c_void_p * len(cfg.vocab))(*[e.data_ptr() for e in self.E])
            chk(lib.cadet_embed_forward(C.byref(self.ecfg), tabs, _vp(inp.ids), T,
                                        C.c_void_p(self.cu_hist.data_ptr() + 4 * inp.n_hist), _vp(self.Hs[0]),
                                        _vp(self._ews), self._ews.numel(), st))
        # context buckets k_t of the impressions from their raw positions
        bnd = (C.c_int32 * len(cfg.boundaries))(*cfg.boundaries)
        chk(lib.cadet_bucketize(_vp(inp.position), n_imp, bnd, len(cfg.boundaries), _vp(self.bucket),
                                C.c_void_p(self.small_ws.data_ptr() + 768), st))
        b = self.batch(inp).struct()
        ws, wsn = _vp(self._ws), self._ws.numel()
        # A1: one mask plan per step, shared by every layer's forward and backward; with the layer-sized
        # workspace the plan call also builds the step's RoPE (cos, sin) table (plan_ready = 2)
        self.acfg.plan_ready = 0
        chk(lib.cadet_mask_plan(C.byref(self.acfg), C.byref(b), ws, wsn, st))
        self.acfg.plan_ready = 2
        cur.wait_event(self._pack_done)  # packed rows H[0]
        # A1-A6: residual layers  H[l+1] = H[l] + Attn(H[l])  (block mode: the pre-norm CADET block)
        for l in range(cfg.n_layers):
            self._layer_forward(l, b, ws, wsn, st, self.Hs[l + 1])
        # A7-A8: towers on impression rows + routed BCE
        hc = L.HeadConfig(cfg.K, d, cfg.dh, 0, 1)  # rows_in_ws: backward reuses the gathered rows
        hw = L.HeadWeights(self.W1.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr(), self.b2.data_ptr())
        chk(lib.cadet_heads_forward(C.byref(hc), C.byref(hw), _vp(self.Hs[-1]), _vp(inp.rows), n_imp,
                                    _vp(self.logits), _vp(self.pre), _vp(self._hws), self._hws.numel(), st))
        if cfg.full_loss:  # Eq. 10: auxiliary heads on the same impression rows
            ahc = L.HeadConfig(cfg.J, d, cfg.da, 0)
            ahw = L.HeadWeights(self.aW1.data_ptr(), self.ab1.data_ptr(), self.aw2.data_ptr(), self.ab2.data_ptr())
            chk(lib.cadet_heads_forward(C.byref(ahc), C.byref(ahw), _vp(self.Hs[-1]), _vp(inp.rows), n_imp,
                                        _vp(self.za), _vp(self.apre), _vp(self._aws), self._aws.numel(), st))
        if not backward:
            return self.logits
        # DP: the towers' gradients are all-reduced once their backward is enqueued; each
        # layer's weight gradients in four groups (W_o | W_qg, W_kg | W_q, W_k, W_v | W_xg), each as soon
        # as cadet_attn_backward_ev's event for that group fires, overlapping the rest of the backward
        nl = cfg.n_layers
        # HSDP (NEXT-4) replaces the overlapped gradient all-reduces by one reduce-scatter after the backward
        hsdp = group is not None and cfg.optimizer == "adamw" and cfg.shard
        dp = None if hsdp else group
        buckets = GradBuckets([self.grads[self._tower_off:self._embed_off]] +
                              ([self.grads[self._embed_off:]] if cfg.embed else []), dp)
        if dp is not None and self._grad_events is None:
            self._side = torch.cuda.Stream(self.dev)
            self._grad_events = [[torch.cuda.Event() for _ in range(6)] for _ in range(nl)]
            for evs in self._grad_events:
                for e in evs:
                    e.record()  # materialises the cudaEvent_t handle
        hg = L.HeadGrads(self.gW1.data_ptr(), self.gb1.data_ptr(), self.gw2.data_ptr(), self.gb2.data_ptr())
        if not cfg.full_loss:  # Eq. 9: routed BCE, fused
            chk(lib.cadet_heads_loss_backward(C.byref(hc), C.byref(hw), _vp(self.Hs[-1]), _vp(inp.rows), n_imp, T,
                                              _vp(self.logits), _vp(self.pre), _vp(self.bucket), _vp(inp.label),
                                              _vp(self.loss), _vp(self.dHs[-1]), C.byref(hg), _vp(self._hws),
                                              self._hws.numel(), st))
        else:
            self._full_loss_backward(inp, group, hc, hw, hg, st)
        buckets.launch(0)
        handles = []
        # A9-A12: layers backward; dX_l = dX_{l+1} (residual) + Attn_l^T(dX_{l+1})
        for l in reversed(range(cfg.n_layers)):
            if cfg.recompute:  # refill the single saved buffer with layer l's activations (deterministic fwd)
                self._layer_forward(l, b, ws, wsn, st, self._rec_y)
            evs = self._grad_events[l] if dp is not None else None

            def reduce(ev, sl):
                self._side.wait_event(ev)
                with torch.cuda.stream(self._side):
                    handles.append(torch.distributed.all_reduce(sl, group=group, async_op=True))
            self._layer_backward(l, b, ws, wsn, st, evs, reduce)
        if cfg.embed:  # NEXT-3: the embedding tables' gradients from dH[0] (deterministic scatter-add)
            dts = (C.c_void_p * len(cfg.vocab))(*[g.data_ptr() for g in self.dE])
            chk(lib.cadet_embed_backward(C.byref(self.ecfg), _vp(inp.ids), T,
                                         C.c_void_p(self.cu_hist.data_ptr() + 4 * inp.n_hist), _vp(self.dHs[0]), dts,
                                         _vp(self._ews), self._ews.numel(), st))
            buckets.launch(1)
        buckets.wait()
        for h in handles:
            h.wait()
        if cfg.optimizer == "adamw":
            self.optimizer_step(group if hsdp else None)
        if group is not None:
            torch.distributed.all_reduce(self.loss, group=group)
        return self.loss

    # -------------------------------------------------------------- NEXT-4: optimizer step (HSDP)
    def optimizer_step(self, group=None):
        """AdamW (R35) on the flat fp32 master parameters.  With `group` (HSDP within the node): the
        gradients are reduce-scattered (SUM, R15) so each rank holds the reduced gradient of its shard,
        AdamW updates that shard of the fp32 master and moments and writes its bf16 copy, and the bf16
        parameters are all-gathered; the fp32-consumed vectors are widened from that bf16 copy.
        Without `group` the (already reduced) full buffer is updated on every rank."""
        cfg = self.cfg
        world = torch.distributed.get_world_size(group) if group is not None else 1
        rank = torch.distributed.get_rank(group) if group is not None else 0
        n = self.n_grad
        lo, hi = shard_range(n, world, rank)
        if self._opt is None or self._opt["world"] != world:
            full = ops.bf16_to_f32(self.wbf)               # matrices: the bf16 values are exact in fp32
            for off, sz, kind in self._slices:
                if kind == "v":
                    full[off:off + sz].copy_(self.wf32[off:off + sz])
            self._opt = dict(world=world, step=0, master=full[lo:hi].clone(),
                             m=torch.zeros(hi - lo, dtype=torch.float32, device=self.dev),
                             v=torch.zeros(hi - lo, dtype=torch.float32, device=self.dev),
                             g=torch.empty(hi - lo, dtype=torch.float32, device=self.dev) if world > 1 else None,
                             cfg=ops.adamw_config(lr=cfg.lr, weight_decay=cfg.weight_decay))
        o = self._opt
        o["step"] += 1
        if world > 1:
            torch.distributed.reduce_scatter_tensor(o["g"], self.grads, group=group)
            g = o["g"]
        else:
            g = self.grads
        ops.adamw_step(o["cfg"], o["step"], g, o["master"], o["m"], o["v"], self.wbf[lo:hi])
        if world > 1:
            torch.distributed.all_gather_into_tensor(self.wbf, self.wbf[lo:hi], group=group)
        ops.bf16_to_f32(self.wbf, self.wf32)

    def capture(self, inp: StepInputs, group=None, host_inp: StepInputs | None = None, loss_h=None):
        """CUDA graph of one whole step: every libcadet launch (and, with host_inp / loss_h, the H2D
        copy of the step's inputs from pinned memory and the D2H of the loss) becomes a graph node,
        replayed with no host work.  Kernel arguments, TMA descriptors included, are copied into
        the nodes at capture, so replays see the same buffers; call step() once first so that
        every buffer is sized."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            if host_inp is not None:
                inp.copy_(host_inp)
            self.step(inp, group)
            if loss_h is not None:
                loss_h.copy_(self.loss, non_blocking=True)
        return g

    def _saved(self, l: int) -> torch.Tensor:
        return self.saved[0 if self.cfg.recompute else l]

    def _layer_forward(self, l, b, ws, wsn, st, Y):
        """Layer l forward into Y: H + Attn(H) (A1-A6), or with cfg.block the pre-norm CADET block
        (S:644): Xn = RMSNorm1(X); H = X + Attn(Xn); Hn = RMSNorm2(H); Y = H + FFN(Hn)."""
        cfg, lib, chk = self.cfg, L.lib(), L.check
        d, T = cfg.d_model, cfg.budget
        w = L.AttnWeights(*[x.data_ptr() for x in self.W[l]])
        X = self.Hs[l]
        if not cfg.block:
            chk(lib.cadet_attn_forward(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(X), _vp(Y), _vp(X),
                                       _vp(self._saved(l)), ws, wsn, st))
            return
        k = self.blk[0 if cfg.recompute else l]
        g1, g2 = self.gam[l]
        chk(lib.cadet_rmsnorm_forward(_vp(X), _vp(g1), T, d, _vp(k["Xn"]), _vp(k["r1"]), st))
        chk(lib.cadet_attn_forward(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(k["Xn"]), _vp(k["H"]), _vp(X),
                                   _vp(self._saved(l)), ws, wsn, st))
        chk(lib.cadet_rmsnorm_forward(_vp(k["H"]), _vp(g2), T, d, _vp(k["Hn"]), _vp(k["r2"]), st))
        chk(lib.cadet_ffn_forward(_vp(k["Hn"]), _vp(self.F[l][0]), _vp(self.F[l][1]), _vp(k["H"]), T, d,
                                  cfg.ffn_mult, _vp(Y), _vp(k["U"]), _vp(k["G"]), st))

    def _layer_backward(self, l, b, ws, wsn, st, evs, reduce):
        """dHs[l] from dHs[l+1] (the residual adds included) and layer l's weight gradients; with DP
        (evs not None) each gradient group is handed to `reduce(event, slice)` as soon as it is final."""
        cfg, lib, chk = self.cfg, L.lib(), L.check
        d, T = cfg.d_model, cfg.budget
        w = L.AttnWeights(*[x.data_ptr() for x in self.W[l]])
        g = L.AttnGrads(*[x.data_ptr() for x in self.gW[l]])
        arr = (C.c_void_p * 4)(*[e.cuda_event for e in evs[:4]]) if evs else None
        dY, dX = self.dHs[l + 1], self.dHs[l]
        grp = self._groups[l]
        if not cfg.block:
            chk(lib.cadet_attn_backward_ev(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(self.Hs[l]),
                                           _vp(self._saved(l)), _vp(dY), _vp(dX), _vp(dY), C.byref(g), ws, wsn, st,
                                           arr))
            if evs:
                for i, sl in enumerate(grp["attn"]):
                    reduce(evs[i], sl)
            return
        k = self.blk[0 if cfg.recompute else l]
        g1, g2 = self.gam[l]
        dW1f, dW2f, dg2, dg1 = self.gF[l]
        dA, dB = self._dA, self._dB
        # FFN^T: dHn = dU W1^T (dA);  RMSNorm2^T + residual: dH = dY + RMSNorm2^T(dHn) (dB)
        chk(lib.cadet_ffn_backward(_vp(k["Hn"]), _vp(self.F[l][0]), _vp(self.F[l][1]), _vp(k["U"]), _vp(k["G"]),
                                   _vp(dY), None, T, d, cfg.ffn_mult, _vp(dA), _vp(dW1f), _vp(dW2f), _vp(self._fws),
                                   self._fws.numel(), st))
        chk(lib.cadet_rmsnorm_backward(_vp(k["H"]), _vp(g2), _vp(k["r2"]), _vp(dA), _vp(dY), T, d, _vp(dB), _vp(dg2),
                                       st))
        if evs:
            evs[4].record()
            reduce(evs[4], grp["ffn"])
        # Attn^T: dXn (dA);  RMSNorm1^T + residual: dX = dH + RMSNorm1^T(dXn)
        chk(lib.cadet_attn_backward_ev(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(k["Xn"]), _vp(self._saved(l)),
                                       _vp(dB), _vp(dA), None, C.byref(g), ws, wsn, st, arr))
        if evs:
            for i, sl in enumerate(grp["attn"]):
                reduce(evs[i], sl)
        chk(lib.cadet_rmsnorm_backward(_vp(self.Hs[l]), _vp(g1), _vp(k["r1"]), _vp(dA), _vp(dB), T, d, _vp(dX),
                                       _vp(dg1), st))
        if evs:
            evs[5].record()
            reduce(evs[5], grp["g1"])

    def _full_loss_backward(self, inp, group, hc, hw, hg, st):
        """NEXT-2 (Eqs. 10-12): routed logits -> (DP) all-gather with labels -> RankNet share of this
        rank -> Eq. 11 logit gradients -> tower and aux-head backward (dH accumulated).  The ranks'
        loss totals sum (all-reduced with the gradients) to the global Eq. 11 loss."""
        cfg, lib, chk = self.cfg, L.lib(), L.check
        d, T, n = cfg.d_model, cfg.budget, inp.rows.numel()
        chk(lib.cadet_routed_logits(_vp(self.logits), cfg.K, _vp(self.bucket), n, _vp(self.zr), st))
        z_all, y_all = dp_gather_scores(self.zr, inp.label, group)
        n_all = int(z_all.numel())
        pwb = lib.cadet_pairwise_workspace_bytes(n, n_all)
        if self._pws is None or self._pws.numel() < pwb:
            self._pws = ops.workspace(pwb, self.dev)
        chk(lib.cadet_pairwise_loss(_vp(self.zr), _vp(inp.label), n, _vp(z_all), _vp(y_all), n_all,
                                    _vp(self.pair_share), _vp(self.dz_pair), _vp(self._pws), self._pws.numel(), st))
        chk(lib.cadet_full_loss_grads(C.byref(self.lcfg), _vp(self.logits), cfg.K, _vp(self.bucket), _vp(inp.label),
                                      _vp(self.dz_pair), _vp(self.pair_share), _vp(self.za), _vp(inp.aux_label), n,
                                      _vp(self.losses), _vp(self.dz_ctx), _vp(self.dz_aux), st))
        chk(lib.cadet_heads_backward(C.byref(hc), C.byref(hw), _vp(self.Hs[-1]), _vp(inp.rows), n, T, _vp(self.pre),
                                     _vp(self.dz_ctx), 0, _vp(self.dHs[-1]), C.byref(hg), _vp(self._hws),
                                     self._hws.numel(), st))
        ahc = L.HeadConfig(cfg.J, d, cfg.da, 0, 1)
        ahw = L.HeadWeights(self.aW1.data_ptr(), self.ab1.data_ptr(), self.aw2.data_ptr(), self.ab2.data_ptr())
        ahg = L.HeadGrads(self.agW1.data_ptr(), self.agb1.data_ptr(), self.agw2.data_ptr(), self.agb2.data_ptr())
        chk(lib.cadet_heads_backward(C.byref(ahc), C.byref(ahw), _vp(self.Hs[-1]), _vp(inp.rows), n, T,
                                     _vp(self.apre), _vp(self.dz_aux), 1, _vp(self.dHs[-1]), C.byref(ahg),
                                     _vp(self._aws), self._aws.numel(), st))
        self.loss.copy_(self.losses[cfg.J + 2:cfg.J + 3])

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
        ops.poll(self.small_ws[512:])      # row-move pack error word
        ops.poll(self.small_ws[768:])      # bucketize error word (positions < 1)
        if self.cfg.embed:
            ops.poll(self._ews)              # embedding ids out of range


# ------------------------------------------------------------------ NEXT-1: serving
class ServingGraph:
    """Latency path for the paper's serving shape: a request = ONE packed sequence
    of n_ctx context tokens followed by n_cand candidates (context causal with Delta = 0, candidates
    see the context and themselves), scored by L gated layers + the K towers on the
    candidate rows (all towers in one pass).  The whole forward -- mask plan, every layer and
    the towers -- is captured ONCE as a CUDA graph over static buffers; a request copies its features
    and timestamps into those buffers and replays the graph (no per-kernel host launches).  The
    paper's kernel "integrates with torch.compile"; a CUDA graph is the B200-native
    equivalent here (no tracing compiler)."""

    def __init__(self, d_model: int, n_heads: int, n_ctx: int, n_cand: int, n_layers: int = 1, K: int = 2,
                 seed: int = 0, device="cuda"):
        from synth import generator as G
        self.dev = torch.device(device)
        self.d, self.H, self.L, self.K = d_model, n_heads, n_layers, K
        self.T = T = n_ctx + n_cand
        self.n_cand = n_cand
        lib = L.lib()
        self.acfg = ops.config(d_model, n_heads, delta_delay_ms=0, delta_cand_ms=0)
        mk = lambda a, dt: torch.tensor(np.asarray(a), dtype=dt, device=self.dev)
        self.cu = mk([0, T], torch.int32)
        self.ncand = mk([n_cand], torch.int32)
        self.t = torch.zeros(T, dtype=torch.int64, device=self.dev)
        self.X = torch.zeros(T, d_model, dtype=torch.bfloat16, device=self.dev)
        self.rows = mk(np.arange(n_ctx, T), torch.int32)
        self.W = [[mk(w, torch.float32).to(torch.bfloat16) for w in G.layer_weights(seed, l, d_model).as_list()]
                  for l in range(n_layers)]
        dh = d_model // 2
        hw = G.head_weights(seed, K, d_model, dh)
        self.W1 = mk(np.concatenate([hw.W1[k] for k in range(K)], axis=1), torch.float32).to(torch.bfloat16)
        self.b1, self.w2, self.b2 = (mk(x.reshape(-1), torch.float32) for x in (hw.b1, hw.w2, hw.b2))
        self.hc = L.HeadConfig(K, d_model, dh, 0)
        self.Hs = [self.X] + [torch.zeros(T, d_model, dtype=torch.bfloat16, device=self.dev) for _ in range(n_layers)]
        self.saved = torch.empty(lib.cadet_attn_saved_bytes(C.byref(self.acfg), T), dtype=torch.uint8,
                                 device=self.dev)
        self.ws = ops.workspace(lib.cadet_attn_workspace_bytes(C.byref(self.acfg), 1, T), self.dev)
        self.hws = ops.workspace(lib.cadet_heads_workspace_bytes(C.byref(self.hc), n_cand), self.dev)
        self.logits = torch.empty(n_cand, K, dtype=torch.float32, device=self.dev)
        self.pre = torch.empty(n_cand, K * dh, dtype=torch.bfloat16, device=self.dev)
        self.graph = None

    def _batch(self):
        return ops.PackedBatch(cu_seqlens=self.cu, timestamps_ms=self.t, total_tokens=self.T, max_seqlen=self.T,
                               n_candidates=self.ncand).struct()

    def forward(self):
        """The eager forward on the static buffers (what the graph replays): plan, layers, towers."""
        lib, chk = L.lib(), L.check
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        b = self._batch()
        self.acfg.plan_ready = 0
        chk(lib.cadet_mask_plan(C.byref(self.acfg), C.byref(b), _vp(self.ws), self.ws.numel(), st))
        self.acfg.plan_ready = 1
        for l in range(self.L):
            w = L.AttnWeights(*[x.data_ptr() for x in self.W[l]])
            chk(lib.cadet_attn_forward(C.byref(self.acfg), C.byref(b), C.byref(w), _vp(self.Hs[l]),
                                       _vp(self.Hs[l + 1]), _vp(self.Hs[l]), _vp(self.saved), _vp(self.ws),
                                       self.ws.numel(), st))
        hw = L.HeadWeights(self.W1.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr(), self.b2.data_ptr())
        chk(lib.cadet_heads_forward(C.byref(self.hc), C.byref(hw), _vp(self.Hs[-1]), _vp(self.rows), self.n_cand,
                                    _vp(self.logits), _vp(self.pre), _vp(self.hws), self.hws.numel(), st))
        return self.logits

    def capture(self):
        self.forward()  # sizes, one-time attributes, TMA descriptors warm
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.forward()
        return self.graph

    def score(self, X: torch.Tensor, t_ms: torch.Tensor) -> torch.Tensor:
        """One request: features [T, d] bf16 and timestamps [T] int64 (context then candidates) ->
        candidate logits [n_cand, K] (the graph's static output buffer)."""
        self.X.copy_(X, non_blocking=True)
        self.t.copy_(t_ms, non_blocking=True)
        if self.graph is None:
            return self.forward()
        self.graph.replay()
        return self.logits
