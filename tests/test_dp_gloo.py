"""Multi-rank (N > 1) host logic on CPU with 2 gloo ranks: sharding whole sequences across ranks
and SUM-all-reducing the flat gradient buffer (model.dp_reduce) equals the gradient of the union
batch (Eq. 9 is a sum, R15).  Gradients come from the fp64 oracle."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _case():
    from oracle import cadet_oracle as O
    from synth import generator as G
    lens = [13, 9, 1, 11, 6, 7]
    b = G.fixed_lengths_batch(lens, seed=4, cfg=G.stress_config())
    cu = np.concatenate([[0], np.cumsum(b.lengths)])
    d, H = 8, 2
    rng = np.random.default_rng(5)
    X = rng.standard_normal((cu[-1], d))
    dY = rng.standard_normal((cu[-1], d))
    W = [rng.standard_normal((d, d)) / np.sqrt(d) for _ in range(7)]
    cfg = O.AttnConfig(d_model=d, n_heads=H, delta_delay_ms=120_000, rope_phi_min=0.5, rope_base=1e4,
                       rope_dt_max_ms=86_400_000)
    return O, b, cu, X, dY, W, cfg


def _grads(O, cu, ts, X, dY, W, cfg, seqs):
    """Oracle flat gradient (7 d x d) of the given whole sequences."""
    flat = []
    g = None
    for s in seqs:
        a, e = int(cu[s]), int(cu[s + 1])
        meta = O.SeqMeta(cu=np.array([0, e - a]), t_ms=ts[a:e], n_cand=np.zeros(1, np.int64))
        _, caches, _ = O.batch_forward(X[a:e], W, meta, cfg)
        _, gW, _ = O.batch_backward(caches, W, meta, dY[a:e], cfg)
        g = gW if g is None else [x + y for x, y in zip(g, gW)]
    return np.concatenate([x.reshape(-1) for x in g])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_11410_b200.model import GradBuckets, dp_gather_scores, dp_reduce, dp_reduce_stats
    O, b, cu, X, dY, W, cfg = _case()
    mine = [s for s in range(len(cu) - 1) if s % world == rank]     # whole sequences per rank
    g = _grads(O, cu, b.timestamps, X, dY, W, cfg, mine)
    flat = torch.tensor(g)
    loss = torch.tensor([float(len(mine))], dtype=torch.float64)
    dp_reduce(flat, loss, dist.group.WORLD)
    # the same gradient through per-layer-style async buckets (three uneven slices of one buffer)
    flat2 = torch.tensor(g)
    n = flat2.numel()
    bk = GradBuckets([flat2[2 * n // 3:], flat2[n // 3:2 * n // 3], flat2[:n // 3]], dist.group.WORLD)
    for i in range(3):
        bk.launch(i)
    bk.wait()
    # loss / impression counts, and variable-count logits + labels (rank r holds r + 2 rows)
    tot_loss, tot_imp = dp_reduce_stats(torch.tensor([1.5 * (rank + 1)]), 10 * (rank + 1), dist.group.WORLD)
    m = rank + 2
    lg = torch.arange(m * 2, dtype=torch.float32).reshape(m, 2) + 100 * rank
    lb = torch.full((m,), float(rank))
    gl, gy = dp_gather_scores(lg, lb, dist.group.WORLD)
    if rank == 0:
        q.put((flat.numpy(), float(loss.item()), flat2.numpy(), tot_loss, tot_imp, gl.numpy(), gy.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_dp_sum_allreduce_equals_union_gradient():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, loss, got2, tot_loss, tot_imp, gl, gy = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O, b, cu, X, dY, W, cfg = _case()
    ref = _grads(O, cu, b.timestamps, X, dY, W, cfg, range(len(cu) - 1))
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    assert np.abs(got2 - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    assert loss == len(cu) - 1
    assert tot_loss == pytest.approx(1.5 + 3.0) and tot_imp == 30
    exp_l = np.concatenate([np.arange(4, dtype=np.float32).reshape(2, 2),
                            np.arange(6, dtype=np.float32).reshape(3, 2) + 100])
    assert np.array_equal(gl, exp_l) and np.array_equal(gy, np.array([0, 0, 1, 1, 1], np.float32))


def test_partition_lpt_balances_under_budget():
    """SURVEY 8(e) host packer: every user placed exactly once, per-rank tokens within the budget,
    users kept in arrival order inside a rank, LPT spread (max - min load <= largest user cost)."""
    from paper_2602_11410_b200.model import chunk_lengths, partition_lpt, user_cost
    from synth import generator as G
    assert chunk_lengths(5000, 2048) == [904, 2048, 2048] and chunk_lengths(2048, 2048) == [2048]
    assert sum(chunk_lengths(8191, 2048)) == 8191
    users = G.gen_users_for_budget(3, 4 * 16384, G.GenConfig())
    lens = [u.length for u in users]
    for world in (1, 2, 3, 4):
        parts = partition_lpt(lens, world, 16384 * 4 // world + 8192, 2048, 352)
        flat = np.sort(np.concatenate(parts))
        assert np.array_equal(flat, np.arange(len(lens)))
        loads = [sum(user_cost(lens[i], 2048, 352) for i in p) for p in parts]
        assert all(sum(lens[i] for i in p) <= 16384 * 4 // world + 8192 for p in parts)
        assert all(np.all(np.diff(p) > 0) for p in parts)
        assert max(loads) - min(loads) <= max(user_cost(m, 2048, 352) for m in lens) + 1e-6
    with pytest.raises(ValueError):
        partition_lpt([10, 20, 30], 2, 25, 2048, 64)


def _hsdp_worker(rank, world, port, q):
    """NEXT-4 host logic on gloo: shard_range + reduce_scatter_tensor + the oracle's AdamW on the
    shard + all_gather_into_tensor (in place) reproduce the unsharded AdamW of the summed gradient."""
    import os
    import torch.distributed as dist
    from oracle import cadet_oracle as O
    from paper_2602_11410_b200.model import shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 64 * world * 5
    rng = np.random.default_rng(7)
    theta = rng.normal(size=n)
    grads = [rng.normal(size=n) for _ in range(world)]            # every rank's local gradient
    lo, hi = shard_range(n, world, rank)
    g_local = torch.tensor(grads[rank])
    g_shard = torch.empty(hi - lo, dtype=torch.float64)
    dist.reduce_scatter_tensor(g_shard, g_local)
    t, m, v = O.adamw_step(theta[lo:hi], np.zeros(hi - lo), np.zeros(hi - lo), g_shard.numpy(), 1, lr=1e-2)
    full = torch.zeros(n, dtype=torch.float64)
    full[lo:hi] = torch.tensor(t)
    dist.all_gather_into_tensor(full, full[lo:hi].clone())
    ref, _, _ = O.adamw_step(theta, np.zeros(n), np.zeros(n), np.sum(grads, axis=0), 1, lr=1e-2)
    q.put((rank, float(np.abs(full.numpy() - ref).max())))
    dist.destroy_process_group()


def test_hsdp_shard_update_equals_unsharded_update():
    import socket
    import torch.multiprocessing as mp
    from paper_2602_11410_b200.model import shard_range
    assert shard_range(512, 4, 2) == (256, 384)
    with pytest.raises(ValueError):
        shard_range(100, 2, 0)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hsdp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(err <= 1e-12 for _, err in res)
