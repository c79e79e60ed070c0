#!/usr/bin/env python
"""bench.py — CADET hot path on B200: packed attention fwd+bwd throughput (tokens/s, TFLOP/s).

One step = one pass of the whole hot path over one packed batch per rank:
pack -> chunk -> plan -> L gated attention layers forward -> towers + routed BCE -> towers and
layers backward -> (N > 1) NCCL all-reduce of the flat fp32 gradient buffer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c3|c2] [--impl ours|reference]

Rank r uses the generator batch of seed 1000*r (weak scaling: fixed per-rank budget T).  Inputs are
resident in HBM for `value`; `e2e` repeats the step through the same public API with the step's
inputs copied from pinned host memory and the loss read back inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
TRAFFIC_PROFILE = "r02c_dram_traffic.json"  # per-class DRAM bytes per launch (scripts/traffic_summary.py)
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

WORKLOADS = {
    # C4 long-history chunked path (the north-star gate config), C3 paper-shaped
    # 8-layer stack, C2 serving shape (forward only, 64 x ~512 with 64 candidates).
    "c4": dict(d_model=1024, n_heads=8, n_layers=1, budget=65536, L_chunk=2048, max_tokens=8192),
    "c3": dict(d_model=352, n_heads=4, n_layers=8, budget=65536, L_chunk=2048, max_tokens=8192),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: NVML every
    5 ms from a background thread (nvidia-smi as fallback, ~200 ms per sample)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, dev_index: int, pci_bus_id: str | None = None):
        self.dev = dev_index
        self.pci = pci_bus_id
        self.proc = None
        self.nv = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], None, set()

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self.nv, self.h = nv, h
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.running = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nv, self.h
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while self.running:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = int(get_r(h))
                for n, bit in self.BITS.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.running = False
            self.t.join(timeout=2)
            return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


# ------------------------------------------------------------------ workload
SHARDS = 8  # the largest scaling run: every N <= 8 takes its ranks' shards from the same 8-way partition


def build_inputs(wl: dict, seed: int, pin: bool, rank: int = 0, world: int = 1, J: int = 0, vocab=None):
    """One rank's batch: one global user stream of max(8, world) x budget tokens is
    partitioned by LPT (whole users, balanced on estimated cost, each shard under the budget) and
    rank r takes shard r.  Every N <= 8 therefore runs shards of equal estimated cost, so the weak
    scaling series compares like with like (N = 1 runs shard 0)."""
    from synth import generator as G
    from paper_2602_11410_b200.model import make_inputs, partition_lpt
    gcfg = G.GenConfig(max_tokens=wl["max_tokens"])
    shards = max(SHARDS, world)
    allu = G.gen_users_for_budget(seed, shards * wl["budget"], gcfg)
    while True:
        try:
            parts = partition_lpt([u.length for u in allu], shards, wl["budget"], wl["L_chunk"], wl["d_model"])
            break
        except ValueError:
            allu = allu[:-1]
    users = [allu[i] for i in parts[rank]]
    return users, make_inputs(users, wl["d_model"], wl["L_chunk"], seed + 1000 * rank, pin=pin, J=J, vocab=vocab)


def step_flops(wl: dict, tokens: int, pairs: int, n_imp: int, dh: int, K: int = 2):
    """Algorithmic FLOPs per step: attention 4 d P fwd + 8 d P bwd per layer;
    seven d x d projections 2 T_r d^2 each fwd, twice that bwd; towers 2 n K d dh fwd, 2x bwd."""
    d, nl = wl["d_model"], wl["n_layers"]
    attn_f = nl * 4.0 * d * pairs
    attn_b = nl * 8.0 * d * pairs
    gemm = nl * (14.0 + 28.0) * tokens * d * d + 6.0 * n_imp * K * d * dh
    if wl.get("block"):  # NEXT-3 FFN: two [d, m d] GEMMs, 2 T d (m d) each fwd, twice that bwd
        gemm += nl * 3.0 * 2.0 * (2.0 * tokens * d * wl.get("ffn_mult", 4) * d)
    return {"gemm": gemm, "attn_fwd": attn_f, "attn_bwd": attn_b}


# ------------------------------------------------------------------ oracle baseline (CPU)
def oracle_sample(users, wl: dict, max_tokens: int):
    """First whole chunks of the batch up to max_tokens tokens (bounded CPU sample)."""
    from synth import generator as G
    L = wl["L_chunk"]
    seqs = []
    total = 0
    for u in users:
        m = u.length
        n = -(-m // L)
        starts = [0] + [m - (n - c) * L for c in range(1, n)]
        ends = starts[1:] + [m]
        for a, e in zip(starts, ends):
            if total + (e - a) > max_tokens:
                return seqs, total
            seqs.append((u, a, e))
            total += e - a
    return seqs, total


def run_oracle_step(seqs, wl: dict, seed: int):
    """One fp64 oracle pass (layers fwd + towers loss/bwd + layers bwd) over the sample."""
    from oracle import cadet_oracle as O
    from synth import generator as G
    d, H, nl = wl["d_model"], wl["n_heads"], wl["n_layers"]
    cfg = O.AttnConfig(d_model=d, n_heads=H)
    Ws = [[w.astype(np.float64) for w in G.layer_weights(seed, l, d).as_list()] for l in range(nl)]
    blk = bool(wl.get("block"))
    if blk:  # NEXT-3: the pre-norm block (RMSNorm, attention, RMSNorm, FFN)
        bws = [G.block_weights(seed, l, d) for l in range(nl)]
        ffs = [(w.W1.astype(np.float64), w.W2.astype(np.float64)) for w in bws]
        gms = [(w.gamma1.astype(np.float64), w.gamma2.astype(np.float64)) for w in bws]
    hw = G.head_weights(seed, 2, d, d // 2)
    rng = np.random.default_rng(seed)
    loss = 0.0
    for (u, a, e) in seqs:
        t = u.timestamps[a:e]
        A = O.mask_dense(t, 0, cfg)
        X = rng.standard_normal((e - a, d))
        caches = []
        for l in range(nl):
            if blk:
                X, c = O.block_forward_seq(X, Ws[l], ffs[l], gms[l], t, A, cfg)
                caches.append((None, c))
                continue
            Y, c = O.layer_forward_seq(X, Ws[l], t, A, cfg)
            caches.append((X, c))
            X = X + Y
        rows = np.arange(0, e - a, 2)
        Lh, z, dH, g = O.heads_loss_backward(X, rows, hw.W1.astype(np.float64), hw.b1.astype(np.float64),
                                             hw.w2.astype(np.float64), hw.b2.astype(np.float64),
                                             O.bucketize(u.positions[a:e][rows], (4,)),
                                             u.labels[a:e][rows].astype(np.float64))
        loss += Lh
        dX = dH
        for l in reversed(range(nl)):
            Xl, c = caches[l]
            if blk:
                dX, _ = O.block_backward_seq(c, Ws[l], ffs[l], gms[l], t, A, dX, cfg)
                continue
            dXa, gW, _ = O.layer_backward_seq(c, Ws[l], t, A, dX, cfg)
            dX = dX + dXa
    return loss


def blas_info():
    """The BLAS the oracle's numpy runs on (threadpoolctl), e.g. openblas / mkl and its thread count."""
    try:
        from threadpoolctl import threadpool_info
        return [{k: i.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception as ex:  # noqa: BLE001
        return f"unavailable: {type(ex).__name__}"


def bind_numa_local(dev_index: int):
    """Pin this rank's host threads to the CPUs of its GPU's NUMA node (sysfs local_cpulist), so the
    pinned input buffers are first-touched on the GPU's local memory and the e2e host->device copies do
    not cross the socket interconnect.  Returns the CPU list or None (no sysfs entry: unchanged)."""
    try:
        import torch
        pp = torch.cuda.get_device_properties(dev_index)
        pci = f"{getattr(pp, 'pci_domain_id', 0):04x}:{pp.pci_bus_id:02x}:{getattr(pp, 'pci_device_id', 0):02x}.0"
        txt = open(f"/sys/bus/pci/devices/{pci}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= set(os.sched_getaffinity(0)) or cpus
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:  # noqa: BLE001
        pass
    return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def time_oracle(users, wl, seed, budget_s=15.0, max_tokens=None):
    """Time the oracle as it stands on the host cores; returns (tokens/s, tokens, seconds, desc)."""
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(cpu_cores())
    except Exception:
        ctx = None
    max_tokens = max_tokens or (24576 if wl["d_model"] >= 1024 else 8192)
    seqs, tok = oracle_sample(users, wl, max_tokens)
    t0 = time.perf_counter()
    run_oracle_step(seqs, wl, seed)
    dt = time.perf_counter() - t0
    desc = (f"first {len(seqs)} whole chunks ({tok} tokens) of the rank-0 batch, {wl['n_layers']} "
            f"{'pre-norm block(s)' if wl.get('block') else 'layer(s)'} fwd+bwd + towers, numpy fp64")
    return tok / dt, tok, dt, desc


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--recompute", action="store_true", help="gradient checkpointing (P:453-455): layers re-run fwd in bwd")
    ap.add_argument("--full-loss", action="store_true",
                    help="NEXT-2: train on Eq. 11 (towers + auxiliary heads + cross-rank RankNet) instead of Eq. 9")
    ap.add_argument("--block", action="store_true",
                    help="NEXT-3: every layer is the pre-norm CADET block (RMSNorm, gated attention, RMSNorm, FFN x4)")
    ap.add_argument("--embed", action="store_true",
                    help="NEXT-3: the step starts from token field ids (summed id + type embeddings, Eq. 1) and ends "
                         "with the embedding gradients (implied by --block: the paper's whole training step)")
    ap.add_argument("--optimizer", default="none", choices=["none", "adamw"],
                    help="NEXT-4: append the AdamW step (R35) to every training step")
    ap.add_argument("--no-shard", action="store_true",
                    help="with --optimizer and N > 1: replicated AdamW after all-reduce instead of HSDP sharding")
    ap.add_argument("--seeds", type=int, default=1,
                    help="also time the step on batches of seeds 0..S-1 (SURVEY 8(d): mean +- sd over seeds); "
                         "the headline value stays seed 0")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as one CUDA graph (measured: no gain over eager launches on C4)")
    args = ap.parse_args()
    args.embed = args.embed or args.block
    wl = dict(WORKLOADS[args.workload], block=args.block)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "packed attention fwd+bwd tokens/s and TFLOP/s (% bf16 peak) at 1/2/4/8 B200"
    workload_name = {"c4": "C4 long-history chunked path: histories <= 8192 events chunked at 2048, d 1024, "
                           "8 heads x 128, 1 gated layer + K=2 towers, fwd+bwd, T=65536/rank",
                     "c3": "C3 paper-shaped: 8 gated layers, d 352, 4 heads x 88, Lc 2048, K=2 towers, fwd+bwd, "
                           "T=65536/rank"}[args.workload]
    if args.block:
        workload_name += "; every layer the pre-norm CADET block (RMSNorm, attention, RMSNorm, FFN x4; NEXT-3)"
    if args.embed:
        workload_name += "; inputs are token field ids: summed id + type embeddings (Eq. 1; vocab 2/16384/8/4)"

    if args.impl == "reference":
        # The reference arm is the CPU oracle (no reference implementation exists): rank 0 only.
        if rank != 0:
            return
        users, _ = build_inputs(wl, 1000 * rank, pin=False)
        times, toks = [], 0
        for i in range(args.warmup + args.steps):
            v, tok, dt, desc = time_oracle(users, wl, 0, max_tokens=2048 if wl["d_model"] >= 1024 else 3072)
            if i >= args.warmup:
                times.append(dt)
                toks = tok
        ms = 1000.0 * float(np.mean(times))
        val = toks / (ms / 1000.0)
        out = {"impl": "reference", "metric": metric, "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": workload_name, "sample": desc},
               "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                                "sample": desc, "blas": blas_info()},
               "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    # keep stdout for the one JSON line: anything else written to fd 1 (NCCL's version / debug lines, other
    # native prints) goes to stderr; the JSON line is printed through a duplicate of the original stdout
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    import torch
    import torch.distributed as dist
    from paper_2602_11410_b200 import build, ops
    from paper_2602_11410_b200.model import CadetStack, StackConfig
    if local == 0:
        build.build(verbose=False)  # no-op when the shipped libcadet.so is current
    torch.cuda.set_device(local)
    # each rank's host threads and pinned inputs on its GPU's NUMA node (N = 1 too: the e2e leg's
    # host -> device copies are the limit of that leg); the CPU oracle baseline gets the full affinity back
    full_affinity = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    numa_cpus = bind_numa_local(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
        dist.barrier()  # local rank 0 finished any rebuild before the others load the library
    dev = torch.device("cuda", local)

    from paper_2602_11410_b200.model import StackConfig as _SC
    vocab = _SC().vocab if args.embed else None
    users, host_inp = build_inputs(wl, 0, pin=True, rank=rank, world=world, J=2 if args.full_loss else 0, vocab=vocab)
    inp = host_inp.to(dev)
    torch.cuda.synchronize()
    scfg = StackConfig(d_model=wl["d_model"], n_heads=wl["n_heads"], n_layers=wl["n_layers"], budget=wl["budget"],
                       L_chunk=wl["L_chunk"], full_loss=args.full_loss, recompute=args.recompute, block=args.block,
                       optimizer=args.optimizer, shard=not args.no_shard, embed=args.embed)
    stack = CadetStack(scfg, seed=0, device=dev)
    pairs = stack.pairs(inp)
    n_imp = inp.rows.numel()
    flops = step_flops(wl, inp.tokens, pairs, n_imp, scfg.dh)
    total_flops = sum(flops.values())

    def barrier():
        if group is not None:
            dist.barrier()

    # diagnostic: CADET_BENCH_NO_COLLECTIVE=1 steps without the gradient all-reduce (rank imbalance only)
    step_group = None if os.environ.get("CADET_BENCH_NO_COLLECTIVE") == "1" else group
    for _ in range(args.warmup):
        stack.step(inp, step_group)
    torch.cuda.synchronize()
    stack.poll()

    # ---------------- timed region (inputs resident in HBM)
    pp = torch.cuda.get_device_properties(local)
    pci = None
    if hasattr(pp, "pci_bus_id"):
        pci = f"{getattr(pp, 'pci_domain_id', 0):08x}:{pp.pci_bus_id:02x}:{getattr(pp, 'pci_device_id', 0):02x}.0"
    # --graph: the step as one CUDA graph; the per-class CUDA events are nodes of the graph, so after
    # the timed replays they hold the last timed step.  Eager fallback if capture fails.
    graph, graph_err = None, None
    if args.graph and args.optimizer != "none":
        graph_err = "not captured: the optimizer's bias corrections change every step"
    elif args.graph:
        try:
            ops.prof_enable(15, 64 * (wl["n_layers"] + 2))
            n0 = ops.launch_count()
            graph = stack.capture(inp, step_group)
            launches = ops.launch_count() - n0
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001
            graph, graph_err = None, f"{type(ex).__name__}: {ex}"[:200]
            torch.cuda.synchronize()
            ops.prof_read()
    clocks = ClockSampler(local, pci)
    clocks.start()
    if graph is None:
        ops.prof_enable(15, 64 * (args.steps + 1) * (wl["n_layers"] + 2))
        n0 = ops.launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            stack.step(inp, step_group)
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    if graph is None:
        launches = (ops.launch_count() - n0) // max(1, args.steps)
    prof = ops.prof_read()
    prof_steps = 1 if graph is not None else max(1, args.steps)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    tok = torch.tensor([inp.tokens], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(tok)
    tokens_all = float(tok.item())
    value = tokens_all / (ms_max / 1000.0)
    fl = torch.tensor([total_flops], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(fl)  # ranks hold different batches: sum their algorithmic FLOPs
    tflops_all = float(fl.item()) / (ms_max / 1000.0) / 1e12

    # ---------------- e2e: same step through the public API from pinned host buffers.  Every step's
    # inputs are copied host -> device inside the timed region (and its loss read back); the copy of
    # step i + 1's inputs runs on a copy stream into the second of two device buffers while step i
    # computes (a prefetching data loader), so e2e = max(copy, compute) per step in steady state.
    e2e = None
    if not args.no_e2e:
        steps = args.steps
        loss_h = torch.zeros(steps + 2, dtype=torch.float32).pin_memory()
        logits_h = torch.zeros(2, n_imp, scfg.K, dtype=torch.float32).pin_memory()  # the step's result: tower logits
        bufs = [inp, host_inp.to(dev)]
        main = torch.cuda.current_stream()
        copy_st = torch.cuda.Stream(dev)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]

        def run(n):
            copy_st.wait_stream(main)
            with torch.cuda.stream(copy_st):
                bufs[0].copy_(host_inp)
                ready[0].record(copy_st)
            for i in range(n):
                bi = i & 1
                if i + 1 < n:
                    nb = (i + 1) & 1
                    with torch.cuda.stream(copy_st):
                        if i >= 1:
                            copy_st.wait_event(free[nb])  # step i - 1 finished reading buffer nb
                        bufs[nb].copy_(host_inp)
                        ready[nb].record(copy_st)
                main.wait_event(ready[bi])
                stack.step(bufs[bi], step_group)
                free[bi].record(main)
                loss_h[i:i + 1].copy_(stack.loss, non_blocking=True)
                logits_h[i & 1].copy_(stack.logits, non_blocking=True)
        run(2)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(steps)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens_all / (float(ems.item()) / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(host_inp.nbytes()), "d2h_bytes_per_step": 4 + 4 * n_imp * scfg.K,
               "d2h": "loss + the K tower logits of every impression (the north star's output)",
               "ms_per_step": float(ems.item()),
               "pipeline": "inputs of step i+1 copied (pinned host -> HBM, copy stream) while step i computes",
               "host_numa_cpus": None if numa_cpus is None else f"{len(numa_cpus)} cpus local to the GPU"}
    stack.poll()

    # ---------------- other batches (seeds 1..S-1), each timed like seed 0 (resident inputs)
    seeds = None
    if args.seeds > 1:
        per = [(0, ms_max, inp.tokens, total_flops)]
        for sd in range(1, args.seeds):
            _, h_s = build_inputs(wl, sd, pin=False, rank=rank, world=world, J=2 if args.full_loss else 0,
                                  vocab=vocab)
            inp_s = h_s.to(dev)
            fl_s = sum(step_flops(wl, inp_s.tokens, stack.pairs(inp_s), inp_s.rows.numel(), scfg.dh).values())
            for _ in range(args.warmup):
                stack.step(inp_s, step_group)
            torch.cuda.synchronize()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(args.steps):
                stack.step(inp_s, step_group)
            a1.record()
            torch.cuda.synchronize()
            barrier()
            tt = torch.tensor([a0.elapsed_time(a1) / args.steps], dtype=torch.float64, device=dev)
            if group is not None:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            per.append((sd, float(tt.item()), inp_s.tokens, fl_s))
            stack.poll()
        msv = np.array([p_[1] for p_ in per])
        tokv = np.array([p_[2] for p_ in per]) * world / (msv / 1000.0)
        tfv = np.array([p_[3] for p_ in per]) / (msv / 1000.0) / 1e12
        seeds = {"n": len(per), "ms_per_step": {"mean": float(msv.mean()), "sd": float(msv.std(ddof=1))},
                 "tokens_per_s": {"mean": float(tokv.mean()), "sd": float(tokv.std(ddof=1))},
                 "tflops_per_gpu": {"mean": float(tfv.mean()), "sd": float(tfv.std(ddof=1))},
                 "per_seed": [{"seed": p_[0], "ms": p_[1], "tokens": p_[2]} for p_ in per]}

    if rank != 0:
        if group is not None:
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel class (live CUDA-event times)
    peaks, peak_src = load_peaks()
    per_step_ms = {k: v[0] / prof_steps for k, v in prof.items()}
    dom = max(("gemm", "attn_fwd", "attn_bwd"), key=lambda k: per_step_ms[k])
    achieved = flops[dom] / (per_step_ms[dom] / 1000.0) / 1e12 if per_step_ms[dom] > 0 else 0.0
    # Peak: the measured BURST bf16 rate for a timed region shorter than a second at full clocks with no
    # power capping (the driver's burst figure is the matmul timed alone); the SUSTAINED rate when the
    # region is long or the clocks show capping / throttling (MEASURED_PEAKS.json holds both)
    region_s = ms * args.steps / 1000.0
    # (a sw_power_cap flag with the median SM clock at max does not lower the rate; a median clock below
    # 95 % of max or a thermal / hardware slowdown does)
    hard = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(clk.get("reasons") or [])
    capped = bool(hard) or (clk.get("sm_mhz") or 0) < 0.95 * (clk.get("sm_max_mhz") or 1)
    burst = region_s < 1.0 and not capped
    peak_key = "bf16_tflops" if burst else "bf16_tflops_sustained"
    peak = float(peaks.get(peak_key, peaks.get("bf16_tflops")))
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", TRAFFIC_PROFILE)
    if os.path.exists(tpath) and args.workload == "c4":
        tj = json.load(open(tpath))
        if dom in tj:
            traffic, traffic_src = tj[dom]["dram_bytes_per_launch"], f"profiles/{TRAFFIC_PROFILE} ({tj.get('method', '')})"
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_unit": "DRAM bytes per launch",
                "traffic_source": traffic_src,
                "peak_source": f"{peak_src} {peak_key}",
                "peak_rule": (f"timed region {region_s:.3f} s, clocks median {clk.get('sm_mhz')} of {clk.get('sm_max_mhz')} "
                              f"MHz, reasons {clk.get('reasons')}: burst if < 1 s, median clock >= 95 % of max and no thermal / "
                              f"hw slowdown, else sustained"),
                "share_of_step": per_step_ms[dom] / ms, "per_class_ms_per_step": per_step_ms,
                "launches_per_step": {k: v[1] / prof_steps for k, v in prof.items()}}
    # the attention core alone (SURVEY 8(d) view 2): A5 + A10 algorithmic FLOPs on allowed pairs
    # (4 d P fwd + 8 d P bwd per layer), against the same peak; the FlashAttention convention
    # (bwd = 2.5 x fwd) printed for comparability; DRAM bytes vs the 8 d / 20 d B per token per layer
    attn_ms = per_step_ms["attn_fwd"] + per_step_ms["attn_bwd"]
    attn_fl = flops["attn_fwd"] + flops["attn_bwd"]
    attn_tf = attn_fl / (attn_ms / 1000.0) / 1e12 if attn_ms > 0 else 0.0
    attn_view = {"flops_per_step": attn_fl, "ms_per_step": attn_ms, "achieved": attn_tf, "peak": peak,
                 "unit": "TFLOP/s", "frac": attn_tf / peak,
                 "fwd": {"ms": per_step_ms["attn_fwd"], "tflops": flops["attn_fwd"] / max(per_step_ms["attn_fwd"], 1e-9) / 1e9},
                 "bwd": {"ms": per_step_ms["attn_bwd"], "tflops": flops["attn_bwd"] / max(per_step_ms["attn_bwd"], 1e-9) / 1e9},
                 "flash_attention_convention_tflops": 3.5 * flops["attn_fwd"] / (attn_ms / 1000.0) / 1e12 if attn_ms > 0 else 0.0,
                 "algorithmic_bytes_per_step": {"fwd": 8.0 * wl["d_model"] * inp.tokens * wl["n_layers"],
                                                "bwd": 20.0 * wl["d_model"] * inp.tokens * wl["n_layers"]}}
    if os.path.exists(tpath) and args.workload == "c4":
        tj = json.load(open(tpath))
        attn_view["dram_bytes_per_step"] = {k: tj[k]["dram_bytes_per_step"] for k in ("attn_fwd", "attn_bwd") if k in tj}
        attn_view["dram_source"] = f"profiles/{TRAFFIC_PROFILE}"
    cpu = None
    if not args.no_cpu and world == 1:
        if full_affinity:
            os.sched_setaffinity(0, full_affinity)
        v, tokc, dt, desc = time_oracle(users, wl, 0)
        cpu = {"value": v, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle", "sample": desc,
               "seconds": dt, "blas": blas_info()}
    out = {
        "metric": metric, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": workload_name, "tokens_real_per_rank": inp.tokens, "budget_T": wl["budget"],
                   "sequences_per_rank": inp.n_chunks, "histories_per_rank": inp.n_hist,
                   "allowed_pairs_per_head": pairs, "impressions": n_imp, "layers": wl["n_layers"],
                   "d_model": wl["d_model"], "heads": wl["n_heads"], "L_chunk": wl["L_chunk"],
                   "l2": "inputs > L2 (X 128 MB + activations > 1 GB per step); no flush needed",
                   "parallelism": f"dp{world}", "loss": "Eq. 11 full (NEXT-2)" if args.full_loss else "Eq. 9 routed BCE",
                   "recompute": bool(args.recompute),
                   "optimizer": "none (step ends at the gradients, SURVEY 8(a))" if args.optimizer == "none" else
                   ("AdamW (R35), HSDP: reduce-scatter grads, shard update, all-gather bf16 params" if
                    (world > 1 and not args.no_shard) else "AdamW (R35), replicated after the gradient all-reduce"),
                   "layer": "pre-norm CADET block: RMSNorm, gated attention, RMSNorm, FFN x4 (NEXT-3)" if args.block
                   else "gated attention layer (Eq. 3-7) + residual",
                   "partition": "rank r = shard r of an LPT partition of one user stream into 8 budgets"},
        "tflops": tflops_all, "tflops_per_gpu": tflops_all / world,
        "frac_of_peak_measured": tflops_all / world / peak, "peak_measured": {"key": peak_key, "tflops": peak},
        "frac_of_peak_spec": tflops_all / world / 2250.0,
        "flops_per_step_per_rank": flops,
        "roofline": roofline, "attention_core": attn_view, "seeds": seeds,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "cuda_graph": graph is not None, "cuda_graph_error": graph_err,
    }
    json_out.write(json.dumps(out) + "\n")
    json_out.flush()
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
