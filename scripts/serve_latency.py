#!/usr/bin/env python
"""NEXT-1: the paper's serving benchmark shape on one B200 — ONE request of 4,096
context tokens + 512 candidates (context causal with Delta = 0, candidates see the context and
themselves: P:533-546), forward only.  Reports the attention-core latency (the quantity the paper
gives for A100: 792 us fmha -> 262 us custom kernel) and the full gated-layer forward
latency, device time from CUDA events over repeated calls with the plan built once.  Inputs are
synthetic (seeded); prints one JSON line."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_11410_b200 import _lib as L  # noqa: E402
from paper_2602_11410_b200 import build, ops  # noqa: E402
from synth import generator as G  # noqa: E402


def request(n_ctx=4096, n_cand=512, seed=0):
    rng = np.random.default_rng(seed)
    T = n_ctx + n_cand
    t_ctx = np.cumsum(rng.integers(1, 600_000, size=n_ctx)).astype(np.int64) + 1_700_000_000_000
    t = np.concatenate([t_ctx, np.full(n_cand, t_ctx[-1] + 1, np.int64)])
    cu = np.array([0, T], np.int32)
    return cu, t, np.zeros(T, np.int32), np.array([n_cand], np.int32), T


def time_calls(fn, iters=200, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / iters  # us


def main():
    build.build(verbose=False)
    lib = L.lib()
    cu, t, s, nc, T = request()
    dev = "cuda"
    out = {"workload": "NEXT-1: one request, 4096 context + 512 candidates, fwd only",
           "paper_A100_us": {"fmha_baseline": 792, "custom_kernel": 262}, "results": []}
    for d, H in ((352, 4), (1024, 8)):
        hd = d // H
        b = ops.PackedBatch(cu_seqlens=torch.tensor(cu, device=dev), timestamps_ms=torch.tensor(t, device=dev),
                            total_tokens=T, max_seqlen=T, session_ids=torch.tensor(s, device=dev),
                            n_candidates=torch.tensor(nc, device=dev))
        cfg = ops.config(d, H, delta_delay_ms=0, delta_cand_ms=0)
        g = torch.Generator(device="cpu").manual_seed(1)
        Qr, Kr, V = [(torch.randn(T, d, generator=g) * 0.5).to(torch.bfloat16).to(dev) for _ in range(3)]
        ws = ops.workspace(lib.cadet_attn_workspace_bytes(C.byref(cfg), 1, T))
        ops.mask_plan(cfg, b, ws)
        cfg.plan_ready = 1
        O = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(H, T, dtype=torch.float32, device=dev)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        bs = b.struct()

        def core():
            L.check(lib.cadet_attn_core_forward(C.byref(cfg), C.byref(bs), C.c_void_p(Qr.data_ptr()),
                                                C.c_void_p(Kr.data_ptr()), C.c_void_p(V.data_ptr()),
                                                C.c_void_p(O.data_ptr()), C.c_void_p(lse.data_ptr()),
                                                C.c_void_p(ws.data_ptr()), ws.numel(), st))
        core_us = time_calls(core)
        # full gated layer forward (A2-A6) for the request
        W = [torch.tensor(w).to(torch.bfloat16).to(dev) for w in G.layer_weights(0, 0, d).as_list()]
        w = L.AttnWeights(*[x.data_ptr() for x in W])
        X = (torch.randn(T, d, generator=g)).to(torch.bfloat16).to(dev)
        Y = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        saved = torch.empty(lib.cadet_attn_saved_bytes(C.byref(cfg), T), dtype=torch.uint8, device=dev)
        cfg.plan_ready = 0
        ops.mask_plan(cfg, b, ws)
        cfg.plan_ready = 2

        def layer():
            L.check(lib.cadet_attn_forward(C.byref(cfg), C.byref(bs), C.byref(w), C.c_void_p(X.data_ptr()),
                                           C.c_void_p(Y.data_ptr()), None, C.c_void_p(saved.data_ptr()),
                                           C.c_void_p(ws.data_ptr()), ws.numel(), st))
        layer_us = time_calls(layer, iters=100)
        pairs = (4096 * 4097) // 2 + 512 * 4097  # L(L+1)/2 + N(L+1) (SURVEY: exact allowed pairs)
        flops = 4.0 * hd * H * pairs
        ops.poll(ws)
        # the whole request (plan + layer + towers on the 512 candidates): eager launches vs the CUDA graph
        # (model.ServingGraph), device time per request and host wall time per request (synchronised)
        from paper_2602_11410_b200.model import ServingGraph
        import time
        sg = ServingGraph(d, H, 4096, 512, n_layers=1)
        Xr = (torch.randn(T, d, generator=g)).to(torch.bfloat16).to(dev)
        tr = torch.tensor(t, device=dev)
        eager_us = time_calls(lambda: sg.score(Xr, tr), iters=100)
        sg.capture()
        graph_us = time_calls(lambda: sg.score(Xr, tr), iters=200)

        def wall(n=200):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(n):
                sg.score(Xr, tr)
                torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e6 / n
        graph_wall = wall()
        sg.graph = None
        eager_wall = wall(100)
        ops.poll(sg.ws)
        out["results"].append({"d_model": d, "heads": H, "head_dim": hd, "attn_core_us": core_us,
                               "attn_core_tflops_on_allowed_pairs": flops / (core_us * 1e-6) / 1e12,
                               "layer_fwd_us": layer_us, "allowed_pairs_per_head": pairs,
                               "request_eager_device_us": eager_us, "request_graph_device_us": graph_us,
                               "request_eager_wall_us": eager_wall, "request_graph_wall_us": graph_wall,
                               "request": "plan + 1 gated layer + K=2 towers on 512 candidates"})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
