#!/usr/bin/env python
"""configs[1] (C2, serving shape) throughput on one B200: 64 histories of U{448..576} tokens, the
last 64 of each are candidates (context causal with Delta = 0, candidates see the context and
themselves: P:533-546), d 512, 8 heads x 64, one gated layer forward + the K = 2 towers on the
4,096 candidate rows.  Device time from CUDA events over repeated calls (the mask plan and RoPE
table built once per batch, as a server would per request batch); synthetic seeded inputs.
Prints one JSON line."""
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
from tests.helpers import bf16_tensor, make_case, to_dev_batch  # noqa: E402


def main(iters: int = 50):
    build.build(verbose=False)
    rng = np.random.default_rng(2)
    lens = rng.integers(448, 577, size=64)
    cu, t, s, ncv, T = make_case(list(lens), n_cand=[64] * 64, seed=2, stress=False)
    d, H, K, dh = 512, 8, 2, 256
    X = G.normal_bf16(2, 1, (T, d))
    W = G.layer_weights(2, 0, d)
    cfg = ops.config(d, H, delta_delay_ms=0, delta_cand_ms=0)
    b = to_dev_batch(cu, t, s, ncv, T)
    lib = L.lib()
    Xd = bf16_tensor(X)
    Wd = [bf16_tensor(w) for w in W.as_list()]
    w = L.AttnWeights(*[x.data_ptr() for x in Wd])
    saved = torch.zeros(lib.cadet_attn_saved_bytes(C.byref(cfg), T), dtype=torch.uint8, device="cuda")
    ws = ops.workspace(lib.cadet_attn_workspace_bytes(C.byref(cfg), b.n_seqs, T))
    Y = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    rows = torch.tensor(np.concatenate([np.arange(cu[i + 1] - 64, cu[i + 1]) for i in range(64)]).astype(np.int32),
                        device="cuda")
    hw = G.head_weights(2, K, d, dh)
    W1d = bf16_tensor(np.concatenate([hw.W1[k] for k in range(K)], axis=1))
    tens = [torch.tensor(v, device="cuda") for v in (hw.b1.reshape(-1), hw.w2.reshape(-1), hw.b2)]
    hc = L.HeadConfig(K, d, dh, 0)
    hwst = L.HeadWeights(W1d.data_ptr(), tens[0].data_ptr(), tens[1].data_ptr(), tens[2].data_ptr())
    n = rows.numel()
    hws = ops.workspace(lib.cadet_heads_workspace_bytes(C.byref(hc), n))
    logits = torch.empty(n, K, dtype=torch.float32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda x: C.c_void_p(x.data_ptr())
    bs = b.struct()
    cfg.plan_ready = 0
    L.check(lib.cadet_mask_plan(C.byref(cfg), C.byref(bs), vp(ws), ws.numel(), st))  # plan + RoPE table
    cfg.plan_ready = 2

    def serve():
        L.check(lib.cadet_attn_forward(C.byref(cfg), C.byref(bs), C.byref(w), vp(Xd), vp(Y), None, vp(saved), vp(ws),
                                       ws.numel(), st))
        L.check(lib.cadet_heads_forward(C.byref(hc), C.byref(hwst), vp(Y), vp(rows), n, vp(logits), None, vp(hws),
                                        hws.numel(), st))

    for _ in range(5):
        serve()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        serve()
    e.record()
    torch.cuda.synchronize()
    ops.poll(ws)
    ops.poll(hws)
    us = a.elapsed_time(e) * 1000.0 / iters
    tokens = int(cu[-1])
    print(json.dumps({"workload": "C2 serving (configs[1]): 64 histories U{448..576}, 64 candidates each, d 512, "
                                  "8 x 64, 1 gated layer fwd + K=2 towers on 4,096 candidates",
                      "us_per_batch": us, "tokens": tokens, "tokens_per_s": tokens / (us * 1e-6),
                      "candidates_per_s": n / (us * 1e-6), "iters": iters, "plan": "built once per batch"}))


if __name__ == "__main__":
    main()
