"""Micro-benchmark of the NEXT-3 RMSNorm kernels at the C4 shape (T = 65536, d = 1024): CUDA-event
time per launch and achieved HBM GB/s against the algorithmic bytes (fwd 4d + 4 B per row, bwd with
dresid 8d B per row)."""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2602_11410_b200 import ops  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    out = {}
    for T, d in ((65536, 1024), (65536, 352)):
        X = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        dY = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        dR = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        g = torch.ones(d, device="cuda")
        Y, r = ops.rmsnorm_forward(X, g)
        dX, dg = ops.rmsnorm_backward(X, g, r, dY, dresid=dR)
        tf = timeit(lambda: ops.rmsnorm_forward(X, g, Y, r))
        tb = timeit(lambda: ops.rmsnorm_backward(X, g, r, dY, dresid=dR, dX=dX, dgamma=dg))
        bf, bb = T * (4 * d + 4), T * (8 * d + 4)
        out[f"T{T}_d{d}"] = {"fwd_us": tf * 1e3, "fwd_GBs": bf / tf / 1e6, "bwd_us": tb * 1e3, "bwd_GBs": bb / tb / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
