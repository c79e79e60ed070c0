"""Diagnostic (2 GPUs): sharded vs replicated AdamW after each step, per parameter slice."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import bench
    from paper_2602_11410_b200.model import CadetStack, StackConfig
    wl = dict(bench.WORKLOADS["c3"], budget=16384, n_layers=2)
    users, hinp = bench.build_inputs(wl, 0, pin=False, rank=rank, world=2)
    inp = hinp.to("cuda")
    mk = lambda shard: CadetStack(StackConfig(d_model=wl["d_model"], n_heads=wl["n_heads"], n_layers=wl["n_layers"],
                                              budget=wl["budget"], L_chunk=wl["L_chunk"], optimizer="adamw", lr=1e-3,
                                              shard=shard), seed=0, device="cuda")
    a, b = mk(True), mk(False)
    for step in range(2):
        a.step(inp, dist.group.WORLD)
        b.step(inp, dist.group.WORLD)
        torch.cuda.synchronize()
        ga, gb = a.grads.clone(), b.grads.clone()
        if rank == 0:
            wa, wb = a.wbf.float().cpu().numpy(), b.wbf.float().cpu().numpy()
            for i, (off, sz, kind) in enumerate(a._slices):
                d = np.abs(wa[off:off + sz] - wb[off:off + sz])
                print(f"step {step} slice {i} {kind} n={sz} frac_diff={np.mean(d > 0):.4f} max={d.max():.3e}")
            # grads: replicated = all-reduced full; sharded = local (not reduced) full buffer
            print("grad local(sharded) vs reduced(replicated): max", float((ga - gb).abs().max()))
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
