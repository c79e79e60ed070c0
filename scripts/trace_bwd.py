"""Profiling-build experiment: per-CTA timelines of the two backward attention kernels (C4)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_11410_b200 import build as B  # noqa: E402

lib_dbg = os.path.join(B.HERE, "libcadet_dbg.so")
objs = []
for src in B.sources():
    obj = os.path.join(B.HERE, "build", os.path.basename(src) + ".dbg.o")
    subprocess.check_call(["nvcc", *B.FLAGS, "-DCADET_PHASE_TIMING", "-c", src, "-o", obj])
    objs.append(obj)
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", lib_dbg,
                       "-lcudart"])
from paper_2602_11410_b200 import _lib  # noqa: E402
_lib.LIB_PATH = lib_dbg
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_11410_b200.model import CadetStack, StackConfig  # noqa: E402

wl = bench.WORKLOADS["c4"]
users, hinp = bench.build_inputs(wl, 0, pin=False)
inp = hinp.to("cuda")
st = CadetStack(StackConfig(d_model=1024, n_heads=8, n_layers=1, budget=65536, L_chunk=2048), device="cuda")
for _ in range(3):
    st.step(inp)
torch.cuda.synchronize()
L = _lib.lib()
buf = (C.c_ulonglong * (8192 * 12))()
L.cadet_debug_trace_read(buf, 8192 * 12)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 2, 6).astype(np.float64)
for k, name in enumerate(["dq", "dkv"]):
    t = a[:, k, :]
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    ent, first, done, ext, sm, n = [t[:, i] for i in range(6)]
    span = ext.max() - t0
    print(f"== {name}: CTAs {len(t)}  span {span / 1e3:.1f} us  mean n {n.mean():.2f}")
    print(f"  setup (entry->first MMA result) mean {np.mean(first - ent) / 1e3:.2f} us")
    print(f"  loop  (first->all MMAs done)    mean {np.mean(done - first) / 1e3:.2f} us "
          f" per item {np.sum(done - first) / max(n.sum(), 1) / 1e3:.3f} us")
    print(f"  epilogue (done->exit)           mean {np.mean(ext - done) / 1e3:.2f} us")
    busy = np.zeros(148)
    gaps = []
    for s in range(148):
        m = sm == s
        if not m.any():
            continue
        e, x = ent[m], ext[m]
        o = np.argsort(e)
        e, x = e[o], x[o]
        busy[s] = np.sum(x - e)
        gaps += list(e[1:] - x[:-1])
    print(f"  SM busy frac mean {busy.mean() / span:.3f}  min {busy.min() / span:.3f}  "
          f"inter-CTA gap mean {np.mean(gaps) / 1e3:.2f} us  CTAs/SM {len(t) / 148:.1f}")
    last = np.sort(ext - t0)[-148:]
    print(f"  tail: last-SM-finish spread {(last[-1] - last[0]) / 1e3:.1f} us")
buf2 = (C.c_ulonglong * (8192 * 8))()
L.cadet_debug_phase_reset()
st.step(inp)
torch.cuda.synchronize()
L.cadet_debug_phase_read(buf2, 8192 * 8)
ph = np.frombuffer(buf2, dtype=np.uint64).reshape(8192, 8).astype(np.float64)
used = ph[ph.sum(1) > 0]
items = a[:, 1, 5][a[:, 1, 0] > 0].sum()
names = ["cmp: vec st+bar", "cmp: sdp wait", "cmp: tmem ld", "cmp: math+st", "cmp: st_wait+arrive+loop",
         "mma: issue sdp", "mma: pds wait", "mma: dVdK issue"]
for i, nm in enumerate(names):
    print(f"{nm:26s} per item {used[:, i].sum() / items:10.0f} clk")
