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
    ent, ext = t[:, 0], t[:, 3]
    span = ext.max() - ent.min()
    print(f"== {name}: CTAs {len(t)}  span {span / 1e3:.1f} us  CTA time mean {np.mean(ext - ent) / 1e3:.1f} "
          f"min {np.min(ext - ent) / 1e3:.1f} max {np.max(ext - ent) / 1e3:.1f} us  "
          f"start spread {(ent.max() - ent.min()) / 1e3:.1f} us")
buf2 = (C.c_ulonglong * (8192 * 8))()
L.cadet_debug_phase_reset()
st.step(inp)
torch.cuda.synchronize()
L.cadet_debug_phase_read(buf2, 8192 * 8)
ph = np.frombuffer(buf2, dtype=np.uint64).reshape(8192, 8).astype(np.float64)
used = ph[ph.sum(1) > 0]
items = 4840  # C4 dkv work items (k-tiles x heads)
names = ["mma: kv_full wait", "mma: acc_free wait", "mma: pds wait", "mma: issue", "mma: q/dO full wait",
         "cmp: vec st+fetch+bar", "cmp: sdp wait", "cmp: math+st+arrive (+drain at item end)"]
for i, nm in enumerate(names):
    print(f"{nm:26s} per item {used[:, i].sum() / items:10.0f} clk  per CTA {used[:, i].mean() / 1.9e3:8.1f} us")
