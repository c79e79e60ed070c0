"""Profiling-build experiment: per-phase clock64 sums of the dK/dV backward kernel (C4 batch)."""
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
    subprocess.check_call(["nvcc", *B.FLAGS, "-DCADET_PHASE_TIMING", *os.environ.get("PHASE_FLAGS", "").split(), "-c", src, "-o", obj])
    objs.append(obj)
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", lib_dbg, "-lcudart"])
from paper_2602_11410_b200 import _lib  # noqa: E402
_lib.LIB_PATH = lib_dbg
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2602_11410_b200.model import CadetStack, StackConfig  # noqa: E402

wl = bench.WORKLOADS["c4"]
users, hinp = bench.build_inputs(wl, 0, pin=False)
inp = hinp.to("cuda")
st = CadetStack(StackConfig(d_model=1024, n_heads=8, n_layers=1, budget=65536, L_chunk=2048), device="cuda")
st.step(inp)
torch.cuda.synchronize()
L = _lib.lib()
L.cadet_debug_phase_reset()
L.cadet_debug_phase_reset_fwd()
L.cadet_debug_tl_reset()
st.step(inp)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8192 * 16))()
L.cadet_debug_phase_read(buf, 8192 * 16)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 16).astype(np.float64)
used = a[a.sum(1) > 0]
names = ["mma: kv wait", "mma: acc_free wait", "mma: pds wait", "mma: issue", "cmp x2: mma_done wait",
         "cmp x2: dK/dV drain", "cmp x2: vec+sdp wait", "cmp x2: dS store+loop", "cmp x2: ldtm", "cmp x2: math",
         "cmp x2: sttm+arrive", "mma: q/dO wait", "-", "-", "-", "-"]
print("CTAs", len(used))
for i, n in enumerate(names):
    print(f"{n:22s} mean per CTA {used[:, i].mean():12.0f} clk")

buf16 = (C.c_ulonglong * (8192 * 16))()
L.cadet_debug_phase_read_fwd(buf16, 8192 * 16)
a = np.frombuffer(buf16, dtype=np.uint64).reshape(8192, 16).astype(np.float64)
used = a[a.sum(1) > 0]
names = ["mma: item wait", "mma: k/q wait", "mma: p_full wait", "mma: o_free/v wait", "mma: issue+other",
         "smx0: s_full wait", "smx0: (rest)", "smx0: item wait+decode", "smx0: ldtm", "smx0: mask+max",
         "smx0: exp+sttm", "smx0: rescale+arrive", "smx0: o_full wait", "smx0: drain+store", "-", "-"]
if os.environ.get("CADET_FWD_PAIRED") != "1":
    names = ["mma: q wait", "mma: k_full wait", "mma: S issue+p_full wait", "mma: v_full wait", "smx: s_full wait",
             "smx: pass1", "smx: rescale+pass2+arrive", "-"]
print("FWD CTAs", len(used))
for i, n in enumerate(names):
    print(f"{n:26s} mean per CTA {used[:, i].mean():12.0f} clk")

# dK/dV timeline of CTA 7: (code, index, clock); codes 1/2 issue S+dP(hh+1) start/end, 3 pds_ready(hh) seen,
# 4 dV/dK(hh) issued; 10+g sdp seen by group g, 12+g arrive, 14+g dS stores done
tl = (C.c_ulonglong * (4 * 4096))()
L.cadet_debug_tl_read(tl, 4 * 4096)
t = np.frombuffer(tl, dtype=np.uint64).copy()
t = t[t > 0]
clk = (t >> 16).astype(np.int64)
code = ((t >> 10) & 63).astype(np.int64)
idx = (t & 1023).astype(np.int64)
o = np.argsort(clk)
clk, code, idx = clk[o], code[o], idx[o]
print("timeline events", len(t))
for c, k, i in list(zip(clk - clk[0], code, idx))[:200]:
    print(f"{c:9d}  {k:3d}  {i}")
