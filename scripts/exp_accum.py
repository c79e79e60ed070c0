"""Experiment: tensor-core accumulation error vs K (bf16-exact operands) and the 3xTF32 GEMM."""
import ctypes as C
import numpy as np
import torch
from paper_2602_11410_b200 import _lib as L, ops
from synth import generator as G

lib = L.lib()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for pos in (False, True):
    for K in (64, 256, 1024, 4096):
        M, N = 256, 256
        rng = np.random.default_rng(K)
        A = G.bf16_round(rng.standard_normal((M, K)).astype(np.float32))
        B = G.bf16_round(rng.standard_normal((K, N)).astype(np.float32))
        if pos:
            A, B = np.abs(A), np.abs(B)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        Ad = torch.tensor(A).cuda().bfloat16()
        Bd = torch.tensor(B.T.copy()).cuda().bfloat16()
        Cg = ops.gemm(Ad, Bd, out_f32=True)
        e16 = np.abs(Cg.cpu().numpy() - ref) / np.abs(ref).max()
        # 3xTF32
        Af, Bf = torch.tensor(A).cuda(), torch.tensor(B).cuda()
        Cf = torch.empty(M, N, device="cuda")
        wsb = lib.cadet_gemm_fp32_workspace_bytes(M, N, K)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        L.check(lib.cadet_gemm_fp32(M, N, K, C.c_void_p(Af.data_ptr()), 0, C.c_void_p(Bf.data_ptr()), 0,
                                    C.c_void_p(Cf.data_ptr()), None, C.c_void_p(ws.data_ptr()), wsb, st))
        torch.cuda.synchronize()
        d32 = Cf.cpu().numpy() - ref
        e32 = np.abs(d32) / np.abs(ref).max()
        print(f"pos={pos} K={K}: bf16-exact GEMM max rel {e16.max():.2e} mean {e16.mean():.2e} | 3xTF32 max rel "
              f"{e32.max():.2e} mean {e32.mean():.2e} mean signed {(d32 / np.abs(ref).max()).mean():.2e}")
