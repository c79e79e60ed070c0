"""Experiment: where the 3xTF32 GEMM error comes from (split vs accumulation), fp32 normal inputs."""
import ctypes as C
import numpy as np
import torch
from paper_2602_11410_b200 import _lib as L

lib = L.lib()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def tf32_rn(x):
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def tf32_tr(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def gpu(A, B, M, N, K, a_t, b_t):
    Af = torch.tensor(A.T.copy() if a_t else A).cuda()
    Bf = torch.tensor(B.T.copy() if b_t else B).cuda()
    Cf = torch.empty(M, N, device="cuda")
    wsb = lib.cadet_gemm_fp32_workspace_bytes(M, N, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    L.check(lib.cadet_gemm_fp32(M, N, K, C.c_void_p(Af.data_ptr()), a_t, C.c_void_p(Bf.data_ptr()), b_t,
                                C.c_void_p(Cf.data_ptr()), None, C.c_void_p(ws.data_ptr()), wsb, st))
    torch.cuda.synchronize()
    return Cf.cpu().numpy().astype(np.float64)


for (M, N, K) in ((256, 256, 1024), (257, 512, 1024), (256, 256, 64)):
    rng = np.random.default_rng(K + M)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    sc = np.abs(ref).max()
    ah, bh = tf32_rn(A), tf32_rn(B)
    al, bl = A - ah, B - bh
    f = lambda x: x.astype(np.float64)
    em_tr = f(ah) @ f(bh) + f(ah) @ f(tf32_tr(bl)) + f(tf32_tr(al)) @ f(bh)
    em_1 = f(ah) @ f(bh)
    em_1t = f(tf32_tr(A)) @ f(tf32_tr(B))
    print(f"{M}x{N}x{K}: emul 3x(trunc lo) {np.abs(em_tr-ref).max()/sc:.2e}  emul 1x RN {np.abs(em_1-ref).max()/sc:.2e}"
          f"  emul 1x trunc {np.abs(em_1t-ref).max()/sc:.2e}")
    for a_t in (0, 1):
        for b_t in (0, 1):
            g = gpu(A, B, M, N, K, a_t, b_t)
            print(f"   gpu a_t={a_t} b_t={b_t}: vs ref {np.abs(g-ref).max()/sc:.2e}  vs emul3x {np.abs(g-em_tr).max()/sc:.2e}"
                  f"  vs emul1x {np.abs(g-em_1).max()/sc:.2e}")
