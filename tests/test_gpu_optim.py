"""NEXT-4 GPU parity: the AdamW step of the HSDP training step (reading R35)
through the C ABI against oracle.adamw_step, the bf16 compute copy, the widening of fp32-consumed
parameters, and CadetStack(optimizer="adamw") updating its flat parameters from the step's own
gradients (the 2-GPU sharded-vs-replicated check is in test_gpu_dp.py)."""
import numpy as np
import pytest

from oracle import cadet_oracle as O
from synth import generator as G

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ops():
    from paper_2602_11410_b200 import build, ops as _ops
    build.build()
    return _ops


@pytest.mark.parametrize("n,wd", [(1, 0.0), (1_000_003, 0.01), (4096, 0.0)])
def test_adamw_matches_oracle_over_steps(ops, n, wd):
    rng = np.random.default_rng(n)
    p0 = rng.normal(size=n).astype(np.float32)
    cfg = ops.adamw_config(lr=1e-3, weight_decay=wd)
    p, m, v = (torch.tensor(a, device="cuda") for a in (p0, np.zeros(n, np.float32), np.zeros(n, np.float32)))
    pbf = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ref = (p0.astype(np.float64), np.zeros(n), np.zeros(n))
    mabs = np.zeros(n)  # sum of |terms| of m: the scale of its fp32 rounding (m can cancel)
    for step in range(1, 4):
        # gradients over 8 decades, including exact zeros
        g = (rng.normal(size=n) * 10.0 ** rng.uniform(-6, 2, size=n)).astype(np.float32)
        g[::97] = 0.0
        ops.adamw_step(cfg, step, torch.tensor(g, device="cuda"), p, m, v, pbf)
        # the ABI takes fp32 hyper-parameters: the oracle gets the same (fp32-rounded) values (R20)
        f = lambda x: float(np.float32(x))
        ref = O.adamw_step(*ref, g.astype(np.float64), step, lr=f(1e-3), beta1=f(0.9), beta2=f(0.999), eps=f(1e-8),
                           weight_decay=f(wd))
        mabs = 0.9 * mabs + 0.1 * np.abs(g.astype(np.float64))
    torch.cuda.synchronize()
    pg, mg, vg = (t.cpu().numpy().astype(np.float64) for t in (p, m, v))
    # fp32 arithmetic on an O(lr) update of O(1) values: a few fp32 ulps of the parameter
    assert np.abs(pg - ref[0]).max() <= 4e-7 * max(1.0, np.abs(ref[0]).max())
    assert np.all(np.abs(mg - ref[1]) <= 1e-6 * mabs + 1e-30)
    assert np.all(np.abs(vg - ref[2]) <= 1e-6 * np.abs(ref[2]) + 1e-30)
    # the compute copy is exactly the bf16 rounding of the updated master
    assert torch.equal(pbf, p.to(torch.bfloat16))


def test_bf16_to_f32_is_exact(ops):
    x = torch.randn(100_001, device="cuda").to(torch.bfloat16)
    assert torch.equal(ops.bf16_to_f32(x), x.float())


def test_stack_adamw_step_updates_flat_parameters():
    """One CadetStack step with optimizer="adamw": the fp32 master moves by the oracle's AdamW update
    of the step's own gradients, every matrix view the kernels read holds bf16(master), and every
    fp32-consumed vector holds the widened bf16 value."""
    import bench
    from paper_2602_11410_b200 import build
    from paper_2602_11410_b200.model import CadetStack, StackConfig
    build.build()
    wl = dict(bench.WORKLOADS["c3"], budget=16384, n_layers=2)
    users, hinp = bench.build_inputs(wl, 0, pin=False)
    inp = hinp.to("cuda")
    st = CadetStack(StackConfig(d_model=wl["d_model"], n_heads=wl["n_heads"], n_layers=wl["n_layers"],
                                budget=wl["budget"], L_chunk=wl["L_chunk"], optimizer="adamw", lr=1e-3,
                                weight_decay=0.01, block=True), device="cuda")
    before = st.wbf.float().cpu().numpy().astype(np.float64)
    vec_before = st.wf32.cpu().numpy().astype(np.float64)
    for off, sz, kind in st._slices:
        if kind == "v":
            before[off:off + sz] = vec_before[off:off + sz]
    W0 = st.W[0][1].float().cpu().numpy()
    st.step(inp)
    torch.cuda.synchronize()
    g = st.grads.cpu().numpy().astype(np.float64)
    f = lambda x: float(np.float32(x))
    ref, _, _ = O.adamw_step(before, np.zeros_like(before), np.zeros_like(before), g, 1, lr=f(1e-3), beta1=f(0.9),
                             beta2=f(0.999), eps=f(1e-8), weight_decay=f(0.01))
    master = st._opt["master"].cpu().numpy().astype(np.float64)
    assert np.abs(master - ref).max() <= 4e-7 * max(1.0, np.abs(ref).max())
    wbf = st.wbf.float().cpu().numpy()
    assert np.array_equal(wbf, st._opt["master"].to(torch.bfloat16).float().cpu().numpy())
    W1 = st.W[0][1].float().cpu().numpy()
    assert not np.array_equal(W0, W1)                       # the views the kernels read moved
    off, sz, _ = st._slices[1]
    assert np.array_equal(W1.reshape(-1), wbf[off:off + sz])
    for off, sz, kind in st._slices:
        if kind == "v":
            assert np.array_equal(st.wf32[off:off + sz].cpu().numpy(), wbf[off:off + sz])
    assert np.isfinite(float(st.loss.item()))
