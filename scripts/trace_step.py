"""Timeline of one C4 training step (torch.profiler / CUPTI activity records): every kernel and
memset with its start / duration, and the idle gaps between consecutive GPU operations — to see
where the step's time goes outside the kernels.  Diagnostic only (numbers taken under a tracer)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    from paper_2602_11410_b200.model import CadetStack, StackConfig
    wl = bench.WORKLOADS[os.environ.get("WL", "c4")]
    users, hinp = bench.build_inputs(wl, 0, pin=False)
    inp = hinp.to("cuda")
    st = CadetStack(StackConfig(d_model=wl["d_model"], n_heads=wl["n_heads"], n_layers=wl["n_layers"],
                                budget=wl["budget"], L_chunk=wl["L_chunk"]), device="cuda")
    for _ in range(3):
        st.step(inp)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            st.step(inp)
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        evs.append((e.time_range.start, e.time_range.end, e.name))
    evs.sort()
    # the second step: split at the pack kernel that starts it
    starts = [i for i, e in enumerate(evs) if "pack_offsets" in e[2]]
    a = starts[-1]
    step = evs[a:]
    t0 = step[0][0]
    rows, busy, gaps = [], 0.0, []
    prev_end = t0
    for s, e, n in step:
        gap = s - prev_end
        if gap > 0:
            gaps.append((gap, n))
        busy += e - s
        rows.append({"t_us": round(s - t0, 1), "dur_us": round(e - s, 1), "gap_before_us": round(max(gap, 0), 1),
                     "name": n[:80]})
        prev_end = max(prev_end, e)
    total = prev_end - t0
    out = {"step_us": round(total, 1), "busy_us": round(busy, 1), "idle_us": round(total - busy, 1),
           "n_ops": len(step), "ops": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
