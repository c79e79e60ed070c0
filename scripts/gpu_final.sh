#!/bin/bash
# end-of-round evidence: full GPU tests, smoke, the default bench line (C4), the C3 bench line, the per-launch
# DRAM-traffic list of one C4 step, results under gpurun_out/<tag>_*
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-fin}
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rA > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?"
tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke -> $?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo "bench c4 -> $?"
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err; echo "bench c3 -> $?"
bash scripts/gpu_traffic.sh ${TAG}_tr > /dev/null 2>&1; echo "traffic -> $?"
python - <<PY
import json
for w in ("c4", "c3"):
    d = json.load(open("gpurun_out/${TAG}_bench_%s.json" % w))
    e = d.get("e2e") or {}
    print(w, "ms %.3f" % d["ms_per_step"], "Mtok/s %.2f" % (d["value"] / 1e6), "TF/s %.0f" % d["tflops"],
          "frac %.3f" % d["frac_of_peak_measured"], "e2e %.2f" % (e.get("value", 0) / 1e6),
          {k: round(v, 3) for k, v in d["roofline"]["per_class_ms_per_step"].items()})
PY
