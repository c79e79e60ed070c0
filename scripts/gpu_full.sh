#!/bin/bash
# full GPU test suite + smoke + bench (C4 default), results under gpurun_out/<tag>_*
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-full}
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rA ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?" > gpurun_out/${TAG}_summary.txt
tail -3 gpurun_out/${TAG}_tests.log >> gpurun_out/${TAG}_summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke -> $?" >> gpurun_out/${TAG}_summary.txt
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench -> $?" >> gpurun_out/${TAG}_summary.txt
cat gpurun_out/${TAG}_summary.txt
grep -E "passed|failed" gpurun_out/${TAG}_tests.log | tail -2
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('ms/step', round(d['ms_per_step'],3), 'Mtok/s', round(d['value']/1e6,3), 'TF/s', round(d['tflops'],1))
print({k: round(v,3) for k,v in d['roofline']['per_class_ms_per_step'].items()})
PY
