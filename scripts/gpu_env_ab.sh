#!/bin/bash
# tests (pytest -k filter $2) then same-box A/B of an environment switch: scripts/gpu_env_ab.sh TAG "k-filter" "ENV=1"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-ea}
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -k "$2" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?"
  tail -3 gpurun_out/${TAG}_tests.log
fi
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then ENVV="$3"; else ENVV=""; fi
    env $ENVV timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG}_$v$i.json 2> gpurun_out/${TAG}_$v$i.err
    python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})" || tail -5 gpurun_out/${TAG}_$v$i.err
  done
done
