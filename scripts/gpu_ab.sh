#!/bin/bash
# A/B on one GPU: alternate benches with libcadet_A.so and the in-tree libcadet.so (B)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-ab}
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then export CADET_LIB=$PWD/paper_2602_11410_b200/libcadet_A.so; else unset CADET_LIB; fi
    timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_$v$i.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})"
  done
done
