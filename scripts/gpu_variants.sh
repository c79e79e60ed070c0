#!/bin/bash
# Same-GPU comparison of prebuilt libcadet_<V>.so variants (and the in-tree build as "base")
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
for i in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then unset CADET_LIB; else export CADET_LIB=$PWD/paper_2602_11410_b200/libcadet_$v.so; fi
    timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_$v$i.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})"
  done
done
