#!/bin/bash
# bench each prebuilt paper_2602_11410_b200/libcadet_<v>.so (CADET_LIB) alternately: scripts/gpu_variants_bench.sh TAG v1 v2 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
for i in 1 2; do
  for v in "$@"; do
    CADET_LIB=$PWD/paper_2602_11410_b200/libcadet_$v.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG}_$v$i.json 2> gpurun_out/${TAG}_$v$i.err
    python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})" || tail -5 gpurun_out/${TAG}_$v$i.err
  done
done
