#!/bin/bash
# ONE ncu --set full capture per gpurun call (after the same command ran clean without ncu).
# usage: gpu_prof_one.sh TAG KERNEL_REGEX SKIP COUNT
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; RE=$2; SKIP=${3:-0}; CNT=${4:-1}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c $CNT -o gpurun_out/${TAG} $CMD \
  > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"
