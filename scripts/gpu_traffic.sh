#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-tr}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu ${2}"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"
