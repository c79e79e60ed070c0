#!/bin/bash
# ncu evidence for one bench configuration: launch list (per-kernel device time) + full captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 17 -c 4 -o gpurun_out/${TAG}_gemm $CMD > gpurun_out/${TAG}_ncu_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 2 -c 2 -o gpurun_out/${TAG}_attn $CMD > gpurun_out/${TAG}_ncu_attn.log 2>&1
echo "exit $?"
ls -la gpurun_out/ | grep ${TAG}
