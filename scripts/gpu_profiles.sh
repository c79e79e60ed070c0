#!/bin/bash
# round evidence for the default bench (C4): plain JSON, ncu launch list, DRAM traffic per launch, and
# `ncu --set full` captures of the top kernels (each after its command exited 0 without ncu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import paper_2602_11410_b200.build as b; b.build()" > /dev/null
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_traffic.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -s 14 -c 5 -o gpurun_out/${TAG}_gemm $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_" -s 3 -c 3 -o gpurun_out/${TAG}_attn $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rope_gate|gate_rope" -s 2 -c 2 -o gpurun_out/${TAG}_elem $CMD > /dev/null 2>&1
ls -la gpurun_out/ | grep ${TAG}
