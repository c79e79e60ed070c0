#!/bin/bash
# ncu --set full of the step's main kernels (one launch each) after a clean run of the same command
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-pf}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
python -c "import paper_2602_11410_b200.build as b; b.build()" > /dev/null 2>&1
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"attn_|gemm_pair|rope_gate|gate_rope" -s 18 -c 12 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"
