#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_smi.txt 2>&1
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/s1_build.log 2>&1
for k in gemm "mask_plan or chunk or pack" attn_core_forward; do
  timeout 600 python -m pytest tests/test_gpu_core.py -q -m gpu -k "$k" -x > "gpurun_out/s1_$(echo $k | cut -c1-8 | tr ' ' _).log" 2>&1
  echo "$k -> $?" >> gpurun_out/s1_summary.txt
done
tail -3 gpurun_out/s1_*.log
