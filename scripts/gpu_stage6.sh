#!/bin/bash
# tests (grouped, separate processes), smoke, bench, ncu launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/s6_build.log 2>&1
for k in "gemm or mask_plan or chunk or pack or attn_core_forward" attn_core_backward heads layer_forward layer_backward; do
  f="gpurun_out/s6_$(echo $k | cut -c1-12 | tr ' ' _).log"
  timeout 600 python -m pytest tests/test_gpu_core.py tests/test_gpu_layer.py -q -m gpu -k "$k" -s -rA > "$f" 2>&1
  echo "$k -> $?" >> gpurun_out/s6_summary.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke.log 2>&1; echo "smoke -> $?" >> gpurun_out/s6_summary.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s6_bench.json 2> gpurun_out/s6_bench.err; echo "bench -> $?" >> gpurun_out/s6_summary.txt
cat gpurun_out/s6_summary.txt
tail -c 3000 gpurun_out/s6_bench.json
