#!/bin/bash
# quick check: attention parity tests + bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-q}
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_core.py tests/test_gpu_layer.py -q -m gpu -x -k "${2:-attn_core or layer}" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?"
tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench -> $?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('ms/step', round(d['ms_per_step'],3), 'Mtok/s', round(d['value']/1e6,3), 'TF/s', round(d['tflops'],1), 'roofline', d['roofline']['kernel'], round(d['roofline']['frac'],3))
print({k: round(v,3) for k,v in d['roofline']['per_class_ms_per_step'].items()})
"
