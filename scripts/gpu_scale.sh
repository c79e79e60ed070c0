#!/bin/bash
# multi-GPU: the 2-GPU NCCL tests, then bench at N = 1 .. $NG (torchrun), JSON lines -> gpurun_out/<tag>_scale.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-sc}; NG=${2:-2}
mkdir -p gpurun_out
python -c "import paper_2602_11410_b200.build as b; b.build()" > /dev/null
timeout 900 python -m pytest -q -m gpu tests/test_gpu_dp.py -rA > gpurun_out/${TAG}_dp_tests.log 2>&1; echo "dp tests -> $?"; tail -1 gpurun_out/${TAG}_dp_tests.log
: > gpurun_out/${TAG}_scale.jsonl
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n = 1 ]; then
    timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu ${BENCH_ARGS} >> gpurun_out/${TAG}_scale.jsonl 2> gpurun_out/${TAG}_n$n.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $n --steps 20 --warmup 5 ${BENCH_ARGS} >> gpurun_out/${TAG}_scale.jsonl 2> gpurun_out/${TAG}_n$n.err
  fi
  echo "n=$n -> $?"
done
python - <<PY
import json
for l in open('gpurun_out/${TAG}_scale.jsonl'):
    d=json.loads(l); e=d.get('e2e') or {}
    print(d['n_gpus'], 'value %.2fM tok/s' % (d['value']/1e6), 'ms %.3f' % d['ms_per_step'], 'e2e %.2fM' % (e.get('value',0)/1e6), e.get('host_numa_cpus'))
PY
