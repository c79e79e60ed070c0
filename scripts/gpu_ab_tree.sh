#!/bin/bash
# tests (-k filter $2, optional) then same-box A/B of the working tree vs _ab/$3 (built by scripts/ab_tree.sh)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ -n "$2" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x -k "$2" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?"
  tail -3 gpurun_out/${TAG}_tests.log
fi
for i in 1 2; do
  for v in $3 new; do
    if [ $v = new ]; then dir=.; else dir=_ab/$v; fi
    (cd $dir && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > /tmp/ab_$v$i.json 2>/tmp/ab_$v$i.err)
    cp /tmp/ab_$v$i.json gpurun_out/${TAG}_$v$i.json
    python -c "
import json; d=json.load(open('/tmp/ab_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})" || tail -3 /tmp/ab_$v$i.err
  done
done
