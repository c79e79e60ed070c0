#!/bin/bash
# same-box A/B of the working tree vs _ab/<name>: 3 alternating bench runs each (kernel-only, C4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import paper_2602_11410_b200.build as b; b.build()" > /dev/null
for i in 1 2 3 4; do
  order="base $@"
  [ $((i % 2)) = 0 ] && order="$@ base"   # alternate which tree runs first (the second run of a pair is slower)
  for v in $order; do
    if [ $v = base ]; then dir=.; else dir=_ab/$v; fi
    (cd $dir && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > /tmp/ab_$v$i.json 2>/dev/null)
    python -c "
import json; d=json.load(open('/tmp/ab_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})"
  done
done
