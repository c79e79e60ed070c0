#!/bin/bash
# Same-box A/B: the working tree ("base") and each _ab/<name> tree, alternating, 2 rounds.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for i in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then dir=.; else dir=_ab/$v; fi
    (cd $dir && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > /tmp/ab_$v$i.json 2>/dev/null)
    python -c "
import json; d=json.load(open('/tmp/ab_$v$i.json'))
print('$v$i', 'ms/step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['roofline']['per_class_ms_per_step'].items()})"
  done
done
