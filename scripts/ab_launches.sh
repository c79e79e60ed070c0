#!/bin/bash
# per-kernel device time of one bench step (ncu launch list) for the working tree and _ab/<name>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import paper_2602_11410_b200.build as b; b.build()" > /dev/null
for v in base "$@"; do
  if [ $v = base ]; then dir=.; else dir=_ab/$v; fi
  (cd $dir && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l_$v.csv \
     python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1)
  cp /tmp/l_$v.csv gpurun_out/ab_launches_$v.csv
done
python scripts/launch_diff.py gpurun_out/ab_launches_base.csv $(for v in "$@"; do echo gpurun_out/ab_launches_$v.csv; done)
