#!/bin/bash
# Build libcadet from git revision $1 into paper_2602_11410_b200/libcadet_$2.so (A/B comparisons)
set -e
cd /root/repo
REV=$1; NAME=$2
D=$(mktemp -d)
git archive $REV paper_2602_11410_b200/csrc include | tar -x -C $D
OBJS=""
for f in $D/paper_2602_11410_b200/csrc/*.cu; do
  o=$D/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -diag-suppress 550,177 -c $f -o $o &
  OBJS="$OBJS $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OBJS -o paper_2602_11410_b200/libcadet_$NAME.so -lcudart
rm -rf $D
echo built libcadet_$NAME.so
