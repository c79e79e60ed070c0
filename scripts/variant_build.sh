#!/bin/bash
# Build libcadet from the working tree with extra compile flags into paper_2602_11410_b200/libcadet_$1.so
# (profiling experiments only; e.g. scripts/variant_build.sh V1 -DCADET_EXP_NOSRC)
set -e
cd /root/repo
NAME=$1; shift
D=$(mktemp -d)
OBJS=""
for f in paper_2602_11410_b200/csrc/*.cu; do
  o=$D/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -diag-suppress 550,177 "$@" -c $f -o $o &
  OBJS="$OBJS $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OBJS -o paper_2602_11410_b200/libcadet_$NAME.so -lcudart
rm -rf $D
echo built libcadet_$NAME.so
