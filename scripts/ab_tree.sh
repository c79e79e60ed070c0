#!/bin/bash
# Export commit $1's tree into _ab/$2/ and build its libcadet.so there, for same-box A/B benches
# of whole-tree states (model.py as well as kernels): run `python _ab/$2/bench.py` next to `python bench.py`.
set -e
cd /root/repo
REV=$1; NAME=$2
rm -rf _ab/$NAME && mkdir -p _ab/$NAME
git archive $REV | tar -x -C _ab/$NAME
(cd _ab/$NAME && python -c "from paper_2602_11410_b200 import build; build.build()" > /dev/null)
echo "_ab/$NAME built from $(git rev-parse --short $REV)"
