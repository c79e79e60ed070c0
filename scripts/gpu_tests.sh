#!/bin/bash
# selected GPU tests: scripts/gpu_tests.sh TAG "pytest args..."
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-t}
shift
python -c "import paper_2602_11410_b200.build as b; b.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest -q -m gpu -rA "$@" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests -> $?"
grep -E "^(PASSED|FAILED|ERROR)|passed|failed" gpurun_out/${TAG}_tests.log | tail -60
