#!/usr/bin/env bash
# K3 / K4 loop: their GPU tests, the planner subtask bench, ncu captures.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_greedy.py tests/test_gpu_layout.py -x -q > gpurun_out/k34_test.log 2>&1; echo "k34 tests rc=$?"; tail -3 gpurun_out/k34_test.log
timeout 900 python tools/k234_bench.py --configs ${K34_CONFIGS:-bert-large gpt2-xl} --out gpurun_out/k234.json > gpurun_out/k234.log 2>&1; echo "k234 rc=$?"; tail -5 gpurun_out/k234.log
if [ "${1:-}" = "ncu" ]; then
timeout 900 bash tools/ncu_k2345.sh > gpurun_out/ncu_k2345.log 2>&1; echo "ncu rc=$?"
fi
