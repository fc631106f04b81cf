#!/usr/bin/env bash
# K3 iteration on one B200: layout/plan parity tests, K2-K4 subtask bench, plan bench.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_pack.py tests/test_gpu_plan.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k3.log
timeout 900 python tools/k234_bench.py --configs layered bert-large gpt2-xl --out gpurun_out/k234.json > gpurun_out/k234.log 2>&1; echo "k234 rc=$?"; tail -8 gpurun_out/k234.log
timeout 1200 python tools/plan_bench.py --configs layered gpt2-small bert-large gpt2-xl ref-transformer_block-600 --out gpurun_out/plan_bench.json > gpurun_out/plan_bench.log 2>&1; echo "plan rc=$?"; cut -c1-400 gpurun_out/plan_bench.log | tail -5
