#!/usr/bin/env bash
# K1 iteration loop on one B200: eval parity tests, A/B timing, bench, one
# full ncu capture of the default K1 kernel.  Each step bounded by a timeout.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eval.py -x -q > gpurun_out/pytest_eval.log 2>&1; echo "pytest-eval rc=$?"; tail -3 gpurun_out/pytest_eval.log
timeout 300 python tools/k1_ab.py ${K1_GRAPHS:-} > gpurun_out/k1_ab.jsonl 2>&1; echo "k1_ab rc=$?"; cat gpurun_out/k1_ab.jsonl
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${1:-}" != "noprof" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1.*eval_orders -s 2 -c 1 -o gpurun_out/k1_full -f python bench.py --steps 3 --warmup 2 --profile > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
fi
