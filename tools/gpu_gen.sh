#!/usr/bin/env bash
# Candidate generator: GPU tests, timing of both forms, one ncu capture.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eval.py -x -q -k "generator" > gpurun_out/gen_test.log 2>&1; echo "gen tests rc=$?"; tail -3 gpurun_out/gen_test.log
timeout 300 python tools/gen_probe.py ${GEN_ARGS:-} > gpurun_out/gen_bench.txt 2>&1; cat gpurun_out/gen_bench.txt
if [ "${1:-}" = "ncu" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gen_thread -c 1 -o gpurun_out/gen_full -f python tools/gen_probe.py --graphs gpt2-xl --once > gpurun_out/ncu_gen.log 2>&1; echo "ncu rc=$?"
fi
