#!/usr/bin/env bash
# Round-end evidence on one B200: build, GPU tests, smoke, bench (both arms),
# ncu launch list + one full K1 capture, plan bench, K2-K4 bench, config 5.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash tools/gpu_check.sh
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench-ref rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
timeout 1200 python tools/plan_bench.py --configs layered gpt2-small bert-large gpt2-xl ref-transformer_block-600 --out gpurun_out/plan_bench.json > gpurun_out/plan_bench.log 2>&1; echo "plan rc=$?"
timeout 900 python tools/k234_bench.py --configs layered bert-large gpt2-xl --out gpurun_out/k234.json > gpurun_out/k234.log 2>&1; echo "k234 rc=$?"
timeout 900 python tools/config5.py > gpurun_out/config5.json 2> gpurun_out/config5.err; echo "config5 rc=$?"; cat gpurun_out/config5.json
