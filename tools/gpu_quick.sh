#!/usr/bin/env bash
# Quick K1 loop: microbenchmarks, GPU eval tests, bench x2, one ncu full capture of K1.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
[ -x tools/mb/shfl_vs_lds ] && timeout 60 tools/mb/shfl_vs_lds > gpurun_out/mb_shfl.txt 2>&1; cat gpurun_out/mb_shfl.txt 2>/dev/null
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_K:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$i.json'));print(d['value'],d['roofline']['frac'],d['roofline']['k1_ms'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1.*eval_orders -s 2 -c 1 -o gpurun_out/k1_full -f python bench.py --steps 3 --warmup 2 --profile > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
