#!/usr/bin/env bash
# K1 loop: eval GPU tests, bench x2, ncu full capture of the bench's K1.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eval.py tests/test_gpu_config5.py -x -q > gpurun_out/k1_test.log 2>&1; echo "k1 tests rc=$?"; tail -2 gpurun_out/k1_test.log
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$i.json'));print(d['value'],d['roofline']['frac'],d['roofline']['k1_ms'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1.*eval_orders -s 2 -c 1 -o gpurun_out/k1_full -f python bench.py --steps 3 --warmup 2 --profile > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
