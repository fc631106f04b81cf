#!/usr/bin/env bash
# K1 A/B on one B200: GPU eval tests, then the bench under each environment
# setting given as arguments (e.g. "ROAM_K1_BULK=0" "ROAM_K1_BULK=1"), twice
# each, then one ncu full capture of K1 under the first setting.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu ${PYTEST_FILES:-tests/test_gpu_eval.py tests/test_gpu_config5.py} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
i=0
for setting in "$@"; do
  for rep in 1 2; do
    i=$((i+1))
    env $setting timeout 300 python bench.py > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$i.json'));print('$setting', round(d['value']/1e6,1), 'M/s frac', round(d['roofline']['frac'],4), 'k1_ms', round(d['roofline']['k1_ms'],5))" 2>&1 | tail -1
  done
done
env ${1:-X=1} timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1.*eval_orders -s 2 -c 1 -o gpurun_out/k1_full -f python bench.py --steps 3 --warmup 2 --profile > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
