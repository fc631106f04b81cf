#!/usr/bin/env bash
# K1 A/B on the bench: variants given as args (0 = auto), two runs each.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eval.py -x -q -k "variants or uint16 or fused" > gpurun_out/k1ab_test.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/k1ab_test.log
for v in "$@"; do for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --k1-variant $v > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('variant $v', d['value'],d['roofline']['frac'],d['roofline']['k1_ms'])"
done; done
