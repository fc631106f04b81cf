#!/usr/bin/env bash
# GPT2-XL (traced, 11k ops): config 5 sample, generator, plan parity + time.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eval.py -x -q -k "nccl or generator" > gpurun_out/xl_test.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/xl_test.log
timeout 600 python tools/config5.py --total ${XL_TOTAL:-262144} > gpurun_out/xl_config5.json 2> gpurun_out/xl_config5.err; echo "config5 rc=$?"; cat gpurun_out/xl_config5.json; tail -3 gpurun_out/xl_config5.err
timeout 300 python tools/gen_probe.py --graphs gpt2-xl --B 262144 --forms 0 > gpurun_out/xl_gen.txt 2>&1; cat gpurun_out/xl_gen.txt
timeout 1200 python tools/plan_bench.py --configs gpt2-xl --out gpurun_out/xl_plan.json > gpurun_out/xl_plan.log 2>&1; echo "plan rc=$?"; tail -3 gpurun_out/xl_plan.log
