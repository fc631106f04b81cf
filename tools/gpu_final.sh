#!/usr/bin/env bash
# Round-end evidence on one B200: build, GPU tests, smoke, bench (both arms),
# ncu launch list + one full K1 capture, plan bench, K2-K4 bench, config 5,
# generator probe, ncu captures of K2-K5, compute-sanitizer.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash tools/gpu_check.sh
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench-ref rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
timeout 1500 python tools/plan_bench.py --configs layered gpt2-small bert-large gpt2-xl ref-transformer_block-600 --out gpurun_out/plan_bench.json > gpurun_out/plan_bench.log 2>&1; echo "plan rc=$?"
timeout 900 python tools/k234_bench.py --configs layered bert-large gpt2-xl --out gpurun_out/k234.json > gpurun_out/k234.log 2>&1; echo "k234 rc=$?"
timeout 900 python tools/config5.py > gpurun_out/config5.json 2> gpurun_out/config5.err; echo "config5 rc=$?"; cat gpurun_out/config5.json
timeout 300 python tools/gen_probe.py --graphs gpt2-small bert-large gpt2-xl --B 262144 > gpurun_out/gen_probe.txt 2>&1; echo "gen rc=$?"; cat gpurun_out/gen_probe.txt
if [ "${1:-}" != "quick" ]; then
timeout 1500 bash tools/ncu_k2345.sh > gpurun_out/ncu_k2345.log 2>&1; echo "ncu k2-5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gen_thread -c 1 -o gpurun_out/gen_full -f python tools/gen_probe.py --graphs gpt2-xl --once > gpurun_out/ncu_gen.log 2>&1; echo "ncu gen rc=$?"
bash tools/gpu_sanitize.sh
fi
