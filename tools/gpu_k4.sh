#!/usr/bin/env bash
# K4 loop: its GPU tests (greedy, exact incumbents, plan documents), the
# planner-subtask bench, ncu launch times and one full capture.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as e; e.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_greedy.py tests/test_gpu_exact.py ${K4_TESTS:-tests/test_gpu_plan.py} -x -q > gpurun_out/k4_test.log 2>&1; echo "k4 tests rc=$?"; tail -3 gpurun_out/k4_test.log
timeout 900 python tools/k234_bench.py --configs bert-large gpt2-xl --out gpurun_out/k234.json > gpurun_out/k234.log 2>&1; echo "k234 rc=$?"; tail -3 gpurun_out/k234.log | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k4_greedy --csv --log-file gpurun_out/k4_launch.csv python tools/k234_bench.py --configs gpt2-xl > gpurun_out/ncu_k4_launch.log 2>&1; echo "ncu rc=$?"; grep k4_greedy gpurun_out/k4_launch.csv | cut -c1-400 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_greedy -c 1 -o gpurun_out/k4_greedy_full -f python tools/k234_bench.py --configs gpt2-xl > gpurun_out/ncu_k4_full.log 2>&1; echo "ncu full rc=$?"
