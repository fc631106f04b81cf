set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python tools/plan_bench.py --configs layered gpt2-small bert-large gpt2-xl ref-transformer_block-600 --out gpurun_out/plan_bench.json > gpurun_out/plan_bench.log 2>&1; echo "plan rc=$?"; tail -5 gpurun_out/plan_bench.log
