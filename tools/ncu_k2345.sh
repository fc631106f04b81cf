set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for k in k3_llfb k4_greedy k2_pairs; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${k}_full -f python tools/k234_bench.py --configs gpt2-xl > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
timeout 600 ncu --set full --clock-control none -k regex:k5_exact -c 1 -o gpurun_out/k5_exact_full -f python tools/plan_bench.py --configs gpt2-xl --skip-ref > gpurun_out/ncu_k5.log 2>&1; echo "k5 rc=$?"
