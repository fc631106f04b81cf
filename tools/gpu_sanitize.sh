#!/usr/bin/env bash
# compute-sanitizer over every libroam kernel (tools/sanitize_run.py):
# memcheck, racecheck, synccheck, initcheck; logs to gpurun_out/sanitize_*.log
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_run.py ${1:-all} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
