#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# scripts/sanitize_drive.py (tiny tank: both solvers, graph + host-driven,
# audit, halo pack/unpack).  Summaries -> gpurun_out/sanitize_<tool>.log
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 900 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python scripts/sanitize_drive.py ${1:-all} > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
