#!/bin/bash
# WCSPH RTS vs global baselines: whole-run probe + launch lists of both modes
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python scripts/wcsph_whole_run.py ${1:-0.5} 0.05 > gpurun_out/wcsph_whole_run.log 2>&1
for m in rts baseline; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/wcsph_launch_$m.csv python scripts/prof_wcsph.py 8 $m > gpurun_out/wcsph_launch_$m.log 2>&1
done
