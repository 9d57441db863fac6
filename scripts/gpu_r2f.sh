#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "not parity_scale" > gpurun_out/tests_r2f.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2f.log
scripts/ab_lib.sh r2f paper_2009_14514_b200/librtssph.so build/variants/nocull.so
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
$B > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_refresh -c 1 -o gpurun_out/full_r2f_refresh $B > /dev/null 2>&1
echo done > gpurun_out/done_r2f
