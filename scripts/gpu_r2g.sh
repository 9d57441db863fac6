#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tests_r2g.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2g.log
scripts/ab_lib.sh r2g build/variants/cm8.so build/variants/cm6.so build/variants/cm5.so build/variants/nocull.so
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r2g.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k k_refresh -c 1 -o gpurun_out/full_r2g_refresh $B > /dev/null 2>&1
cp build/variants/nocull.so paper_2009_14514_b200/librtssph.so
ncu --set full --import-source on --clock-control none -k k_refresh -c 1 -o gpurun_out/full_r2g_refresh_nocull $B > /dev/null 2>&1
echo done > gpurun_out/done_r2g
