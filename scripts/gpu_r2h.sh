#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/tests_r2h.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2h.log
scripts/ab_lib.sh r2h build/variants/r8.so build/variants/r6.so build/variants/r8g1.so build/variants/r6g1.so
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r2h.csv $B > /dev/null 2>&1
timeout 900 python scripts/parity_probe.py f32twin16k f32twin1m wcsph1m > gpurun_out/probe_r2h.log 2>&1; echo "exit $?" >> gpurun_out/probe_r2h.log
echo done > gpurun_out/done_r2h
