#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -k "parity_scale or variance" > gpurun_out/tests_r2j.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2j.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
$B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_density|k_pforces" -c 2 -o gpurun_out/full_r2j_pair $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k k_refresh -c 1 -o gpurun_out/full_r2j_refresh $B > /dev/null 2>&1
echo done > gpurun_out/done_r2j
