#!/bin/bash
# same-box A/B: round-1 tree (build/base_r1) vs this tree; ncu of k_density in both
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
(cd build/base_r1 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph) > gpurun_out/ab_r2c_base.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/ab_r2c_new.log 2>&1
(cd build/base_r1 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph) > gpurun_out/ab_r2c_base2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/ab_r2c_new2.log 2>&1
$B > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_density -c 1 -o gpurun_out/full_r2c_dens $B > /dev/null 2>&1
(cd build/base_r1 && $B > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_density -c 1 -o ../../gpurun_out/full_r2c_dens_base $B > /dev/null 2>&1)
echo done > gpurun_out/done_r2c
