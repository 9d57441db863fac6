#!/bin/bash
# Round-2 evidence for profiles/: bench lines (cfg2 default + BASELINE's other
# workloads), the ncu launch list and DRAM traffic per kernel of the same
# command, and --set full captures of the PCISPH pair kernels and the refresh.
# Every ncu run follows a plain run of the same command that exited 0.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
T=${1:-r02}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "exit $?" >> gpurun_out/${T}_bench.log
for w in cfg4 cfg5-pcisph cfg5-wcsph; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_wl_$w.log 2>&1; echo "exit $?" >> gpurun_out/${T}_wl_$w.log
done
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
$B > gpurun_out/${T}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_launches.csv $B > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_traffic.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_density|k_pforces" -c 2 -o gpurun_out/${T}_full_pair $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k k_refresh -c 1 -o gpurun_out/${T}_full_refresh $B > /dev/null 2>&1
W="python bench.py --workload cfg5-wcsph --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$W > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_wcsph_launches.csv $W > /dev/null 2>&1
echo done > gpurun_out/${T}_done
