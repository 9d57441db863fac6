#!/bin/bash
# Round-trip for profiles/: tests, bench line, launch list, DRAM traffic per
# kernel and one `ncu --set full` capture of KERNEL (every ncu run follows a
# plain run of the same command that exited 0).
# usage: scripts/profile_cycle.sh TAG [KERNEL]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; K=${2:-k_refresh}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e"
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/tests_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/tests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_$TAG.log
$B > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv $B > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/traffic_$TAG.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k $K -c 1 -o gpurun_out/full_$TAG $B > /dev/null 2>&1
echo done > gpurun_out/done_$TAG
