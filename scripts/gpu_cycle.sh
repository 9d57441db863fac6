#!/bin/bash
# One GPU round trip: parity tests, bench line, ncu launch list (plain run first).
# usage: scripts/gpu_cycle.sh TAG [tests|bench|ncu ...]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; shift
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/tests_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/tests_$TAG.log ;;
    bench) timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_$TAG.log ;;
    ncu) python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
         ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv \
             python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e > gpurun_out/ncu_$TAG.log 2>&1 ;;
  esac
done
