#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tests_r2k.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2k.log
scripts/ab_lib.sh r2k build/variants/s8.so build/variants/s6.so build/variants/nosoa.so
for v in s8 nosoa; do
  cp build/variants/$v.so paper_2009_14514_b200/librtssph.so
  timeout 600 python bench.py --workload cfg5-wcsph --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abw_r2k_$v.log 2>&1
done
echo done > gpurun_out/done_r2k
