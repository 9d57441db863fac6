#!/bin/bash
# A/B of prebuilt library variants on the RTS-WCSPH bench (cfg5-wcsph, 4 M):
#   scripts/ab_wcsph.sh TAG build/variants/a.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; shift
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for lib in "$@"; do
  cp "$lib" paper_2009_14514_b200/librtssph.so
  n=$(basename "$lib" .so)
  timeout 600 python bench.py --workload cfg5-wcsph --steps 20 --no-cpu-baseline --no-e2e \
    > gpurun_out/abw_${TAG}_$n.log 2>&1
  echo "exit $? cfg $n" >> gpurun_out/abw_${TAG}_$n.log
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
