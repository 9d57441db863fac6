#!/bin/bash
# A/B of library variants on the default workload and the 4M-per-GPU scenes:
#   scripts/gpu_ab.sh TAG lib1.so lib2.so ...   (logs: gpurun_out/ab_TAG_<lib>_<workload>.log)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; shift
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for rep in 1 2; do
for lib in "$@"; do
  cp "$lib" paper_2009_14514_b200/librtssph.so
  n=$(basename "$lib" .so)
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/ab_${TAG}_${n}_cfg2_$rep.log 2>&1
  for w in cfg5-pcisph cfg5-wcsph; do
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_${n}_${w}_$rep.log 2>&1
  done
done
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
