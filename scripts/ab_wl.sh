#!/bin/bash
# A/B of prebuilt library variants on cfg2 (default bench, no WCSPH line) and
# the 4M RTS-WCSPH scene, interleaved repetitions:
#   scripts/ab_wl.sh TAG REPS lib1.so lib2.so ...  -> gpurun_out/abw_TAG_<lib>_<wl>_<rep>.log
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; REPS=$2; shift 2
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for rep in $(seq 1 $REPS); do
  for lib in "$@"; do
    cp "$lib" paper_2009_14514_b200/librtssph.so
    n=$(basename "$lib" .so)
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/abw_${TAG}_${n}_cfg2_$rep.log 2>&1
    timeout 600 python bench.py --workload cfg5-wcsph --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abw_${TAG}_${n}_w4m_$rep.log 2>&1
  done
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
