#!/bin/bash
# A/B of prebuilt library variants, interleaved repetitions (cfg2 bench, device-timed):
#   scripts/ab_rep.sh TAG REPS lib1.so lib2.so ...  -> gpurun_out/abr_TAG_<lib>_<rep>.log
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; REPS=$2; shift 2
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for rep in $(seq 1 $REPS); do
  for lib in "$@"; do
    cp "$lib" paper_2009_14514_b200/librtssph.so
    n=$(basename "$lib" .so)
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph $AB_ARGS > gpurun_out/abr_${TAG}_${n}_$rep.log 2>&1
  done
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
