#!/bin/bash
# A/B of prebuilt library variants: scripts/ab_lib.sh TAG build/variants/a.so build/variants/b.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; shift
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for lib in "$@"; do
  cp "$lib" paper_2009_14514_b200/librtssph.so
  n=$(basename "$lib" .so)
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/ab_${TAG}_$n.log 2>&1
  echo "exit $? cfg $n" >> gpurun_out/ab_${TAG}_$n.log
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
