#!/bin/bash
# Run a probe script against prebuilt library variants on one box:
#   scripts/probe_variants.sh TAG "python scripts/refresh_probe.py" build/variants/a.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; CMD=$2; shift 2
mkdir -p gpurun_out
cp paper_2009_14514_b200/librtssph.so /tmp/librtssph.keep.so
for rep in 1 2; do
for lib in "$@"; do
  cp "$lib" paper_2009_14514_b200/librtssph.so
  n=$(basename "$lib" .so)
  echo "== $n rep $rep" >> gpurun_out/probe_${TAG}.log
  timeout 300 $CMD >> gpurun_out/probe_${TAG}.log 2>&1
done
done
cp /tmp/librtssph.keep.so paper_2009_14514_b200/librtssph.so
