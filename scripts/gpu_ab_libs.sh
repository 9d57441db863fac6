#!/bin/bash
# A/B of library variants: cfg2 bench (twice, alternating) + WCSPH phase probe.
#   scripts/gpu_ab_libs.sh TAG a.so b.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename "$lib" .so)
    RTS_SPH_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-wcsph \
      > gpurun_out/abl_${TAG}_${n}_$rep.log 2>&1
  done
done
for lib in "$@"; do
  n=$(basename "$lib" .so)
  RTS_SPH_LIB=$lib timeout 300 python scripts/wcsph_phase_probe.py 40 > gpurun_out/abl_${TAG}_${n}_wcsph.log 2>&1
done
