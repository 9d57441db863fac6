#!/bin/bash
# FMA peaks + ncu --set full of the WCSPH pair kernels (1M RTS step and 1M
# global step) + the WCSPH step A/B against a base library.
#   scripts/gpu_wcsph_evidence.sh TAG build/variants/base.so
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; BASE=$2
mkdir -p gpurun_out build
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fma_peak scripts/fma_peak.cu && \
  build/fma_peak > gpurun_out/fma_peak.json 2>&1
bash scripts/gpu_wcsph_ab.sh $TAG $BASE
for m in rts baseline; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_density|k_forces" \
    --launch-skip 16 --launch-count 2 -o gpurun_out/wpair_$m python scripts/prof_wcsph.py 8 $m \
    > gpurun_out/wpair_$m.log 2>&1
done
