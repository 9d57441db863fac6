#!/bin/bash
# WCSPH step A/B: per-phase probe of a base library variant vs the in-tree one,
# then the WCSPH / grid / levels GPU tests on the in-tree library.
#   scripts/gpu_wcsph_ab.sh TAG build/variants/base.so
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; BASE=$2
mkdir -p gpurun_out
for rep in 1 2; do
  RTS_SPH_LIB=$BASE timeout 300 python scripts/wcsph_phase_probe.py 40 > gpurun_out/wab_${TAG}_base_$rep.log 2>&1
  timeout 300 python scripts/wcsph_phase_probe.py 40 > gpurun_out/wab_${TAG}_new_$rep.log 2>&1
done
timeout 900 python -m pytest -q -x -m gpu tests/test_wcsph_gpu.py tests/test_levels_gpu.py tests/test_grid_api_gpu.py tests/test_regions_api_gpu.py > gpurun_out/wab_${TAG}_tests.log 2>&1
