#!/bin/bash
# The bounds-checked library (every gathered / scattered index of the hot
# kernels range-checked, RTS_ERR_CHECK + site on a violation) and the GPU
# suite run against it: compute-sanitizer's role on a pool where it is closed.
#   scripts/checked_build.sh            (build only: build/variants/checked.so)
#   scripts/checked_build.sh run TAG    (on the GPU box: pytest -m gpu with it)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
if [ "$1" = run ]; then
  mkdir -p gpurun_out
  RTS_SPH_LIB=build/variants/checked.so timeout 1800 python -m pytest tests -q -m gpu \
      > gpurun_out/checked_${2:-x}.log 2>&1
  echo "exit $?" >> gpurun_out/checked_${2:-x}.log
else
  scripts/build_variant.sh checked "-DRTS_CHECKED=1"
fi
