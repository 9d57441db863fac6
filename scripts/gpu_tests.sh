#!/bin/bash
# the GPU suite + smoke: gpurun_out/tests_TAG.log, smoke_TAG.log
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -q -m gpu "$@" > gpurun_out/tests_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/tests_$TAG.log
