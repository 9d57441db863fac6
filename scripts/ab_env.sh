#!/bin/bash
# A/B runs of bench.py under environment overrides.
# usage: scripts/ab_env.sh TAG "RTS_CULL=4,RTS_PAIR_LANES=8" "RTS_CULL=0" ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=${1:-x}; shift
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $(echo "$cfg" | tr ',' ' ') timeout 600 python bench.py --no-cpu-baseline --no-e2e \
      > gpurun_out/ab_${TAG}_$i.log 2>&1
  echo "exit $? cfg $cfg" >> gpurun_out/ab_${TAG}_$i.log
done
