#!/bin/bash
# A/B of two source trees (this one and TREE, e.g. a worktree of another
# commit under build/): bench lines of both, alternating, on one box.
#   scripts/gpu_ab_tree.sh TAG TREE
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
TAG=$1; TREE=$2
mkdir -p gpurun_out
here=$(pwd)
for rep in 1 2; do
  for side in base new; do
    dir=$here; [ $side = base ] && dir=$here/$TREE
    (cd $dir && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-wcsph) > gpurun_out/ab_${TAG}_${side}_cfg2_$rep.log 2>&1
    (cd $dir && timeout 600 python bench.py --workload cfg5-pcisph --steps 10 --warmup 3 --no-cpu-baseline --no-e2e) > gpurun_out/ab_${TAG}_${side}_cfg5-pcisph_$rep.log 2>&1
  done
done
