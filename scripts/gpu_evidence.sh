#!/bin/bash
# One evidence run for profiles/ (scripts/write_profiles.sh TAG reads it):
# GPU suite + smoke, bench lines and ncu captures (gpu_profile_r02.sh), the
# refresh / graph-phase probes with a full capture of the major-start
# refresh, and the reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
T=${1:-ev}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $T
bash scripts/gpu_profile_r02.sh $T
timeout 600 python scripts/refresh_probe.py 20 > gpurun_out/${T}_refresh_probe.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:'k_refresh$' -s 3 -c 1 \
      -o gpurun_out/${T}_refresh_probe_full python scripts/refresh_probe.py 2 > /dev/null 2>&1
timeout 600 python scripts/graph_phase_probe.py 20 3 > gpurun_out/${T}_graph_phase.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1; echo "exit $?" >> gpurun_out/${T}_ref.log
echo done > gpurun_out/${T}_evidence_done
