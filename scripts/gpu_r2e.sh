#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1500 python scripts/parity_probe.py pcisph16k pcisph1m wcsph1m twin16k twin1m > gpurun_out/probe_r2e.log 2>&1; echo "exit $?" >> gpurun_out/probe_r2e.log
