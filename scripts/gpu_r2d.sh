#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
scripts/ab_lib.sh r2d paper_2009_14514_b200/librtssph.so build/variants/dc3m10.so build/variants/dc2m10.so build/variants/dc4m8.so build/variants/pc2m6.so build/variants/pc4m4.so
timeout 900 python scripts/parity_probe.py series16k series1m > gpurun_out/probe_r2d.log 2>&1; echo "exit $?" >> gpurun_out/probe_r2d.log
