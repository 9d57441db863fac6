#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2i.log 2>&1; echo "exit $?" >> gpurun_out/smoke_r2i.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/tests_r2i.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2i.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2i.log 2>&1; echo "exit $?" >> gpurun_out/bench_r2i.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_r2i.log 2>&1; echo "exit $?" >> gpurun_out/ref_r2i.log
timeout 900 python scripts/parity_probe.py argmax1m > gpurun_out/probe_r2i.log 2>&1; echo "exit $?" >> gpurun_out/probe_r2i.log
echo done > gpurun_out/done_r2i
