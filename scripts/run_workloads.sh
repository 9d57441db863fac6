cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x > gpurun_out/wl_tests.log 2>&1; echo "exit $?" >> gpurun_out/wl_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-wcsph > gpurun_out/wl_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/wl_cfg2.log
for w in cfg4 cfg5-pcisph cfg5-wcsph; do
timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/wl_$w.log 2>&1; echo "exit $?" >> gpurun_out/wl_$w.log
done
timeout 600 python bench.py --impl reference --workload cfg5-wcsph --steps 3 --warmup 1 > gpurun_out/wl_ref5w.log 2>&1; echo "exit $?" >> gpurun_out/wl_ref5w.log
