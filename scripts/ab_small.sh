cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in b e; do cp build/variants/$v.so paper_2009_14514_b200/librtssph.so; timeout 300 python scripts/c6_probe.py > gpurun_out/c6_$v.log 2>&1; done
cp build/variants/e.so paper_2009_14514_b200/librtssph.so
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t_e.log 2>&1; echo "exit $?" >> gpurun_out/t_e.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-wcsph > gpurun_out/b_e.log 2>&1
