cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/ab_lib.sh rf build/variants/a.so build/variants/b.so build/variants/c.so build/variants/d.so
for v in a c; do cp build/variants/$v.so paper_2009_14514_b200/librtssph.so; timeout 300 python scripts/c6_probe.py > gpurun_out/c6_$v.log 2>&1; done
