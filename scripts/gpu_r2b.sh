make -s -C paper_2009_14514_b200/csrc >/dev/null; make -s -C oracle
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tests_r2b.log 2>&1; echo "exit $?" >> gpurun_out/tests_r2b.log
timeout 600 python scripts/parity_probe.py pcisph16k pcisph1m > gpurun_out/probe_r2b.log 2>&1; echo "exit $?" >> gpurun_out/probe_r2b.log
scripts/ab_lib.sh r2b build/variants/d10p8.so build/variants/d8p8.so build/variants/d8p6.so build/variants/d8p5.so build/variants/d6p6.so
