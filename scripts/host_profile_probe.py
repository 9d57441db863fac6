"""Probe (not the bench): cProfile of the host side of PcisphSolver.advance()
(graph mode, cfg2) -- where the ~35 us between majors go."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

s = bench.make_device_solver("pcisph", torch.device("cuda", 0), "cfg2")
for _ in range(3):
    s.advance()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(40):
    s.advance()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
