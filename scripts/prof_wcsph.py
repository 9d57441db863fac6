"""Profiling driver: 1M WCSPH (configs[2] geometry), a few warm steps then N steps.

    python scripts/prof_wcsph.py [N=8] [rts|baseline]   (baseline: dt_cap = 4 dt_base)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
sys.argv += [None] * 2
n = int(sys.argv[1]) if sys.argv[1] else 8
mode = sys.argv[2] or "rts"
dev = torch.device("cuda", 0)
if mode == "rts":
    s = bench.make_device_solver("wcsph", dev)
else:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from wcsph_whole_run import make
    s = make("baseline", 4.0)
for _ in range(8):
    s.step()
torch.cuda.synchronize()
for _ in range(n):
    s.step()
torch.cuda.synchronize()
print("ok")
