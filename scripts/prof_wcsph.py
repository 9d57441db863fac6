"""Profiling driver: 1M RTS-WCSPH (configs[2] geometry), a few warm steps then N steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
s = bench.make_device_solver("wcsph", torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for _ in range(8):
    s.step()
torch.cuda.synchronize()
for _ in range(n):
    s.step()
torch.cuda.synchronize()
print("ok")
