"""Probe (not the bench): host time between the end of one major's read-back
and the next major's graph launch in PcisphSolver.advance() (the GPU idles
through it), and where advance() spends it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_14514_b200 import _native as N  # noqa: E402
from paper_2009_14514_b200 import pcisph as P  # noqa: E402

dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, "cfg2")
for _ in range(3):
    s.advance()
torch.cuda.synchronize()
T = {"launch": [], "read_begin": [], "read_end": [], "adv_begin": [], "adv_end": []}
orig_call = N.call


def call(name, *a):
    if name == "rts_graph_launch":
        T["launch"].append(time.perf_counter_ns())
    return orig_call(name, *a)


P.N.call = call
orig_read = s._read_control


def read():
    T["read_begin"].append(time.perf_counter_ns())
    r = orig_read()
    T["read_end"].append(time.perf_counter_ns())
    return r


s._read_control = read
for _ in range(20):
    T["adv_begin"].append(time.perf_counter_ns())
    s.advance()
    T["adv_end"].append(time.perf_counter_ns())
k = 20
us = lambda v: sum(v) / len(v) / 1e3  # noqa: E731
print(f"advance() entry -> graph launch call: {us([T['launch'][i] - T['adv_begin'][i] for i in range(k)]):7.1f} us")
print(f"graph launch call -> read-back begin: {us([T['read_begin'][i] - T['launch'][i] for i in range(k)]):7.1f} us")
print(f"read-back (waits for the GPU):        {us([T['read_end'][i] - T['read_begin'][i] for i in range(k)]):7.1f} us")
print(f"read-back end -> advance() return:    {us([T['adv_end'][i] - T['read_end'][i] for i in range(k)]):7.1f} us")
print(f"read-back end -> next graph launch:   {us([T['launch'][i + 1] - T['read_end'][i] for i in range(k - 1)]):7.1f} us")
