"""Probe (not the bench): warm per-phase device times of the 1M RTS-WCSPH base
step (configs[2] geometry, calm start), each phase launched on its own
between CUDA events, plus the graph step time.

    python scripts/wcsph_phase_probe.py [steps=20]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_14514_b200 import _native as N  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
s = bench.make_device_solver("wcsph", dev)
for _ in range(8):
    s.step()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(steps):
    s.step()
b.record(st)
b.synchronize()
print(f"graph step {a.elapsed_time(b) / steps * 1e3:8.1f} us")

phases = [("keys", "rts_grid_keys", (1, 0)), ("sort", "rts_grid_sort", ()),
          ("levels", "rts_block_levels", (0,)), ("propagate", "rts_wcsph_propagate", ()),
          ("density", "rts_wcsph_density", ()), ("forces", "rts_wcsph_forces", ()),
          ("integrate", "rts_wcsph_integrate", ())]
tot = {k: 0.0 for k, *_ in phases}
for _ in range(steps):
    s._sync_params()
    p = s.params
    p.dt = s.dt_base
    s.counters.reset(st)
    for name, fn, args in phases:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        N.call(fn, p, s.arena.buf, *args, st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        tot[name] += e0.elapsed_time(e1)
    c = s.counters.read(st)
    s.grid.n_sorted = int(c.n_sorted)
for k, v in tot.items():
    print(f"{k:10s} {v / steps * 1e3:8.1f} us")
print(f"{'sum':10s} {sum(tot.values()) / steps * 1e3:8.1f} us")
