"""Probe (not the bench): warm device time of the full PCISPH refresh
(rts_pci_refresh, every fluid particle: search + rows + f_ext) at the cfg2
scene, CUDA events around repeated launches on the solver stream.

    python scripts/refresh_probe.py [reps=20]      (WL=cfg2 | cfg5-pcisph ...)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
wl = os.environ.get("WL", "cfg2")
s = bench.make_device_solver("pcisph", dev, wl)
for _ in range(int(os.environ.get("MAJORS", "3"))):
    s.advance()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
s._rebuild(False)  # fresh grid + candidate copies at the current positions (a major start)
s._call("rts_pci_major_begin")
for _ in range(3):
    s._call("rts_pci_refresh", 1, 0)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(reps):
    s._call("rts_pci_refresh", 1, 0)
b.record(st)
b.synchronize()
cnt = s.cnt if hasattr(s, "cnt") else None
print(f"{wl} full refresh {a.elapsed_time(b) / reps * 1e3:9.1f} us  "
      f"(n_fluid {s.n_fluid}, mean row {float(cnt.float().mean()) if cnt is not None else -1:.1f})")
