"""Probe (not the bench): device time of the major-step start of cfg2 RTS-PCISPH
(counters reset + grid keys + grid sort + candidate gather; block levels;
major particles) with CUDA events, after warm majors."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_14514_b200 import _native as N  # noqa: E402

dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, os.environ.get("WL", "cfg2"))
for _ in range(int(os.environ.get("MAJORS", "3"))):
    s.advance()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
p = s.params
reps = 20


def timed(label, fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    print(f"{label:34s} {a.elapsed_time(b) / reps * 1e3:8.1f} us", flush=True)


buf = s.arena.buf
timed("counters reset", lambda: s.counters.reset(st))
timed("grid keys (+ maxima)", lambda: N.call("rts_grid_keys", p, buf, 1, 1, st.cuda_stream))
timed("keys + sort", lambda: (s.counters.reset(st), s.grid.launch_rebuild(p, st, want_maxima=True, add_fp=True)))
timed("rebuild + gather (_rebuild)", lambda: s._rebuild(True))
timed("block levels", lambda: s._call("rts_block_levels", 1))
timed("major particles", lambda: s._call("rts_pci_major_particles"))
timed("major begin", lambda: s._call("rts_pci_major_begin"))
