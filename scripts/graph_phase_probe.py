"""Probe (not the bench): where the whole-major CUDA graph spends its time,
from the in-graph %globaltimer stamps of every minor step (StepStats
t_neighbor = refresh phase, t_physics = correction loop, t_rts =
integrate + mid-major marking) over warm graph-mode majors.

    python scripts/graph_phase_probe.py [majors=20] [warm=3]   (WL=cfg2 ...)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

majors = int(sys.argv[1]) if len(sys.argv) > 1 else 20
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, os.environ.get("WL", "cfg2"))
for _ in range(warm):
    s.advance()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
tn = tp = tr = 0.0
its = minors = 0
corr = 0
per = [[0.0, 0.0, 0.0, 0, 0] for _ in range(8)]  # by minor index: refresh, loop, tail, its, n
between = []  # last minor's end of major k -> first minor's begin of major k+1 (ns)
prev_end = None
a.record(st)
for _ in range(majors):
    rows_k = s.advance()
    ctl = s._ctl_cache
    if prev_end is not None:
        between.append(ctl.stats[0].t_begin - prev_end)
    prev_end = ctl.stats[len(rows_k) - 1].t_end
    for m, r in enumerate(rows_k):
        q = per[m]
        q[0] += r.t_neighbor
        q[1] += r.t_physics
        q[2] += r.t_rts
        q[3] += r.iterations
        q[4] += 1
        tn += r.t_neighbor
        tp += r.t_physics
        tr += r.t_rts
        its += r.iterations
        corr += r.corrected
        minors += 1
b.record(st)
b.synchronize()
tot = a.elapsed_time(b) * 1e-3
us = 1e6 / majors
print(f"major {tot * us:8.1f} us  (minors {minors / majors:.2f}, iterations/minor {its / max(minors, 1):.2f}, "
      f"corrected/minor/nf {corr / max(minors, 1) / s.n_fluid:.3f})")
print(f"  refresh phase {tn * us:8.1f} us   loop {tp * us:8.1f} us ({tp * 1e6 / max(its, 1):.1f} us/iteration)"
      f"   integrate+marking {tr * us:8.1f} us   rest (rebuild, levels, host) {(tot - tn - tp - tr) * us:8.1f} us")
for m, q in enumerate(per):
    if q[4]:
        n = q[4]
        print(f"  minor {m}: refresh {q[0] / n * 1e6:7.1f} us  loop {q[1] / n * 1e6:7.1f} us "
              f"({q[3] / n:.2f} it)  tail {q[2] / n * 1e6:6.1f} us")
if between:
    print(f"  between majors (end of the last minor -> begin of the next major's first minor: "
          f"host gap + rebuild + levels): {sum(between) / len(between) / 1e3:7.1f} us")
