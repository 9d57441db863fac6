"""Probe (not the bench): does particle order cost locality late in the run?
After WARM cfg2 majors, a second solver is seeded with the same state with
its particles renumbered in CSR (block) order; both then run the same
majors and their graph-mode major times are compared.

    python scripts/reorder_probe.py [warm=100] [majors=10]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 100
majors = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
a = bench.make_device_solver("pcisph", dev, "cfg2")
for _ in range(warm):
    a.advance()
torch.cuda.synchronize()
nf = a.n_fluid
order = a.grid.order.long()
perm = order[order < nf]  # fluid particles in CSR order
assert perm.numel() == nf
b = bench.make_device_solver("pcisph", dev, "cfg2")
b.pos[:nf] = a.pos[:nf][perm]
b.vel[:] = a.vel[perm]
b.xstar[:] = b.pos[:nf]
b.controller.n_current = a.controller.n_current
b.controller.recovery_left = a.controller.recovery_left
b.dt = a.dt
torch.cuda.synchronize()


def run(s, k):
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    m = 0
    for _ in range(k):
        m += len(s.advance())
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k, m


b.advance()  # build graphs
for rep in range(2):
    ta, ma = run(a, majors)
    tb, mb = run(b, majors)
    print(f"warm {warm}: particle order {ta:8.1f} us/major ({ma} minors)   CSR order {tb:8.1f} us/major ({mb} minors)", flush=True)
