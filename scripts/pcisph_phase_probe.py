"""Probe (not the bench): warm per-entry-point device times of the cfg2 RTS-PCISPH
major step, host-driven with CUDA events around every launch, plus the graph
major time.

    python scripts/pcisph_phase_probe.py [majors=6]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

majors = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, os.environ.get("WL", "cfg2"))
for _ in range(int(os.environ.get("WARM", "3"))):
    s.advance()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(majors):
    s.advance()
b.record(st)
b.synchronize()
print(f"graph major {a.elapsed_time(b) / majors * 1e3:9.1f} us")
names = ["rts_pci_major_begin", "rts_pci_gather", "rts_block_levels", "rts_pci_major_particles",
         "rts_pci_minor_begin", "rts_pci_refresh", "rts_pci_zero_pressure", "rts_pci_observed",
         "rts_pci_motion", "rts_pci_sets", "rts_pci_density", "rts_pci_se_reduce",
         "rts_pci_pforces", "rts_pci_control", "rts_pci_integrate", "rts_block_maxima",
         "rts_pci_mark_updates", "rts_pci_minor_end"]
s.time_kernels(names)
s.use_graphs = False
for _ in range(majors):
    s.advance()
torch.cuda.synchronize()
tot = 0.0
for n in names:
    t = s.kernel_times(n)
    if t:
        tot += sum(t)
        print(f"{n:26s} {len(t) / majors:5.1f}/major {sum(t) / majors * 1e6:9.1f} us/major")
print(f"{'sum':26s} {'':11s} {tot / majors * 1e6:9.1f} us/major")
