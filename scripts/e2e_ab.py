"""Probe (not the bench): e2e step time of cfg2 majors with the host round
trip back to back (chunks 0) or chunked with the two PCIe directions
overlapped (bench.HostRoundTrip), alternating on one solver."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, os.environ.get("WL", "cfg2"))
for _ in range(3):
    s.advance()
nf = s.n_fluid
hp = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hv = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hp.copy_(s.pos[:nf])
hv.copy_(s.vel)
rt = bench.HostRoundTrip(dev)
torch.cuda.synchronize()
for rep in range(3):
    for ch in (0, 1, 2, 4, 8):
        k = 6
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.upload((s.pos[:nf], s.vel), (hp, hv))
        for j in range(k):
            s.advance()
            if j + 1 < k:
                rt.round_trip((s.pos[:nf], s.vel), (hp, hv), chunks=ch)
            else:
                rt.download((s.pos[:nf], s.vel), (hp, hv))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / k
        print(f"rep {rep} chunks {ch}: {dt * 1e3:7.3f} ms per e2e major", flush=True)
