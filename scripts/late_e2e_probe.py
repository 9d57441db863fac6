"""Probe (not the bench): per-major wall time late in the cfg2 run (after
WARM majors), advance() alone vs with the host round trip of pos+vel
(download after, upload before; back to back), alternating blocks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 136
dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, "cfg2")
for _ in range(warm):
    s.advance()
nf = s.n_fluid
hp = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hv = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hp.copy_(s.pos[:nf])
hv.copy_(s.vel)
torch.cuda.synchronize()
for rep in range(2):
    for mode in ("advance", "e2e"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            if mode == "e2e":
                s.pos[:nf].copy_(hp, non_blocking=True)
                s.vel.copy_(hv, non_blocking=True)
            s.advance()
            if mode == "e2e":
                hp.copy_(s.pos[:nf], non_blocking=True)
                hv.copy_(s.vel, non_blocking=True)
        torch.cuda.synchronize()
        print(f"warm {warm} {mode:8s} {(time.perf_counter() - t0) / 5 * 1e3:7.3f} ms/major", flush=True)
