"""Long-horizon stability probe on the bench scenes: cfg2 (1M RTS-PCISPH) for
500 majors (2000 minor steps) and cfg3 (1M RTS-WCSPH) for 4000 base steps;
prints iterations, error maxima, escapes and wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev)
t0 = time.perf_counter()
rows = []
for _ in range(500):
    rows += s.advance()
torch.cuda.synchronize()
print(f"pcisph: {len(rows)} minors, sim {s.sim_time:.4f} s, wall {time.perf_counter()-t0:.2f} s, "
      f"max iters {max(r.iterations for r in rows)}, early {sum(r.early_term for r in rows)}, "
      f"worst max_err {max(r.max_err for r in rows):.4%}, mean iters "
      f"{sum(r.iterations for r in rows)/len(rows):.2f}, finite {bool(torch.isfinite(s.pos).all())}")
del s
w = bench.make_device_solver("wcsph", dev)
t0 = time.perf_counter()
fr = 0.0
for _ in range(4000):
    fr += w.step().frac_compute
torch.cuda.synchronize()
rho = w.rho.double()
print(f"wcsph: 4000 steps, sim {w.sim_time:.4f} s, wall {time.perf_counter()-t0:.2f} s, "
      f"mean active {fr/4000:.3f}, rho err mean {float((rho/1000-1).mean()):.4%} max "
      f"{float((rho/1000-1).max()):.4%}, finite {bool(torch.isfinite(w.pos).all())}")
