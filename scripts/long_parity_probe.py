"""Long-horizon parity probe: cfg1 (16k RTS-WCSPH) for 2000 steps on the B200
and in the oracle from the same jittered state; prints the statistics."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from parity import apply_jitter
from oracle.sph import OracleWcsph
from paper_2009_14514_b200 import Scene, WcsphSolver
scene = Scene(domain_min=(0, 0, 0), domain_max=(1.0, 0.5, 1.0),
              fluid_boxes=(((0, 0, 0), (0.4, 0.4, 0.8)),), spacing=0.02)
dev = WcsphSolver(scene, mode="rts")
orc = OracleWcsph(scene, mode="rts")
apply_jitter(dev, orc, seed=1234)
def stats(rho, vel, mass):
    e = (rho - 1000.0) / 1000.0
    return float(e.mean()), float(e.max()), 0.5 * mass * float((vel * vel).sum())
t0 = time.time()
for k in range(1, 2001):
    dev.step(); orc.step()
    if k in (200, 500, 1000, 1500, 2000):
        a = stats(dev.host("rho"), dev.host("vel"), dev.mass)
        b = stats(orc.rho, orc.vel, orc.mass)
        print(k, f"t={dev.sim_time:.4f}", "dev", [f"{x:.5g}" for x in a], "orc", [f"{x:.5g}" for x in b],
              f"{time.time()-t0:.0f}s", flush=True)
