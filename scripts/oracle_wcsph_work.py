"""Probe (CPU, the oracle = the reference's algorithm): particle updates per
simulated time of RTS-WCSPH against the global baseline at dt_cap = 4 dt_base
and dt_cap = dt_base, on the configs[2] dam break at a coarse spacing, from
t = 0 to T.  Shows that the RTS/adaptive work ratio is a property of the
algorithm, not of the B200 implementation.

    python scripts/oracle_wcsph_work.py [spacing=0.04] [T=0.5]
"""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.sph import OracleWcsph  # noqa: E402
from paper_2009_14514_b200 import Scene  # noqa: E402

sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.04
T = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
sc = Scene(domain_min=(0, 0, 0), domain_max=(2.5, 1.25, 2.5),
           fluid_boxes=(((0, 0, 0), (1, 1, 1)),), spacing=sp,
           sound_speed=10 * math.sqrt(2 * 9.81))
for mode, cap in (("rts", 1.0), ("baseline", 4.0), ("baseline", 1.0)):
    o = OracleWcsph(sc, mode=mode)
    o.dt_cap = cap * o.dt_base
    nf = o.n_fluid
    o.pos[:nf] += np.random.default_rng(7).uniform(-0.01 * sp, 0.01 * sp, (nf, 3))
    t, k, upd, t0 = 0.0, 0, 0, time.time()
    while t < T:
        st = o.step()
        t += st.dt
        k += 1
        upd += st.n_compute
    print(mode, cap, f"n_fluid {nf} steps {k} updates per particle per dt_base "
          f"{upd / nf / (t / o.dt_base):.3f} wall {time.time() - t0:.1f}s", flush=True)
