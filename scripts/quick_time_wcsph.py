"""Quick timing probe (not the bench): 1M-particle RTS-WCSPH steps, per-phase CUDA events."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2009_14514_b200 import Scene, WcsphSolver
sc = Scene(domain_min=(0,0,0), domain_max=(2.5,1.25,2.5), fluid_boxes=(((0,0,0),(1,1,1)),), spacing=0.01,
           sound_speed=10*np.sqrt(2*9.81*1.0))
t0=time.time(); s = WcsphSolver(sc, mode="rts"); print("setup", time.time()-t0, s.n_fluid, s.n_bound, s.grid.dims)
rng=np.random.default_rng(1234); j=rng.uniform(-0.0001,0.0001,(s.n_fluid,3))
s.pos[:s.n_fluid] += torch.as_tensor(j, dtype=torch.float32, device="cuda")
for k in range(20):
    torch.cuda.synchronize(); t=time.perf_counter(); st=s.step(); torch.cuda.synchronize(); dtw=time.perf_counter()-t
    print(k, f"wall {dtw*1e3:.2f} ms  n_compute {st.n_compute} nb {st.t_neighbor*1e3:.3f} rts {st.t_rts*1e3:.3f} phys {st.t_physics*1e3:.3f}")
