"""Per-major cost of the x-slab driver at world size 1 (no peers): the
re-pack / host-driven-loop overhead of DistributedPcisph vs the graph path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2009_14514_b200.distributed import DistributedPcisph
from paper_2009_14514_b200.scene import seed_particles
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
print("backend", os.environ.get("RTS_DIST_BACKEND", "nccl"))
dist.init_process_group(os.environ.get("RTS_DIST_BACKEND", "nccl"), rank=0, world_size=1)
sc = bench.scene_cfg2(1)
n = len(seed_particles(sc)[0])
d = DistributedPcisph(sc, device=torch.device("cuda", 0), jitter=bench.jitter_np(n, sc.spacing),
                      iteration_cap=50)
for _ in range(3):
    d.advance()
torch.cuda.synchronize()
t0 = time.perf_counter()
K = 10
for _ in range(K):
    d.advance()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / K
print(f"distributed driver, world 1: {dt*1e3:.2f} ms per major")
s = d.solver
t0 = time.perf_counter()
for _ in range(K):
    s.major_step()
torch.cuda.synchronize()
print(f"host-driven major_step only: {(time.perf_counter() - t0) / K * 1e3:.2f} ms per major")

# phase breakdown of DistributedPcisph.advance
def timed(f, *a):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(*a); torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3
s = d.solver
T = {}
for _ in range(5):
    (d.gid, d.state), T["migrate"] = timed(d.driver.migrate, d.gid, d.state)
    d.state, T["cast"] = timed(s._cast_state, d.state)
    (ggid, gstate), T["ghost_rows"] = timed(d.driver.ghost_rows, d.gid, d.state)
    (allg, merged, owned), T["merged"] = timed(d.driver.merged, d.gid, d.state, ggid, gstate)
    merged, T["cast2"] = timed(s._cast_state, merged)
    _, T["set_local"] = timed(s._set_local_particles, merged, None, None, False, ~owned)
    (send, recv), T["lists"] = timed(d._lists, allg, merged, owned)
    from paper_2009_14514_b200.distributed import PcisphExchange
    s._xch = PcisphExchange(d.driver, send, recv)
    rows, T["major"] = timed(s.major_step)
    s._xch = None
    out, T["get_local"] = timed(s._get_local_state)
    def ext():
        idx = torch.nonzero(owned).reshape(-1)
        return {k: v[idx] for k, v in out.items()}, allg[idx]
    (d.state, d.gid), T["extract"] = timed(ext)
print({k: round(v, 2) for k, v in T.items()})
