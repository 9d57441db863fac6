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
from paper_2009_14514_b200.distributed import PcisphExchange
T = {}
for _ in range(5):
    _, T["migrate"] = timed(d._migrate)
    _, T["ghosts"] = timed(d._ghosts)
    (send, recv), T["lists"] = timed(d._lists)
    s._xch = PcisphExchange(d.driver, send, recv)
    rows, T["major"] = timed(s.major_step)
    s._xch = None
print({k: round(v, 2) for k, v in T.items()})
