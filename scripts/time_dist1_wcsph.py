"""Per-step cost of the resident x-slab RTS-WCSPH driver at world size 1
(no peers) against the graph-captured single-GPU step, cfg5 scene (4 M)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2009_14514_b200.distributed import DistributedWcsph
from paper_2009_14514_b200.scene import seed_particles
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29556")
dist.init_process_group(os.environ.get("RTS_DIST_BACKEND", "nccl"), rank=0, world_size=1)
wl = os.environ.get("RTS_WORKLOAD", "cfg5-wcsph")
sc = bench.workload_scene(wl, 1)
lat = seed_particles(sc)[0]
d = DistributedWcsph(sc, device=torch.device("cuda", 0), jitter=bench.jitter_np(len(lat), sc.spacing),
                     velocity=bench.initial_velocity(wl, lat))
for _ in range(8):
    d.step()
K = 20
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K):
    d.step()
torch.cuda.synchronize()
print(f"{wl}: distributed driver, world 1: {(time.perf_counter() - t0) / K * 1e3:.3f} ms per step")
s = bench.make_device_solver("wcsph", torch.device("cuda", 0), wl)
for _ in range(8):
    s.step()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K):
    s.step()
torch.cuda.synchronize()
print(f"{wl}: single-GPU graph step: {(time.perf_counter() - t0) / K * 1e3:.3f} ms per step")
def timed(f, *a):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(*a); torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3
T = {}
for _ in range(5):
    _, T["ghosts"] = timed(d._ghosts)
    _, T["step"] = timed(d.solver.step)
    d.solver._resize_fluid(d.n_own)
    _, T["migrate"] = timed(d._migrate)
print({k: round(v, 3) for k, v in T.items()})
