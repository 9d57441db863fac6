"""Host-side profile (cProfile) of DistributedPcisph.advance at world size 1:
where the rank driver's per-major host time goes."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2009_14514_b200.distributed import DistributedPcisph
from paper_2009_14514_b200.scene import seed_particles
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29556")
dist.init_process_group("nccl", rank=0, world_size=1)
sc = bench.scene_cfg2(1)
n = len(seed_particles(sc)[0])
d = DistributedPcisph(sc, device=torch.device("cuda", 0), jitter=bench.jitter_np(n, sc.spacing),
                      iteration_cap=50)
for _ in range(3):
    d.advance()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    d.advance()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
dist.destroy_process_group()
