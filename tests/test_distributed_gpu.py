"""GPU: the B200 RTS-WCSPH solver inside the x-slab decomposition.

Two ranks on the one visible GPU (gloo transport through host memory --
the kernels of the two processes never wait on each other) must reproduce
the single-GPU run of the same scene bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _scene():
    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0, 0, 0), domain_max=(0.6, 0.3, 0.2),
                 fluid_boxes=(((0.0, 0.0, 0.0), (0.5, 0.2, 0.2)),), spacing=0.02)


def _jitter(n, s=0.02):
    return np.random.default_rng(1234).uniform(-0.01 * s, 0.01 * s, (n, 3))


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_2009_14514_b200.distributed import DistributedWcsph
        from paper_2009_14514_b200.scene import seed_particles
        sc = _scene()
        nf = len(seed_particles(sc)[0])
        d = DistributedWcsph(sc, mode="rts", device="cuda:0", jitter=_jitter(nf))
        for _ in range(steps):
            d.step()
        q.put((rank, d.gid.cpu().numpy(), d.state["pos"].cpu().numpy(),
               d.state["vel"].cpu().numpy(), d.state["rho"].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_gpu_bitwise():
    from paper_2009_14514_b200 import WcsphSolver
    steps = 12
    sc = _scene()
    ref = WcsphSolver(sc, mode="rts")
    nf = ref.n_fluid
    from paper_2009_14514_b200.scene import seed_particles
    x = (seed_particles(sc)[0] + _jitter(nf)).astype(np.float32)
    ref.pos[:nf] = torch.as_tensor(x, device=ref.device)
    for _ in range(steps):
        ref.step()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    gid = np.concatenate([r[1] for r in res])
    order = np.argsort(gid)
    assert np.array_equal(gid[order], np.arange(nf))
    assert np.array_equal(np.concatenate([r[2] for r in res])[order], ref.host("pos")[:nf])
    assert np.array_equal(np.concatenate([r[3] for r in res])[order], ref.host("vel"))
    assert np.array_equal(np.concatenate([r[4] for r in res])[order], ref.host("rho"))
