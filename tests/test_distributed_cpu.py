"""CPU (gloo, world_size 2): the x-slab decomposition of distributed.py --
ghost exchange, local step on owned + ghosts sorted by global id, owned
extraction, migration -- reproduces the single-domain RTS-WCSPH run bit for
bit.  The per-rank local step here is the oracle (the B200 solver needs a
GPU; test_distributed_gpu.py runs the same protocol with it)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _scene():
    from paper_2009_14514_b200 import Scene
    # a column collapsing along x across the slab cut
    return Scene(domain_min=(0, 0, 0), domain_max=(0.6, 0.3, 0.2),
                 fluid_boxes=(((0.0, 0.0, 0.0), (0.5, 0.2, 0.2)),), spacing=0.02)


def _jitter(n, s=0.02):
    return np.random.default_rng(1234).uniform(-0.01 * s, 0.01 * s, (n, 3))


class OracleLocal:
    """Adapter: the oracle as the per-rank local step (CPU tensors)."""

    FIELDS = ("vel", "acc", "acc_prev", "force", "rho", "pres", "dt_since", "dt_corr",
              "validity", "region", "compute")

    def __init__(self, scene, mode="rts"):
        from oracle.sph import OracleWcsph
        self.o = OracleWcsph(scene, mode=mode)
        self.scene = scene

    def _fresh_state(self, pos):
        n = pos.shape[0]
        z3 = torch.zeros((n, 3), dtype=torch.float64)
        return {"pos": pos.double(), "vel": z3.clone(), "acc": z3.clone(), "acc_prev": z3.clone(),
                "force": z3.clone(), "rho": torch.full((n,), self.scene.rest_density, dtype=torch.float64),
                "pres": torch.zeros(n, dtype=torch.float64), "dt_since": torch.zeros(n, dtype=torch.float64),
                "dt_corr": torch.zeros(n, dtype=torch.float64),
                "validity": torch.zeros(n, dtype=torch.int32), "region": torch.ones(n, dtype=torch.int8),
                "compute": torch.ones(n, dtype=torch.bool)}

    def _cast_state(self, st):
        out = {k: v.double() for k, v in st.items()}
        out["validity"] = st["validity"].to(torch.int32)
        out["region"] = st["region"].to(torch.int8)
        out["compute"] = st["compute"] != 0
        return out

    def _set_local_particles(self, state, walls, capacity=None, init=False):
        o = self.o
        if walls is not None:
            self.walls = np.asarray(walls, dtype=np.float64)
        nf = 0 if state is None else state["pos"].shape[0]
        fl = np.zeros((0, 3)) if state is None else state["pos"].numpy()
        o.n_fluid = nf
        o.pos = np.concatenate([fl, self.walls])
        if state is not None:
            for k in self.FIELDS:
                v = state[k].numpy()
                setattr(o, k, v.astype({"validity": np.int32, "region": np.int8,
                                         "compute": bool}.get(k, np.float64)).copy())
        o.nbr = np.zeros((max(nf, 1), 128), dtype=np.int64)
        o.cnt = np.zeros(max(nf, 1), dtype=np.int64)

    def _get_local_state(self):
        o = self.o
        out = {"pos": torch.from_numpy(o.pos[:o.n_fluid].copy())}
        for k in self.FIELDS:
            out[k] = torch.from_numpy(np.asarray(getattr(o, k)).copy())
        return out

    def step(self):
        return self.o.step()


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_2009_14514_b200.distributed import SlabWcsph
        from paper_2009_14514_b200.scene import seed_particles
        sc = _scene()
        nf = len(seed_particles(sc)[0])
        d = SlabWcsph(sc, OracleLocal(sc), mode="rts", device="cpu", jitter=_jitter(nf))
        ncomp = []
        for _ in range(steps):
            st = d.step()
            t = torch.tensor([st.n_compute], dtype=torch.int64)
            dist.all_reduce(t)
            ncomp.append(int(t))
        q.put((rank, d.gid.numpy().copy(), d.state["pos"].numpy().copy(),
               d.state["vel"].numpy().copy(), d.state["rho"].numpy().copy(), ncomp))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_domain_bitwise(world):
    from oracle.sph import OracleWcsph
    steps = 16
    sc = _scene()
    ref = OracleWcsph(sc, mode="rts")
    nf = ref.n_fluid
    ref.pos[:nf] = (ref.pos[:nf] + _jitter(nf)).astype(np.float32).astype(np.float64)
    ref_nc = [ref.step().n_compute for _ in range(steps)]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    gid = np.concatenate([r[1] for r in res])
    pos = np.concatenate([r[2] for r in res])
    vel = np.concatenate([r[3] for r in res])
    rho = np.concatenate([r[4] for r in res])
    assert np.array_equal(np.sort(gid), np.arange(nf))  # every particle owned exactly once
    order = np.argsort(gid)
    assert np.array_equal(pos[order], ref.pos[:nf])
    assert np.array_equal(vel[order], ref.vel)
    assert np.array_equal(rho[order], ref.rho)
    assert res[0][5] == ref_nc
    # the cut actually had traffic: both ranks own particles
    assert all(len(r[1]) > 0 for r in res)


def test_rebalanced_cuts_move_toward_equal_work_one_slab_at_most():
    """SlabPartition.rebalanced: cuts at equal cumulative work, each moved by
    less than the narrower neighbouring slab (migrants only go next door)."""
    from paper_2009_14514_b200.distributed import SlabPartition
    part = SlabPartition(origin_x=0.0, inv_block=1.0, nx=40, world=4, halo=2)  # even: 10 each
    w = np.zeros(40)
    w[:10] = 10.0  # all the work in the first slab
    w[10:] = 1.0
    cuts = part.rebalanced(w)
    old = [0, 10, 20, 30, 40]
    assert cuts[0] == 0 and cuts[-1] == 40
    assert all(a < b for a, b in zip(cuts, cuts[1:]))
    for r in range(1, 4):
        shift = min(old[r] - old[r - 1], old[r + 1] - old[r]) - 1
        assert abs(cuts[r] - old[r]) <= shift
    work = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
    assert max(work) < w[:10].sum()  # the busiest slab shed work
    # repeated rebalancing converges to near-equal work
    for _ in range(6):
        part.cuts = cuts
        cuts = part.rebalanced(w)
    work = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
    assert max(work) <= 1.25 * (w.sum() / 4)
    # uniform work: the even cuts stay
    part.cuts = ()
    assert part.rebalanced(np.ones(40)) == (0, 10, 20, 30, 40)


def test_slabs_narrower_than_the_ghost_band_are_rejected():
    """a slab narrower than the ghost band would silently miss
    rows two ranks away -> ConfigError at partition time; a rebalance never
    produces one."""
    from paper_2009_14514_b200 import ConfigError
    from paper_2009_14514_b200.distributed import SlabPartition
    from paper_2009_14514_b200.scene import Scene
    sc = Scene(domain_min=(0, 0, 0), domain_max=(0.4, 0.2, 0.2),
               fluid_boxes=(((0, 0, 0), (0.4, 0.1, 0.1)),), spacing=0.02)
    # 0.4 m + walls at 2.2 s = 0.044 m blocks: 11 columns, 4 ranks x halo 6 cannot fit
    with pytest.raises(ConfigError, match="narrower than the 6-column ghost band"):
        SlabPartition.for_scene(sc, "pcisph", 4, halo=6)
    part = SlabPartition.for_scene(sc, "wcsph", 2, halo=2)
    assert min(part.widths()) >= 2
    part = SlabPartition(origin_x=0.0, inv_block=1.0, nx=12, world=3, halo=4)  # 4 | 4 | 4
    w = np.zeros(12)
    w[:4] = 100.0
    assert part.rebalanced(w) == (0, 4, 8, 12)  # any move would leave a slab < 4 wide
