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


def _scene(width=0.6):
    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0, 0, 0), domain_max=(width, 0.3, 0.2),
                 fluid_boxes=(((0.0, 0.0, 0.0), (width - 0.1, 0.2, 0.2)),), spacing=0.02)


def _jitter(n, s=0.02):
    return np.random.default_rng(1234).uniform(-0.01 * s, 0.01 * s, (n, 3))


def _collect(q, procs, n=2):
    """Results of the n rank processes; a rank's exception fails the test at
    once (the other rank is then stuck in a collective and is terminated)."""
    res = []
    for _ in range(n):
        r = q.get(timeout=300)
        if r[0] == "error":
            for p in procs:
                p.kill()
            pytest.fail(f"rank {r[1]} raised:\n{r[2]}")
        res.append(r)
    return res


def _worker(rank, world, port, steps, q, drift=0.0, rebalance=0):
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
        vel = np.zeros((nf, 3))
        vel[:, 0] = drift
        d = DistributedWcsph(sc, mode="rts", device="cuda:0", jitter=_jitter(nf), velocity=vel,
                             balance=not rebalance, rebalance_every=rebalance)
        cuts0 = [d.part.bounds(r) for r in range(world)]
        g0 = set(d.gid.tolist())
        for _ in range(steps):
            d.step()
        q.put((rank, d.gid.cpu().numpy(), d.state["pos"].cpu().numpy(),
               d.state["vel"].cpu().numpy(), d.state["rho"].cpu().numpy(),
               len(g0 ^ set(d.gid.tolist())),
               cuts0 != [d.part.bounds(r) for r in range(world)]))
    except Exception:  # report instead of leaving the parent waiting
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        q.close()
        q.join_thread()  # flush the report before the hard exit
        os._exit(1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("steps,drift,rebalance", [(12, 0.0, 0), (40, 3.0, 0), (24, 0.0, 4)])
def test_two_ranks_on_one_gpu_match_single_gpu_bitwise(steps, drift, rebalance):
    """Owned rows of two WCSPH x-slab ranks equal the single-GPU run bit for
    bit; with a uniform +x drift (3 m/s, 1.6 cm over 40 steps) particles
    migrate across the cut, exercising hole filling and arrivals; with an
    unbalanced initial split (even columns) and rebalancing every 4 steps
    the cut moves and whole columns of particles change rank."""
    from paper_2009_14514_b200 import WcsphSolver
    sc = _scene()
    ref = WcsphSolver(sc, mode="rts")
    nf = ref.n_fluid
    from paper_2009_14514_b200.scene import seed_particles
    x = (seed_particles(sc)[0] + _jitter(nf)).astype(np.float32)
    ref.pos[:nf] = torch.as_tensor(x, device=ref.device)
    ref.vel[:, 0] = drift
    for _ in range(steps):
        ref.step()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, steps, q, drift, rebalance))
             for r in range(2)]
    for p in procs:
        p.start()
    res = _collect(q, procs)
    for p in procs:
        p.join(timeout=60)
    gid = np.concatenate([r[1] for r in res])
    order = np.argsort(gid)
    assert np.array_equal(gid[order], np.arange(nf))
    assert np.array_equal(np.concatenate([r[2] for r in res])[order], ref.host("pos")[:nf])
    assert np.array_equal(np.concatenate([r[3] for r in res])[order], ref.host("vel"))
    assert np.array_equal(np.concatenate([r[4] for r in res])[order], ref.host("rho"))
    if drift or rebalance:
        assert sum(r[5] for r in res) > 0, "no particle migrated"
    assert all(r[6] for r in res) == bool(rebalance)


def _pworker(rank, world, port, majors, q, width=0.6, drift=0.0, rebalance=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_2009_14514_b200.distributed import DistributedPcisph
        from paper_2009_14514_b200.scene import seed_particles
        sc = _scene(width)
        nf = len(seed_particles(sc)[0])
        vel = np.zeros((nf, 3))
        vel[:, 0] = drift
        d = DistributedPcisph(sc, device="cuda:0", jitter=_jitter(nf) * 0.2, velocity=vel,
                              balance=not rebalance, rebalance_every=rebalance)
        cuts0 = [d.part.bounds(r) for r in range(world)]
        g0 = set(d.gid.tolist())
        stats = []
        for _ in range(majors):
            stats += [(r.n_compute, r.iterations, r.corrected, r.early_term) for r in d.advance()]
        q.put((rank, d.gid.cpu().numpy(), d.state["pos"].cpu().numpy(),
               d.state["rho_star"].cpu().numpy(), stats, d._single_round(),
               len(g0 ^ set(d.gid.tolist())),
               cuts0 != [d.part.bounds(r) for r in range(world)]))
    except Exception:  # report instead of leaving the parent waiting
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        q.close()
        q.join_thread()  # flush the report before the hard exit
        os._exit(1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("width,one_round,drift,rebalance",
                         [(0.6, False, 0.0, 0), (1.0, True, 2.5, 0), (1.0, True, 0.0, 2)])
def test_pcisph_two_ranks_on_one_gpu_match_single_gpu(width, one_round, drift, rebalance):
    """RTS-PCISPH over two x-slabs (per-iteration ghost x*/p/err exchange and
    all-reduced convergence scalars) takes the single-GPU run's decisions
    (refresh counts, iterations, corrected work per minor step) and stays
    within fp32 rounding of its trajectory -- with the two-round major-start
    exchange (slabs of 7 columns, halo 6) and the single round (12 columns,
    with a +x drift of 2.5 m/s over 7 majors so that particles migrate across
    the cut; and from an even-column split rebalanced by work every 2 majors)."""
    from paper_2009_14514_b200 import PcisphSolver
    from paper_2009_14514_b200.scene import seed_particles
    majors = 7 if drift else (5 if rebalance else 3)
    sc = _scene(width)
    ref = PcisphSolver(sc, mode="rts")
    nf = ref.n_fluid
    x = (seed_particles(sc)[0] + _jitter(nf) * 0.2).astype(np.float32)
    ref.pos[:nf] = torch.as_tensor(x, device=ref.device)
    ref.xstar[:] = ref.pos[:nf]
    ref.vel[:, 0] = drift
    rstats = []
    for _ in range(majors):
        rstats += [(r.n_compute, r.iterations, r.corrected, r.early_term) for r in ref.advance()]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pworker, args=(r, 2, port, majors, q, width, drift,
                                                           rebalance)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(_collect(q, procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    assert res[0][5] == one_round and res[1][5] == one_round
    if drift or rebalance:
        assert res[0][6] + res[1][6] > 0, "no particle migrated"
    assert res[0][7] == res[1][7] == bool(rebalance)
    assert res[0][4] == rstats and res[1][4] == rstats
    gid = np.concatenate([r[1] for r in res])
    order = np.argsort(gid)
    assert np.array_equal(gid[order], np.arange(nf))
    pos = np.concatenate([r[2] for r in res])[order]
    assert np.abs(pos - ref.host("pos")[:nf]).max() < 1e-5
    rho = np.concatenate([r[3] for r in res])[order]
    assert np.abs(rho - ref.host("rho_star")).max() / 1000.0 < 1e-5


def _cworker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
        from paper_2009_14514_b200.distributed import DistributedPcisph, DistributedWcsph
        sc = _scene()
        w = WcsphSolver(sc, "rts", comm=dist.group.WORLD, device="cuda:0")
        p = PcisphSolver(sc, mode="rts", comm=dist.group.WORLD, device="cuda:0")
        assert isinstance(w, DistributedWcsph) and isinstance(p, DistributedPcisph)
        for _ in range(steps):
            w.advance()
        rows = p.advance()
        q.put((rank, w.gid.cpu().numpy(), w.pos.cpu().numpy(), w.n_fluid, w.step_index,
               [(r.n_compute, r.iterations) for r in rows]))
    except Exception:  # report instead of leaving the parent waiting
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        q.close()
        q.join_thread()
        os._exit(1)
    finally:
        dist.destroy_process_group()


def test_comm_keyword_makes_the_solvers_x_slab_ranks():
    """``WcsphSolver(..., comm=WORLD)`` / ``PcisphSolver(..., comm=WORLD)`` (the
    drop-in's extra keyword) run as x-slab ranks; their owned rows
    reproduce the single-GPU run."""
    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    steps = 6
    sc = _scene()
    ref = WcsphSolver(sc, mode="rts")
    for _ in range(steps):
        ref.step()
    pref = PcisphSolver(sc, mode="rts")
    prows = [(r.n_compute, r.iterations) for r in pref.advance()]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cworker, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = _collect(q, procs)
    for p in procs:
        p.join(timeout=60)
    gid = np.concatenate([r[1] for r in res])
    order = np.argsort(gid)
    assert np.array_equal(gid[order], np.arange(ref.n_fluid))
    assert sum(r[3] for r in res) == ref.n_fluid
    assert np.array_equal(np.concatenate([r[2] for r in res])[order], ref.host("pos")[:ref.n_fluid])
    assert all(r[4] == steps for r in res)
    assert all(r[5] == prows for r in res)
