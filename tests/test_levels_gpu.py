"""B200 region fields vs the oracle on random block maxima (the reference's
acceptance C5 idea, test_acceptance.py:235-263): assign_regions, smoothing,
fast-region expansion and observed blocks must be bit-exact."""

import numpy as np
import pytest
import torch

from conftest import tiny_tank

pytestmark = pytest.mark.gpu


def _fields(dev, rng, occ_frac):
    nc = dev.grid.n_cells
    occ = rng.random(nc) < occ_frac
    # velocities/forces straddling the level thresholds of the tiny tank
    v = np.where(occ, rng.choice([0.0, 0.05, 0.3, 1.0, 3.0, 8.0, 30.0], nc) * rng.uniform(0.5, 1.5, nc), 0.0)
    f = np.where(occ, rng.choice([0.0, 0.01, 0.1, 1.0, 10.0], nc) * rng.uniform(0.5, 1.5, nc), 0.0)
    return occ, v, f


@pytest.mark.parametrize("mode", ["pcisph", "wcsph"])
def test_levels_bit_exact_on_random_fields(mode):
    from oracle import sph as O
    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    rng = np.random.default_rng(5)
    if mode == "pcisph":
        dev = PcisphSolver(tiny_tank(), mode="rts")
    else:
        dev = WcsphSolver(tiny_tank(), mode="rts")
    dims = dev.grid.dims
    A = dev.arena
    p = dev.params
    for trial in range(25):
        occ, v, f = _fields(dev, rng, rng.uniform(0.2, 0.9))
        A["cell_count"].copy_(torch.as_tensor(occ.astype(np.int32)))
        A["vmax"].copy_(torch.as_tensor(v))
        A["fmax"].copy_(torch.as_tensor(f))
        n_max = int(rng.integers(2, 5))
        p.n_max = n_max
        dev._launch("rts_block_levels", 1 if mode == "pcisph" else 0)
        got = A["block_field"].cpu().numpy()
        raw = O.assign_regions(v, f, occ, dt_base=p.dt_base, block_size=p.block_size,
                               particle_mass=p.mass, sound_speed=p.sound_speed,
                               lambda_v=p.lambda_v, lambda_f=p.lambda_f, alpha=p.alpha,
                               betas=dev.betas, n_max=n_max,
                               use_sound_criterion=(mode == "wcsph"))
        assert np.array_equal(A["block_raw"].cpu().numpy(), raw), trial
        sm, _ = O.smooth_regions(raw, dims)
        want = O.expand_fast_regions(sm, dims) if mode == "pcisph" else sm
        assert np.array_equal(got, want), trial
        if mode == "pcisph":
            dev._launch("rts_pci_observed", 0)
            obs = A["block_tmp"].cpu().numpy().astype(bool)
            assert np.array_equal(obs, O.derive_observed(want, dims, np.zeros(len(want), bool)))


@pytest.mark.parametrize("mode", ["wcsph", "pcisph"])
def test_block_maxima_bit_exact(mode):
    """Per-block max |v| and |F| (grid.py:347-351; PCISPH: |f_ext + f_p|,
    pcisph.py:738-740) from a common state: fp64, bit-exact."""
    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    from parity import apply_jitter
    rng = np.random.default_rng(11)
    if mode == "pcisph":
        from oracle.sph import OraclePcisph
        dev, orc = PcisphSolver(tiny_tank(), mode="rts"), OraclePcisph(tiny_tank(), mode="rts")
    else:
        from oracle.sph import OracleWcsph
        dev, orc = WcsphSolver(tiny_tank(), mode="rts"), OracleWcsph(tiny_tank(), mode="rts")
    apply_jitter(dev, orc, seed=9)
    nf = dev.n_fluid
    vel = rng.normal(0.0, 0.5, (nf, 3)).astype(np.float32)
    fe = rng.normal(0.0, 0.1, (nf, 3)).astype(np.float32)
    dev.vel.copy_(torch.as_tensor(vel))
    orc.vel[:] = vel
    if mode == "pcisph":
        fp = rng.normal(0.0, 0.05, (nf, 3)).astype(np.float32)
        dev.f_ext.copy_(torch.as_tensor(fe))
        dev.f_p.copy_(torch.as_tensor(fp))
        force = fe.astype(np.float64) + fp.astype(np.float64)
    else:
        dev.force.copy_(torch.as_tensor(fe))
        force = fe.astype(np.float64)
    st = torch.cuda.current_stream(dev.device)
    dev._sync_params()
    dev.grid.launch_rebuild(dev.params, st, want_maxima=True, add_fp=(mode == "pcisph"))
    orc.grid.rebuild(orc.pos, orc.n_fluid)
    v_ref = orc.grid.reduce_fluid_max(np.linalg.norm(vel.astype(np.float64), axis=1))
    f_ref = orc.grid.reduce_fluid_max(np.linalg.norm(force, axis=1))
    got_v = dev.arena["vmax"].cpu().numpy().reshape(-1)
    got_f = dev.arena["fmax"].cpu().numpy().reshape(-1)
    assert np.array_equal(got_v, np.asarray(v_ref).reshape(-1))
    assert np.array_equal(got_f, np.asarray(f_ref).reshape(-1))
    if mode == "pcisph":  # the mid-major pass (rts_block_maxima, add_fp)
        dev.arena["vmax"].zero_()
        dev.arena["fmax"].zero_()
        dev._call("rts_block_maxima", 1)
        assert np.array_equal(dev.arena["vmax"].cpu().numpy().reshape(-1),
                              np.asarray(v_ref).reshape(-1))
        assert np.array_equal(dev.arena["fmax"].cpu().numpy().reshape(-1),
                              np.asarray(f_ref).reshape(-1))
