"""Edge cases of the device path against the oracle: coincident particles
(r = 0 pairs), a fluid-free scene (a configuration error, as in the
reference), the neighbour-table overflow error, and particles sitting
exactly on block faces (key rounding)."""

import numpy as np
import pytest
import torch

from conftest import tiny_tank
from parity import WCSPH_STATE, inject, rel_err, vec_rel_err

pytestmark = pytest.mark.gpu


def test_coincident_particles_match_oracle():
    from oracle.sph import OracleWcsph
    from paper_2009_14514_b200 import WcsphSolver
    dev, orc = WcsphSolver(tiny_tank(), mode="baseline"), OracleWcsph(tiny_tank(), mode="baseline")
    nf = dev.n_fluid
    x = orc.pos[:nf].astype(np.float32)
    x[1] = x[0]  # an exact duplicate: r = 0 pair (spiky term 0, viscosity kept)
    x[7] = x[6]
    dev.pos[:nf] = torch.as_tensor(x, device=dev.device)
    orc.pos[:nf] = x.astype(np.float64)
    for _ in range(3):
        inject(dev, orc, WCSPH_STATE)
        dev.step()
        orc.step()
        assert rel_err(dev.host("rho"), orc.rho) <= 1e-4
        assert vec_rel_err(dev.host("acc"), orc.acc) <= 1e-4
        assert np.isfinite(dev.host("pos")).all()


def test_fluid_free_scene_is_a_config_error():
    # as in the reference (scene.py validation): a scene needs a fluid box
    from paper_2009_14514_b200 import ConfigError, Scene
    with pytest.raises(ConfigError, match="no fluid_box"):
        Scene(domain_min=(0, 0, 0), domain_max=(0.3, 0.3, 0.3), fluid_boxes=(), spacing=0.02)


def test_collapsed_particles_raise_table_overflow():
    from paper_2009_14514_b200 import NumericalError, PcisphSolver
    s = PcisphSolver(tiny_tank(), mode="rts")
    nf = s.n_fluid
    # squeeze 300 fluid particles into one support radius: > 128 neighbours
    c = s.pos[:nf].mean(0)
    s.pos[:300] = c + 0.002 * torch.rand((300, 3), device=s.device)
    with pytest.raises(NumericalError, match="overflow"):
        s.advance()


def test_positions_on_block_faces_bin_exactly():
    from oracle.sph import OracleWcsph
    from paper_2009_14514_b200 import WcsphSolver
    dev, orc = WcsphSolver(tiny_tank(), mode="rts"), OracleWcsph(tiny_tank(), mode="rts")
    nf = dev.n_fluid
    bs = dev.grid.block_size
    # snap every particle onto a block face along x (exact multiples in fp32)
    x = orc.pos[:nf].astype(np.float32)
    x[:, 0] = (np.round(x[:, 0] / bs) * bs).astype(np.float32)
    dev.pos[:nf] = torch.as_tensor(x, device=dev.device)
    orc.pos[:nf] = x.astype(np.float64)
    dev.grid.rebuild(dev.pos, nf)
    orc.grid.rebuild(orc.pos, nf)
    assert np.array_equal(dev.grid.fluid_cells.cpu().numpy(), orc.grid.fluid_cells)
    assert np.array_equal(dev.grid.order.cpu().numpy(), orc.grid.order)
