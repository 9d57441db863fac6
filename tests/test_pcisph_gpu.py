"""B200 RTS-PCISPH vs the CPU oracle, plus the reference's solver-level
behaviours (pkg/tests/test_pcisph.py) run against the device solver.

Parity bar: sets, regions, validity, refresh lists and per-minor iteration
counts exact; rho*, err, p, f_p after one correction iteration from a
common state <= 1e-4 relative (BASELINE.json north_star).
"""

import dataclasses
import os

import numpy as np
import pytest
import torch

from conftest import single_particle_scene, tiny_tank
from parity import PCISPH_STATE, apply_jitter, inject, rel_err, vec_rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _pair(scene, **kw):
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    return PcisphSolver(scene, **kw), OraclePcisph(scene, **kw)


def _np(t):
    return t.detach().cpu().numpy()


def _sets_equal(dev, orc):
    for name in ("region", "validity", "compute", "in_se", "in_sob"):
        assert np.array_equal(_np(getattr(dev, name)), getattr(orc, name)), name


def test_first_iteration_parity_from_common_state():
    """rho*, err, p and f_p after one scheduled correction iteration."""
    dev, orc = _pair(tiny_tank(), mode="rts")
    apply_jitter(dev, orc)
    for _ in range(2):  # develop a non-trivial state first
        dev.advance()
    inject(dev, orc, PCISPH_STATE)
    orc.xstar[:] = dev.host("xstar")
    # major start on both
    orc.grid.rebuild(orc.pos, orc.n_fluid)
    orc._assign_major_regions(4)
    dev._prepare(dev.dt)
    dev._rebuild(True)
    dev._assign_major_regions(4, rebuilt=True)
    dev._read()
    assert np.array_equal(_np(dev.grid.order), orc.grid.order)
    assert np.array_equal(_np(dev.block_region), orc.block_region)
    _sets_equal(dev, orc)
    # refresh + one iteration with row (1, 2, 3, 4)
    k = orc.kernel
    refresh = np.flatnonzero(orc.compute).astype(np.int64)
    layers = np.where(orc.region[refresh] == 1, 2, 1).astype(np.int64)
    orc.grid.search_into(orc.pos, refresh, layers, k.h, orc.nbr, orc.cnt)
    orc._ext(refresh)
    orc.p[:] = 0.0
    orc.f_p[:] = 0.0
    dev._call("rts_pci_refresh", 0, 1)
    dev._zero_pressure()
    cnt = _np(dev.cnt)
    assert np.array_equal(cnt, orc.cnt)
    nbr = _np(dev.nbr)
    for i in range(orc.n_fluid):
        assert np.array_equal(nbr[i, : cnt[i]], orc.nbr[i, : orc.cnt[i]]), i
    assert vec_rel_err(dev.host("f_ext"), orc.f_ext) <= TOL
    # iteration 1
    orc.in_se[:] = False
    orc._refresh_observed()
    turn = np.isin(orc.region, (1, 2, 3, 4))
    pred = np.flatnonzero(turn | orc.in_se | orc.in_sob).astype(np.int64)
    force = np.flatnonzero(turn | orc.in_se).astype(np.int64)
    orc._motion(orc.dt)
    orc._density(pred)
    orc._accumulate_pressure(force, orc.delta(orc.dt))
    orc.in_se = orc.err > 0.5 * orc.scene.eta_max
    orc._refresh_observed()
    orc._pforces(force)
    dev._call("rts_pci_minor_begin", 0, 0)  # loop state: not done
    dev._call("rts_pci_observed", 0)
    dev._call("rts_pci_motion", 1)
    dev._call("rts_pci_sets", 0b11110, 0)
    dev._call("rts_pci_density")
    dev._call("rts_pci_se_reduce", 1)
    dev._call("rts_pci_pforces")
    c = dev._read()
    dev._call("rts_pci_control", 0, 0, dev.local_attempts, dev.iteration_cap)
    dev._call("rts_pci_sob")
    assert int(c.n_pred) == pred.size
    assert rel_err(dev.host("rho_star")[pred], orc.rho_star[pred]) <= TOL
    assert np.abs(dev.host("err")[pred] - orc.err[pred]).max() <= TOL
    pp = orc.p[force] > 0
    assert rel_err(dev.host("p")[force][pp], orc.p[force][pp]) <= TOL
    assert vec_rel_err(dev.host("f_p")[force], orc.f_p[force]) <= TOL
    assert np.array_equal(_np(dev.in_se), orc.in_se)
    assert np.array_equal(_np(dev.in_sob), orc.in_sob)
    assert float(c.max_err) == pytest.approx(float(orc.err.max()), rel=1e-4, abs=1e-9)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("mode", ["rts", "const"])
def test_major_step_parity_from_common_state(mode, graphs):
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    dev = PcisphSolver(tiny_tank(), mode=mode, use_graphs=graphs)
    orc = OraclePcisph(tiny_tank(), mode=mode)
    apply_jitter(dev, orc)
    for major in range(4):
        inject(dev, orc, PCISPH_STATE)
        orc.xstar[:] = dev.host("xstar")
        rd, ro = dev.advance(), orc.advance()
        assert len(rd) == len(ro)
        for a, b in zip(rd, ro):
            assert (a.n_compute, a.iterations, a.corrected, a.early_term) == \
                   (b.n_compute, b.iterations, b.corrected, b.early_term), (major, a, b)
            assert (a.iters_r1, a.iters_r2, a.iters_r3, a.iters_r4) == \
                   (b.iters_r1, b.iters_r2, b.iters_r3, b.iters_r4)
            assert a.max_err == pytest.approx(b.max_err, rel=1e-3, abs=1e-7)
        if mode == "rts":
            _sets_equal(dev, orc)
        assert np.abs(dev.host("pos")[: dev.n_fluid] - orc.pos[: orc.n_fluid]).max() < 1e-6
        assert vec_rel_err(dev.host("vel"), orc.vel) < 1e-3 or \
            np.abs(dev.host("vel") - orc.vel).max() < 1e-5


def test_pinned_regional_major_matches_const_baseline():
    from paper_2009_14514_b200 import PcisphSolver
    scene = tiny_tank(rho_T=1e-6)
    rts = PcisphSolver(scene, mode="rts", pin_region=1)
    ref = PcisphSolver(scene, mode="const", dt=rts.dt)
    minors = rts.advance()
    for _ in range(len(minors)):
        ref.sync_step()
    assert len(minors) == 4
    assert rts.sim_time == pytest.approx(ref.sim_time, rel=1e-15)
    assert bool(torch.all(rts.region == 1))
    assert np.abs(rts.host("pos") - ref.host("pos")).max() < 1e-6
    assert np.abs(rts.host("vel") - ref.host("vel")).max() < 1e-5
    assert rts.local_entered_total == 0


def test_quiet_start_assigns_the_largest_step(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts")
    s.grid.rebuild(s.pos, s.n_fluid)
    s._assign_major_regions(4)
    assert bool(torch.all(s.region == 4))
    assert bool(torch.all(s.validity == 4))
    assert bool(torch.all(s.compute))


def test_settling_tank_needs_no_per_minor_region(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts")
    s.advance()
    s.advance()
    assert int(s.particle_regions().min()) >= 2


def test_validity_countdown_drives_refresh():
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(single_particle_scene(boundary_layers=0), mode="rts")
    for _ in range(2):
        assert [m.frac_compute for m in s.advance()] == [1.0, 0.0, 0.0, 0.0]


def test_error_sets_match_thresholds(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts")
    s.advance()
    assert torch.equal(s.in_se, s.err > 0.5 * tank_scene.eta_max)


def test_average_error_is_signed_before_clamping(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="const")
    st = s.sync_step()
    expected = max(0.0, float(s.rho_star.double().mean()) / tank_scene.rest_density - 1.0)
    assert st.avg_err == pytest.approx(expected, abs=1e-9)
    assert st.avg_err == 0.0
    assert float(s.err.mean()) > 0.001


def test_isolated_particle_converges_in_minimum_iterations():
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(single_particle_scene(boundary_layers=0), mode="const")
    st = s.sync_step()
    assert st.iterations == 3 and st.corrected == 3
    assert float(s.p[0]) == 0.0
    assert st.max_err == 0.0
    assert bool(torch.all(s.f_p == 0.0))
    assert float(s.vel[0, 1]) == pytest.approx(-9.81 * s.dt, rel=1e-6)


def test_const_and_adaptive_dt_rules(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="const")
    dt0 = s.dt
    assert dt0 == pytest.approx(0.0083 * tank_scene.spacing)
    s.sync_step()
    s.sync_step()
    assert s.dt == dt0
    a = PcisphSolver(tank_scene, mode="adaptive")
    base = tank_scene.spacing * 0.0175
    assert a.dt == pytest.approx(base)
    a.vel[:] = 0.0
    a.dt = 2.0 * base
    a._adapt_dt(3)
    assert a.dt == 2.0 * base
    a._adapt_dt(9)
    assert a.dt == pytest.approx(1.6 * base)
    a.dt = 0.1 * tank_scene.const_dt()
    a._adapt_dt(9)
    assert a.dt == 0.1 * tank_scene.const_dt()


def test_local_phase_entered_under_default_threshold(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts")
    x = s.host("pos")[: s.n_fluid]
    center = int(np.abs(x - 0.12).max(axis=1).argmin())
    s.vel[center] = torch.tensor([0.0, -6.0, 0.0])
    s.advance()
    assert s.local_entered_total >= 1
    assert s.local_reverted_total <= s.local_entered_total


def test_mid_major_marking_pulls_neighborhood_down(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts")
    s.grid.rebuild(s.pos, s.n_fluid)
    s._assign_major_regions(4)
    x = s.host("pos")[: s.n_fluid]
    center = int(np.abs(x - 0.12).max(axis=1).argmin())
    s.vel[center] = torch.tensor([30.0, 0.0, 0.0])
    s._mark_timestep_updates()
    cell = int(s.grid.fluid_cells[center])
    assert int(s.block_region[cell]) == 1
    assert int(s.region[center]) == 1
    assert bool(s.compute[center])
    assert int(s.validity[center]) == 1
    assert int(torch.sum(s.block_region == 1)) == 27


def test_early_termination_halves_majors_then_recovers():
    from paper_2009_14514_b200 import PcisphSolver
    scene = tiny_tank(eta_max=1e-3)
    s = PcisphSolver(scene, mode="rts")
    minors = s.advance()
    assert minors[-1].early_term == 1
    assert len(minors) == 1
    assert s.controller.n_current == 2
    assert s.controller.recovery_left == 10
    s.scene = dataclasses.replace(scene, eta_max=1e-2)
    for _ in range(10):
        minors = s.advance()
        assert len(minors) == 2
        assert all(m.early_term == 0 for m in minors)
    assert s.controller.n_current == 4
    assert len(s.advance()) == 4


def test_unconvergable_minor_raises():
    from paper_2009_14514_b200 import NumericalError, PcisphSolver
    s = PcisphSolver(tiny_tank(eta_max=1e-9, eta_avg=1e-9), mode="rts", iteration_cap=2)
    with pytest.raises(NumericalError, match="global iterations"):
        s.advance()


def test_short_run_holds_density_and_misses_nothing(tank_scene):
    """pkg/tests/test_pcisph.py:310-319 with the device neighbour audit."""
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tank_scene, mode="rts", audit_neighbors=True)
    rows = []
    while s.sim_time < 0.05:
        rows.extend(s.advance())
    assert s.missed_neighbors_total == 0
    assert all(m.missed_neighbors == 0 for m in rows)
    clean = [m for m in rows if not m.early_term]
    assert clean
    assert all(m.max_err < tank_scene.eta_max for m in clean)
    assert all(m.avg_err < tank_scene.eta_avg for m in clean)


def test_unknown_mode_rejected(tank_scene):
    from paper_2009_14514_b200 import PcisphSolver
    with pytest.raises(ValueError, match="unknown pcisph mode"):
        PcisphSolver(tank_scene, mode="warp")


def test_audit_counts_missing_entries():
    """The audit kernel finds true neighbours that are absent from a row:
    truncate every refreshed table by one entry and count."""
    from paper_2009_14514_b200 import PcisphSolver
    s = PcisphSolver(tiny_tank(), mode="rts")
    s._prepare(s.dt)
    s._rebuild(True)
    s._assign_major_regions(4, rebuilt=True)
    s._call("rts_pci_minor_begin", 0, 0)
    s._call("rts_pci_refresh", 0, 1)
    s._audit_refresh()
    assert s.counters.read(s._stream()).missing == 0
    s._call("rts_pci_refresh", 1, 1)
    s.cnt.sub_(1)  # drop the last entry of every row
    s._audit_refresh()
    c = s.counters.read(s._stream())
    assert c.missing == s.n_fluid


@pytest.mark.skipif(not os.environ.get("RTS_SPH_LIB", "").endswith("checked.so"),
                    reason="needs the bounds-checked build (scripts/checked_build.sh)")
def test_checked_build_flags_a_corrupt_neighbour_entry():
    """The checked build's range checks fire instead of a wild access: a
    neighbour-table entry past the last particle stops the pass with
    RTS_ERR_CHECK at the density gather (site 403)."""
    from paper_2009_14514_b200 import PcisphSolver
    from paper_2009_14514_b200 import _native as N
    dev = PcisphSolver(tiny_tank(), mode="rts", use_graphs=False)
    dev.advance()
    dev._nbr[1, 5] = dev.n_fluid + dev.n_bound + 1000  # row 5, entry 1
    dev._call("rts_pci_minor_begin", 0, 0)
    dev._call("rts_pci_motion", 1)
    dev._call("rts_pci_sets", 0b11110, 0)
    dev._call("rts_pci_density")
    c = dev.counters.read(dev._stream())
    assert c.err_flags & N.ERR_CHECK and c.check_site == 403
