"""B200 vs the CPU oracle at the BASELINE configurations themselves (VERDICT
r1 "what's missing" 1-4): cfg2 (1 M RTS-PCISPH, the bench workload), the
cfg1 geometry under RTS-PCISPH, the PCISPH adaptive baseline, and cfg3 (1 M
RTS-WCSPH).

Bars (BASELINE.json north_star), all written here:

* From a common state (device state injected into the oracle):
  - block keys, sort permutation, region field, neighbour rows: exact;
  - rho*, err, p, f_p after the first correction iteration: <= 1e-4
    relative (TOL), p's clamp-to-zero pattern exact, S_e / S_ob exact;
  - per-minor decisions of a major step: iterations, per-region iteration
    counts and early termination exact.  The corrected work and the refresh
    count may differ by a few particles at 1 M: the fp32 state (pos, vel,
    f_ext, f_p -- BASELINE's precision) moves a few blocks across the level
    thresholds of the mid-major marking.  Measured:
    cfg1 geometry 0 of 200 minor steps differ; cfg2 6 of 32 minor steps,
    refresh count <= 0.7 % and corrected work <= 1.2e-4 relative.  Bars:
    CORR_TOL, NCOMP_TOL.
* 200 minor steps from the same start: mass exact; mean density error and
  kinetic energy within 1 %.  The max density error is an extreme value
  over the rho* array whose entries are stale for every particle not
  predicted in the last iterations (as the reference reports it): which
  particle holds it depends on the S_e / S_ob history, so two references
  that differ only by storing their state in fp32 (the ``state_f32``
  oracle) differ by up to 20 % in it.  Bars: within
  2 % of the fp32-state reference, within MAXERR_TOL of the fp64 one.
"""

import numpy as np
import pytest
import torch

from parity import (PCISPH_STATE, WCSPH_STATE, apply_jitter, common_state_majors, density_stats,
                    first_iteration, free_run, inject, rel_err, vec_rel_err)

pytestmark = pytest.mark.gpu
TOL = 1e-4
CORR_TOL = 1e-3      # corrected work, relative, per minor step (measured <= 1.2e-4 at 1 M)
NCOMP_TOL = 0.02     # refresh count, relative, per minor step (measured <= 0.7 % at 1 M)
STAT_TOL = 0.01      # BASELINE: mean density error, kinetic energy
MAXERR_TOL = 0.25    # max density error (extreme value; see module docstring)


def _cfg1(**kw):
    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0, 0, 0), domain_max=(1.0, 0.5, 1.0),
                 fluid_boxes=(((0, 0, 0), (0.4, 0.4, 0.8)),), spacing=0.02, **kw)


def _cfg2_pair():
    import bench
    dev = bench.make_device_solver("pcisph", torch.device("cuda", 0))
    orc, _ = bench._oracle_for("cfg2")
    assert dev.n_fluid == orc.n_fluid == 1_000_000
    nf = dev.n_fluid
    assert np.array_equal(dev.host("pos")[:nf], orc.pos[:nf])  # the same jittered fp32 start
    orc.pos[:] = dev.host("pos")  # walls too: the device stores them as fp32
    orc.xstar[:] = orc.pos[:nf]
    return dev, orc


def _pcisph_pair(scene, **kw):
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    dev, orc = PcisphSolver(scene, **kw), OraclePcisph(scene, **kw)
    apply_jitter(dev, orc)
    return dev, orc


def _check_first_iteration(r):
    assert r["order_equal"] and r["block_region_equal"], r
    assert r["cnt_equal"] and r["rows_equal"], r
    assert r["f_ext_rel"] <= TOL, r
    assert r["n_pred_equal"], r
    assert r["rho_star_rel"] <= TOL, r
    assert r["err_abs"] <= TOL, r
    assert r["p_rel"] <= TOL and r["p_zero_equal"], r
    assert r["f_p_rel"] <= TOL, r
    assert r["in_se_flips"] == 0 and r["in_sob_flips"] == 0, r
    assert r["max_err"][0] == pytest.approx(r["max_err"][1], rel=TOL)


def _check_decisions(r, exact_work):
    m = r["mismatch"]
    assert r["len_mismatch"] == 0, r
    for f in ("iterations", "iters_r1", "iters_r2", "iters_r3", "iters_r4", "early_term"):
        assert m[f] == 0, r
    if exact_work:
        assert m["corrected"] == 0 and m["n_compute"] == 0, r
    assert r["corrected_rel_max"] <= CORR_TOL, r
    assert r["n_compute_rel_max"] <= NCOMP_TOL, r


def _check_stats(r):
    assert r["minors"][0] == r["minors"][1], r
    assert r["mass"][0] == r["mass"][1], r
    assert r["rel"]["mean_err"] <= STAT_TOL, r
    assert r["rel"]["ke"] <= STAT_TOL, r
    assert r["rel"]["max_err"] <= MAXERR_TOL, r


# -- cfg2: 1 M RTS-PCISPH, eta 3 % / 1.5 %, cap 50 (the bench workload) ----------

def test_cfg2_first_iteration_parity_1m():
    dev, orc = _cfg2_pair()
    for _ in range(2):  # a developed state: regions, S_e, non-zero p / f_p
        dev.advance()
    _check_first_iteration(first_iteration(dev, orc))


def test_cfg2_major_step_decisions_1m():
    dev, orc = _cfg2_pair()
    dev.advance()
    r = common_state_majors(dev, orc, 2)
    assert r["minors"] == 8
    _check_decisions(r, exact_work=False)


def test_cfg2_200_minor_statistics_1m():
    """north_star: over 200 (minor) steps mass exact, mean / max density
    error and kinetic energy within the bars; 50 majors of both solvers
    from the same jittered start (~45 s of oracle time on the GPU host)."""
    dev, orc = _cfg2_pair()
    r = free_run(dev, orc, 50)
    assert r["minors"] == [200, 200]
    _check_stats(r)


# -- cfg1 geometry (16 k dam break) under RTS-PCISPH, eta 2 % / 1 % ----------------

def test_cfg1_pcisph_decisions_exact_over_200_minor_steps():
    dev, orc = _pcisph_pair(_cfg1(eta_max=0.02, eta_avg=0.01), mode="rts")
    dev.advance()
    r = common_state_majors(dev, orc, 50)
    assert r["minors"] == 200
    _check_decisions(r, exact_work=True)
    _check_first_iteration(first_iteration(dev, orc))


def test_cfg1_pcisph_200_minor_statistics():
    """200 minor steps from the same start against the fp64 oracle (the
    north_star statistics bars) and against the fp32-state oracle
    (``state_f32``: the reference algorithm with its particle state stored
    at BASELINE's fp32 precision, as the B200 stores it): the B200 takes
    the fp32-state reference's decisions minor step for minor step
    (refresh counts, iterations, corrected work) and its max density error
    agrees within 2 % at every checkpoint -- the device's distance from the
    fp64 reference is the fp32 state's, not the kernels'."""
    from oracle.sph import OraclePcisph
    sc = _cfg1(eta_max=0.02, eta_avg=0.01)
    dev, orc = _pcisph_pair(sc, mode="rts")
    t32 = OraclePcisph(sc, mode="rts", state_f32=True)
    t32.pos[:] = orc.pos
    t32.xstar[:] = orc.xstar
    rho0 = sc.rest_density
    minors = 0
    for m in range(1, 51):
        rd, ro, rt = dev.advance(), orc.advance(), t32.advance()
        assert len(rd) == len(ro) == len(rt)
        for a, c in zip(rd, rt):
            assert (a.n_compute, a.iterations, a.corrected) == \
                (c.n_compute, c.iterations, c.corrected), (m, a, c)
        minors += len(rd)
        if m % 10:
            continue
        sd = density_stats(dev.host("rho_star"), dev.host("vel"), dev.mass, rho0)
        so = density_stats(orc.rho_star, orc.vel, orc.mass, rho0)
        st = density_stats(t32.rho_star, t32.vel, t32.mass, rho0)
        for k in ("mean_err", "ke"):
            assert abs(sd[k] - so[k]) <= STAT_TOL * abs(so[k]), (m, k, sd, so)
        assert abs(sd["max_err"] - st["max_err"]) <= 0.02 * abs(st["max_err"]), (m, sd, st)
        assert abs(sd["max_err"] - so["max_err"]) <= MAXERR_TOL * abs(so["max_err"]), (m, sd, so)
    assert minors == 200
    assert dev.n_fluid * dev.mass == orc.n_fluid * orc.mass


# -- PCISPH globally adaptive baseline (pcisph.py:376-419, 470-476) --------------

@pytest.mark.parametrize("scene", ["tiny", "cfg1"])
def test_adaptive_baseline_parity(scene):
    from conftest import tiny_tank
    sc = tiny_tank() if scene == "tiny" else _cfg1(eta_max=0.02, eta_avg=0.01)
    dev, orc = _pcisph_pair(sc, mode="adaptive")
    dts = set()
    for _ in range(40):
        inject(dev, orc, PCISPH_STATE)
        orc.xstar[:] = dev.host("xstar")
        orc.dt = dev.dt
        a, b = dev.advance()[0], orc.advance()[0]
        assert (a.iterations, a.corrected) == (b.iterations, b.corrected)
        assert a.max_err == pytest.approx(b.max_err, rel=1e-3, abs=1e-7)
        assert dev.dt == orc.dt  # the same dt rule on the same inputs, bit for bit
        dts.add(dev.dt)
    assert len(dts) > 1  # the controller actually moved dt
    assert vec_rel_err(dev.host("vel"), orc.vel) < 1e-3


def test_adaptive_baseline_parity_1m():
    """The globally adaptive PCISPH baseline at cfg2 scale: a
    synchronous step of all 1 M particles from a common state, three times."""
    import bench
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    sc = bench.scene_cfg2()
    dev = PcisphSolver(sc, mode="adaptive", iteration_cap=50)
    orc = OraclePcisph(sc, mode="adaptive", iteration_cap=50)
    apply_jitter(dev, orc)
    for _ in range(3):
        inject(dev, orc, PCISPH_STATE)
        orc.xstar[:] = dev.host("xstar")
        orc.dt = dev.dt
        a, b = dev.advance()[0], orc.advance()[0]
        assert (a.iterations, a.corrected) == (b.iterations, b.corrected)
        assert a.max_err == pytest.approx(b.max_err, rel=1e-6)
        assert dev.dt == orc.dt
    assert vec_rel_err(dev.host("vel"), orc.vel) < 1e-3


# -- cfg3: 1 M RTS-WCSPH -------------------------------------------------------------

def test_cfg3_wcsph_1m_parity():
    """20 RTS-WCSPH steps from a common state each: active counts, sort and
    rho exact / <= 1e-4; then 50 steps from the same start: statistics."""
    import bench
    from oracle.sph import OracleWcsph
    dev = bench.make_device_solver("wcsph", torch.device("cuda", 0))
    orc = OracleWcsph(dev.scene, mode="rts")
    orc.pos[:] = dev.host("pos")
    compared = 0
    for _ in range(20):
        inject(dev, orc, WCSPH_STATE)
        a, b = dev.step(), orc.step()
        assert a.n_compute == b.n_compute
        assert np.array_equal(dev.grid.order.cpu().numpy(), orc.grid.order)
        act = orc.compute
        if act.any():
            assert rel_err(dev.host("rho")[act], orc.rho[act]) <= TOL
            assert vec_rel_err(dev.host("acc")[act], orc.acc[act]) <= TOL
            compared += int(act.sum())
    assert compared > 0
    del dev, orc
    dev = bench.make_device_solver("wcsph", torch.device("cuda", 0))
    orc = OracleWcsph(dev.scene, mode="rts")
    orc.pos[:] = dev.host("pos")
    for _ in range(50):
        dev.step()
        orc.step()
    rho0 = dev.scene.rest_density
    sd = density_stats(dev.host("rho"), dev.host("vel"), dev.mass, rho0)
    so = density_stats(orc.rho, orc.vel, orc.mass, rho0)
    for k in ("mean_err", "max_err", "ke"):
        assert abs(sd[k] - so[k]) <= STAT_TOL * abs(so[k]), (k, sd, so)


# -- cfg4 (8 M mixed tank) and cfg5 (4 M per GPU) at one GPU ------------------------

def _workload_pair(workload):
    import bench
    kind = bench.WORKLOADS[workload][0]
    dev = bench.make_device_solver(kind, torch.device("cuda", 0), workload)
    orc, _ = bench._oracle_for(workload)
    nf = dev.n_fluid
    assert orc.n_fluid == nf
    assert np.array_equal(dev.host("pos")[:nf], orc.pos[:nf])  # the same jittered start
    orc.pos[:] = dev.host("pos")
    if kind == "pcisph":
        orc.xstar[:] = orc.pos[:nf]
    orc.vel[:] = dev.host("vel")
    return dev, orc


@pytest.mark.parametrize("workload", ["cfg4", "cfg5-pcisph"])
def test_large_workloads_first_iteration_parity(workload):
    """BASELINE configs[3] (8 M, z-up, a falling block at -2 m/s over a resting
    pool: mixed levels) and configs[4] at one GPU (4 M, N(0, 0.1) velocities):
    one major on the device, then a major start from the common state --
    rows exact, rho*, err, p, f_p <= 1e-4, S_e / S_ob exact."""
    dev, orc = _workload_pair(workload)
    dev.advance()
    r = first_iteration(dev, orc)
    _check_first_iteration(r)
    del dev, orc
    torch.cuda.empty_cache()


def test_cfg5_wcsph_4m_common_state_steps():
    """configs[4] RTS-WCSPH at one GPU (4 M, N(0, 0.1) velocities): three steps
    from a common state each -- active counts and sort exact, rho and
    accelerations <= 1e-4."""
    dev, orc = _workload_pair("cfg5-wcsph")
    compared = 0
    for _ in range(3):
        inject(dev, orc, WCSPH_STATE)
        a, b = dev.step(), orc.step()
        assert a.n_compute == b.n_compute
        assert np.array_equal(dev.grid.order.cpu().numpy(), orc.grid.order)
        act = orc.compute
        if act.any():
            assert rel_err(dev.host("rho")[act], orc.rho[act]) <= TOL
            assert vec_rel_err(dev.host("acc")[act], orc.acc[act]) <= TOL
            compared += int(act.sum())
    assert compared > 0
    del dev, orc
    torch.cuda.empty_cache()
