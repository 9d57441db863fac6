"""Parity helpers: seeded fp32 jitter, state injection device -> oracle, and
the comparison metrics of BASELINE.json (bit-exact integer/index work,
<= 1e-4 relative for per-particle fp32 fields, norm-relative for vectors)."""

from __future__ import annotations

import numpy as np

WCSPH_STATE = ("vel", "acc", "acc_prev", "force", "rho", "pres", "dt_since", "dt_corr",
               "validity", "region", "compute")
PCISPH_STATE = ("vel", "f_ext", "f_p", "p", "rho_star", "err", "xstar", "region", "validity",
                "compute", "in_se", "in_sob")


def jitter(n: int, spacing: float, seed: int = 1234, frac: float = 0.01) -> np.ndarray:
    """Seeded uniform jitter of +-frac*spacing (BASELINE.json configs)."""
    return np.random.default_rng(seed).uniform(-frac * spacing, frac * spacing, (n, 3))


def apply_jitter(dev, orc, seed=1234, frac=0.01):
    """Jitter both solvers identically, at fp32-representable positions."""
    nf = dev.n_fluid
    j = jitter(nf, dev.scene.spacing, seed, frac)
    x = (orc.pos[:nf] + j).astype(np.float32)
    import torch
    dev.pos[:nf] = torch.as_tensor(x, device=dev.device)
    orc.pos[:nf] = x.astype(np.float64)
    orc.pos[nf:] = dev.host("pos")[nf:]  # wall samples as the device stores them (fp32)
    if hasattr(orc, "xstar"):
        orc.xstar[:] = orc.pos[:nf]
        dev.xstar[:] = dev.pos[:nf]


def inject(dev, orc, names) -> None:
    """Copy the device state into the oracle (upcast), the 'common state'."""
    nf = dev.n_fluid
    orc.pos[:] = dev.host("pos")
    for n in names:
        v = dev.host(n)
        cur = getattr(orc, n)
        setattr(orc, n, v.astype(cur.dtype).reshape(cur.shape))
    assert orc.n_fluid == nf


def rel_err(a, ref) -> float:
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.abs(a - ref)
    s = np.abs(ref)
    m = s > 0
    out = 0.0
    if m.any():
        out = float((d[m] / s[m]).max())
    if (~m).any():
        out = max(out, float(d[~m].max()))
    return out


def vec_rel_err(a, ref) -> float:
    """max over rows of |a_i - ref_i| / |ref_i| (rows with |ref_i| > 0)."""
    a = np.asarray(a, dtype=np.float64).reshape(-1, 3)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1, 3)
    num = np.linalg.norm(a - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    m = den > 0
    out = float((num[m] / den[m]).max()) if m.any() else 0.0
    if (~m).any():
        out = max(out, float(num[~m].max()))
    return out


# ---- scale probes shared by tests/test_parity_scale_gpu.py and
# scripts/parity_probe.py ---------------------------------------------------

DECISION_FIELDS = ("n_compute", "iterations", "corrected", "iters_r1", "iters_r2", "iters_r3",
                   "iters_r4", "early_term")


def sync_controller(dev, orc) -> None:
    """Major-step controller state and dt of the device solver -> oracle."""
    orc.controller.n_current = dev.controller.n_current
    orc.controller.recovery_left = dev.controller.recovery_left
    orc.dt = dev.dt


def density_stats(rho, vel, mass, rho0) -> dict:
    """mean / max (rho - rho0) / rho0 over the solver's density array (stale
    entries included, as the reference reports it) and kinetic energy."""
    e = (np.asarray(rho, np.float64) - rho0) / rho0
    v = np.asarray(vel, np.float64)
    return {"mean_err": float(e.mean()), "max_err": float(e.max()),
            "ke": float(0.5 * mass * (v * v).sum())}


def common_state_majors(dev, orc, majors: int) -> dict:
    """RTS-PCISPH major steps, the device state injected into the oracle
    before each one; per-minor decision mismatches are counted (each major
    compares one major's decisions taken from identical inputs)."""
    out = {"minors": 0, "mismatch": {f: 0 for f in DECISION_FIELDS}, "len_mismatch": 0,
           "corrected_rel_max": 0.0, "n_compute_rel_max": 0.0, "examples": []}
    for m in range(majors):
        inject(dev, orc, PCISPH_STATE)
        orc.xstar[:] = dev.host("xstar")
        sync_controller(dev, orc)
        rd, ro = dev.advance(), orc.advance()
        if len(rd) != len(ro):
            out["len_mismatch"] += 1
        for a, b in zip(rd, ro):
            out["minors"] += 1
            bad = False
            for f in DECISION_FIELDS:
                if getattr(a, f) != getattr(b, f):
                    out["mismatch"][f] += 1
                    bad = True
            out["corrected_rel_max"] = max(out["corrected_rel_max"],
                                           abs(a.corrected - b.corrected) / max(1, b.corrected))
            out["n_compute_rel_max"] = max(out["n_compute_rel_max"],
                                           abs(a.n_compute - b.n_compute) / max(1, b.n_compute))
            if bad and len(out["examples"]) < 6:
                out["examples"].append({"major": m, **{f: [getattr(a, f), getattr(b, f)]
                                                        for f in DECISION_FIELDS}})
    return out


def first_iteration(dev, orc) -> dict:
    """A major-step start from a common state on both solvers: rebuild,
    region assignment, refresh (neighbour rows, f_ext), then one correction
    iteration with every region scheduled.  f_ext is compared after the
    refresh and then handed to the oracle, so rho*, err, p and f_p compare
    one density / pressure / pressure-force pass from identical inputs
    (pcisph.py:174-271, 432-437)."""
    inject(dev, orc, PCISPH_STATE)
    orc.xstar[:] = dev.host("xstar")
    orc.grid.rebuild(orc.pos, orc.n_fluid)
    orc._assign_major_regions(4)
    dev._prepare(dev.dt)
    dev._rebuild(True)
    dev._assign_major_regions(4, rebuilt=True)
    dev._read()
    res = {"order_equal": bool(np.array_equal(dev.grid.order.cpu().numpy(), orc.grid.order)),
           "block_region_equal": bool(np.array_equal(dev.block_region.cpu().numpy(),
                                                     orc.block_region))}
    k = orc.kernel
    refresh = np.flatnonzero(orc.compute).astype(np.int64)
    layers = np.where(orc.region[refresh] == 1, 2, 1).astype(np.int64)
    orc.grid.search_into(orc.pos, refresh, layers, k.h, orc.nbr, orc.cnt)
    orc._ext(refresh)
    orc.p[:] = 0.0
    orc.f_p[:] = 0.0
    dev._call("rts_pci_refresh", 0, 1)
    dev._zero_pressure()
    cnt = dev.cnt.cpu().numpy()
    nbr = dev.nbr.cpu().numpy()
    mask = np.arange(nbr.shape[1])[None, :] < cnt[:, None]
    res["cnt_equal"] = bool(np.array_equal(cnt, orc.cnt))
    res["rows_equal"] = bool(np.array_equal(np.where(mask, nbr, -1),
                                            np.where(mask, orc.nbr, -1)))
    res["f_ext_rel"] = vec_rel_err(dev.host("f_ext"), orc.f_ext)
    orc.f_ext[:] = dev.host("f_ext")  # common input of the iteration
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
    res["n_pred_equal"] = int(c.n_pred) == pred.size
    res["rho_star_rel"] = rel_err(dev.host("rho_star")[pred], orc.rho_star[pred])
    res["err_abs"] = float(np.abs(dev.host("err")[pred] - orc.err[pred]).max())
    pp = orc.p[force] > 0
    res["p_rel"] = rel_err(dev.host("p")[force][pp], orc.p[force][pp])
    res["p_zero_equal"] = bool(np.array_equal(dev.host("p")[force] == 0, orc.p[force] == 0))
    res["f_p_rel"] = vec_rel_err(dev.host("f_p")[force], orc.f_p[force])
    res["in_se_flips"] = int((dev.host("in_se") != orc.in_se).sum())
    res["in_sob_flips"] = int((dev.host("in_sob") != orc.in_sob).sum())
    res["max_err"] = [float(c.max_err), float(orc.err.max())]
    return res


def free_run(dev, orc, majors: int) -> dict:
    """Both solvers from the same start, no re-injection: end-of-run
    statistics (BASELINE.json north_star: mass, mean / max density error,
    kinetic energy)."""
    rd, ro = [], []
    for _ in range(majors):
        rd += dev.advance()
        ro += orc.advance()
    rho0 = dev.scene.rest_density
    sd = density_stats(dev.host("rho_star"), dev.host("vel"), dev.mass, rho0)
    so = density_stats(orc.rho_star, orc.vel, orc.mass, rho0)
    return {"minors": [len(rd), len(ro)],
            "mass": [dev.n_fluid * dev.mass, orc.n_fluid * orc.mass],
            "dev": sd, "orc": so,
            "rel": {k: abs(sd[k] - so[k]) / max(abs(so[k]), 1e-300) for k in sd},
            "iters": [sum(r.iterations for r in rd), sum(r.iterations for r in ro)],
            "corrected": [sum(r.corrected for r in rd), sum(r.corrected for r in ro)]}
