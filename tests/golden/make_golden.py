"""Generate the golden fixtures that pin the CPU oracle to the reference.

Run in the build container (needs /root/reference and numba):

    python tests/golden/make_golden.py

Every scenario drives the UNMODIFIED reference package ``rts_sph`` (through
``ref_shim.import_reference``) and stores its inputs and outputs as float64
/ int arrays in ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
re-runs the oracle on the same inputs and requires bit-identical results.
The fixtures are small (1,000-particle tiny tank, 16k cfg1 statistics).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from ref_shim import import_reference  # noqa: E402

TINY = """
domain = 0 0 0  0.4 0.4 0.4
spacing = 0.02
fluid_box = 0.02 0.02 0.02  0.22 0.22 0.22
sound_speed = 30
"""


def jitter(n, s, seed, frac=0.01):
    return np.random.default_rng(seed).uniform(-frac * s, frac * s, (n, 3))


def fp32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes raw")


def grid_fixture(R):
    sc = R.parse_scene_text(TINY)
    s = R.WcsphSolver(sc, mode="rts")
    nf = s.n_fluid
    s.pos[:nf] = fp32(s.pos[:nf] + jitter(nf, sc.spacing, 7))
    g = s.grid
    g.rebuild(s.pos, nf)
    nbr = np.zeros((nf, 128), dtype=np.int64)
    cnt = np.zeros(nf, dtype=np.int64)
    idx = np.arange(nf)
    g.search_into(s.pos, idx, np.ones(nf, dtype=np.int64), sc.support_radius, nbr, cnt)
    flat = np.concatenate([nbr[i, : cnt[i]] for i in range(nf)])
    # stale-grid two-layer search (grid.py:116-137) on the PCISPH grid
    gp = R.BlockGrid.for_scene(sc, "pcisph")
    gp.rebuild(s.pos, nf)
    moved = s.pos.copy()
    moved[:nf] = fp32(moved[:nf] + jitter(nf, sc.spacing, 8, frac=0.5))
    nbr2 = np.zeros((nf, 128), dtype=np.int64)
    cnt2 = np.zeros(nf, dtype=np.int64)
    gp.search_into(moved, idx, np.full(nf, 2, dtype=np.int64), sc.support_radius, nbr2, cnt2)
    flat2 = np.concatenate([nbr2[i, : cnt2[i]] for i in range(nf)])
    save("grid_tiny", pos=s.pos, n_fluid=np.int64(nf), fluid_cells=g.fluid_cells,
         starts=g.starts, order=g.order, occupancy=g.occupancy,
         boundary_active=g.boundary_active, cnt=cnt, nbr_flat=flat, moved=moved,
         p_starts=gp.starts, p_order=gp.order, cnt2=cnt2, nbr2_flat=flat2)


def regions_fixture(R):
    rng = np.random.default_rng(11)
    dims = (9, 7, 8)
    nc = int(np.prod(dims))
    occ = rng.random(nc) < 0.7
    v = np.where(occ, rng.uniform(0, 3.0, nc), 0.0)
    f = np.where(occ, rng.uniform(0, 0.5, nc), 0.0)
    f[rng.random(nc) < 0.1] = 0.0
    kw = dict(dt_base=1.75e-4 * 2, block_size=0.044, particle_mass=0.008, sound_speed=30.0,
              lambda_v=0.4, lambda_f=0.25, alpha=1.0, betas=np.array([np.nan, np.inf, 0.4, 0.08,
                                                                       0.016]))
    raw = R.assign_regions(v, f, occ, n_max=4, use_sound_criterion=False, **kw)
    raw_s = R.assign_regions(v, f, occ, n_max=4, use_sound_criterion=True,
                             **{**kw, "dt_base": 1e-4})
    sm, rmin = R.smooth_regions(raw, dims)
    ex = R.expand_fast_regions(sm, dims)
    err = rng.random(nc) < 0.05
    obs = R.derive_observed(ex, dims, err)
    save("regions_random", dims=np.array(dims), occ=occ, v=v, f=f, raw=raw, raw_sound=raw_s,
         smooth=sm, rmin=rmin, expanded=ex, err_blocks=err, observed=obs)


def wcsph_fixture(R):
    out = {}
    for mode, steps in (("rts", 30), ("baseline", 12)):
        sc = R.parse_scene_text(TINY)
        s = R.WcsphSolver(sc, mode=mode)
        nf = s.n_fluid
        s.pos[:nf] = fp32(s.pos[:nf] + jitter(nf, sc.spacing, 1234))
        ncomp, dts = [], []
        for _ in range(steps):
            st = s.step()
            ncomp.append(st.n_compute)
            dts.append(st.dt)
        for k in ("pos", "vel", "acc", "acc_prev", "force", "rho", "pres", "dt_since", "dt_corr",
                  "validity", "region", "compute"):
            out[f"{mode}_{k}"] = getattr(s, k)
        out[f"{mode}_n_compute"] = np.array(ncomp)
        out[f"{mode}_dt"] = np.array(dts)
        out[f"{mode}_steps"] = np.int64(steps)
    save("wcsph_tiny", **out)


def pcisph_fixture(R):
    out = {}
    for mode, majors in (("rts", 3), ("const", 3), ("adaptive", 3)):
        sc = R.parse_scene_text(TINY)
        s = R.PcisphSolver(sc, mode=mode)
        nf = s.n_fluid
        s.pos[:nf] = fp32(s.pos[:nf] + jitter(nf, sc.spacing, 1234, frac=0.002))
        s.xstar[:] = s.pos[:nf]
        rows = []
        for _ in range(majors):
            for st in s.advance():
                rows.append([st.n_compute, st.iterations, st.corrected, st.iters_r1,
                             st.iters_r2, st.iters_r3, st.iters_r4, st.early_term, st.max_err,
                             st.avg_err, st.dt])
        for k in ("pos", "vel", "f_ext", "f_p", "p", "rho_star", "err", "xstar", "region",
                  "validity", "compute", "in_se", "in_sob", "cnt"):
            out[f"{mode}_{k}"] = getattr(s, k)
        out[f"{mode}_stats"] = np.array(rows, dtype=np.float64)
        out[f"{mode}_majors"] = np.int64(majors)
        out[f"{mode}_dt_final"] = np.float64(s.dt)
    save("pcisph_tiny", **out)


def cfg1_fixture(R):
    """BASELINE config 1 statistics after 200 RTS-WCSPH steps (16k)."""
    sc = R.Scene(domain_min=(0, 0, 0), domain_max=(1.0, 0.5, 1.0),
                 fluid_boxes=(((0, 0, 0), (0.4, 0.4, 0.8)),), spacing=0.02)
    s = R.WcsphSolver(sc, mode="rts")
    nf = s.n_fluid
    s.pos[:nf] = fp32(s.pos[:nf] + jitter(nf, sc.spacing, 1234))
    ncomp = [s.step().n_compute for _ in range(200)]
    e = (s.rho - sc.rest_density) / sc.rest_density
    ke = 0.5 * s.mass * float((s.vel * s.vel).sum())
    import hashlib
    digest = hashlib.sha1(np.ascontiguousarray(s.pos).tobytes() +
                          np.ascontiguousarray(s.vel).tobytes() +
                          np.ascontiguousarray(s.rho).tobytes()).hexdigest()
    save("cfg1_stats", n_compute=np.array(ncomp), mean_err=np.float64(e.mean()),
         max_err=np.float64(e.max()), ke=np.float64(ke), mass=np.float64(nf * s.mass),
         sim_time=np.float64(s.sim_time), state_sha1=np.array(digest))


def main():
    R = import_reference()
    grid_fixture(R)
    regions_fixture(R)
    wcsph_fixture(R)
    pcisph_fixture(R)
    cfg1_fixture(R)


if __name__ == "__main__":
    main()
