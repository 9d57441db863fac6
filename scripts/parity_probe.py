"""Decision-flip and statistics probe: the B200 solvers against the CPU
oracle at the BASELINE configs (measurement for DESIGN.md section 2 and the
tolerances of tests/test_parity_scale_gpu.py).

    python scripts/parity_probe.py [pcisph16k|pcisph1m|adaptive|wcsph1m ...]

Per-major (PCISPH) / per-step (WCSPH) common-state runs: the device state is
injected into the oracle before every major, so each comparison measures
one major's decisions from identical inputs.  Free runs: both solvers run
from the same jittered start without re-injection and their statistics
(mass, mean / max density error, kinetic energy) are compared at the end.
Prints one JSON line per probe."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from parity import (PCISPH_STATE, WCSPH_STATE, apply_jitter, common_state_majors,  # noqa
                    density_stats, first_iteration, free_run, inject, rel_err, vec_rel_err)

def scene_cfg1(**kw):
    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0, 0, 0), domain_max=(1.0, 0.5, 1.0),
                 fluid_boxes=(((0, 0, 0), (0.4, 0.4, 0.8)),), spacing=0.02, **kw)


def pair_pcisph(scene, **kw):
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    dev = PcisphSolver(scene, **kw)
    orc = OraclePcisph(scene, **kw)
    apply_jitter(dev, orc)
    return dev, orc


def probe_pcisph(name, scene, kw, warm, majors, free_majors):
    t0 = time.perf_counter()
    dev, orc = pair_pcisph(scene, mode="rts", **kw)
    for _ in range(warm):
        dev.advance()
    out = {"probe": name, "n_fluid": dev.n_fluid}
    out["common_state"] = common_state_majors(dev, orc, majors)
    out["first_iteration"] = first_iteration(dev, orc)
    del dev, orc
    dev, orc = pair_pcisph(scene, mode="rts", **kw)
    out["free_run"] = free_run(dev, orc, free_majors)
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    print(json.dumps(out), flush=True)


def probe_adaptive(scene, steps, name):
    from oracle.sph import OraclePcisph
    from paper_2009_14514_b200 import PcisphSolver
    dev = PcisphSolver(scene, mode="adaptive")
    orc = OraclePcisph(scene, mode="adaptive")
    apply_jitter(dev, orc)
    mism, dts, ex = 0, 0, []
    for s in range(steps):
        inject(dev, orc, PCISPH_STATE)
        orc.xstar[:] = dev.host("xstar")
        orc.dt = dev.dt
        a, b = dev.advance()[0], orc.advance()[0]
        if (a.iterations, a.corrected) != (b.iterations, b.corrected):
            mism += 1
            ex.append([s, a.iterations, b.iterations])
        if dev.dt != orc.dt:
            dts += 1
    print(json.dumps({"probe": name, "steps": steps, "iter_mismatch": mism, "dt_mismatch": dts,
                      "dt_final": [dev.dt, orc.dt], "examples": ex[:6]}), flush=True)


def probe_wcsph1m(steps, free_steps):
    import bench
    from oracle.sph import OracleWcsph
    t0 = time.perf_counter()
    dev = bench.make_device_solver("wcsph", torch.device("cuda", 0))
    orc = OracleWcsph(dev.scene, mode="rts")
    orc.pos[:] = dev.host("pos")
    n_mis, rho_rel, acc_rel, ord_eq, ex = 0, 0.0, 0.0, True, []
    for s in range(steps):
        inject(dev, orc, WCSPH_STATE)
        a, b = dev.step(), orc.step()
        if a.n_compute != b.n_compute:
            n_mis += 1
            ex.append([s, a.n_compute, b.n_compute])
        ord_eq = ord_eq and np.array_equal(dev.grid.order.cpu().numpy(), orc.grid.order)
        act = orc.compute
        if act.any():
            rho_rel = max(rho_rel, rel_err(dev.host("rho")[act], orc.rho[act]))
            acc_rel = max(acc_rel, vec_rel_err(dev.host("acc")[act], orc.acc[act]))
            da = np.linalg.norm(dev.host("acc")[act] - orc.acc[act], axis=1)
            an = np.linalg.norm(orc.acc[act], axis=1)
            bad = da > 1e-4 * an
            g = float(np.linalg.norm(dev.scene.gravity))
            ex.append({"step": s, "n_act": int(act.sum()), "n_over_1e-4": int(bad.sum()),
                       "acc_norm_of_over": [float(x) for x in np.sort(an[bad])[:5]],
                       "max_da_over_g": float(da.max() / g),
                       "max_da_over_max_a_g": float((da / np.maximum(an, g)).max())})
    res = {"probe": "wcsph1m", "steps": steps, "n_compute_mismatch": n_mis, "order_equal": ord_eq,
           "rho_rel_max": rho_rel, "acc_rel_max": acc_rel, "examples": ex[:8]}
    del dev, orc
    dev = bench.make_device_solver("wcsph", torch.device("cuda", 0))
    orc = OracleWcsph(dev.scene, mode="rts")
    orc.pos[:] = dev.host("pos")
    for _ in range(free_steps):
        dev.step()
        orc.step()
    rho0 = dev.scene.rest_density
    sd = density_stats(dev.host("rho"), dev.host("vel"), dev.mass, rho0)
    so = density_stats(orc.rho, orc.vel, orc.mass, rho0)
    res["free_run"] = {"steps": free_steps, "dev": sd, "orc": so,
                       "rel": {k: abs(sd[k] - so[k]) / max(abs(so[k]), 1e-300) for k in sd}}
    res["wall_s"] = round(time.perf_counter() - t0, 1)
    print(json.dumps(res), flush=True)


def twin_oracle(scene, kw, dev):
    """The oracle again, its fluid start perturbed by one fp32 ulp per
    coordinate (seeded signs): the reference's own sensitivity to an
    fp32-rounding-sized change of its state."""
    from oracle.sph import OraclePcisph
    tw = OraclePcisph(scene, mode="rts", **kw)
    nf = tw.n_fluid
    x = dev.host("pos")[:nf].astype(np.float32)
    sign = np.random.default_rng(99).choice([-1.0, 1.0], size=x.shape).astype(np.float32)
    x2 = np.nextafter(x, x + sign * np.float32(1.0))
    tw.pos[:nf] = x2.astype(np.float64)
    tw.xstar[:] = tw.pos[:nf]
    return tw


def probe_twin(name, scene, kw, majors, every, f32=False):
    """Free runs of the device, the oracle and a twin oracle (perturbed
    start, or ``f32``: the fp32-state oracle); statistics of all three every
    ``every`` majors."""
    dev, orc = pair_pcisph(scene, mode="rts", **kw)
    if f32:
        from oracle.sph import OraclePcisph
        tw = OraclePcisph(scene, mode="rts", state_f32=True, **kw)
        tw.pos[:] = orc.pos
        tw.xstar[:] = orc.xstar
    else:
        tw = twin_oracle(scene, kw, dev)
    rho0 = scene.rest_density
    pts = []
    for m in range(1, majors + 1):
        rd, ro, rt = dev.advance(), orc.advance(), tw.advance()
        if m % every == 0:
            st = [density_stats(dev.host("rho_star"), dev.host("vel"), dev.mass, rho0),
                  density_stats(orc.rho_star, orc.vel, orc.mass, rho0),
                  density_stats(tw.rho_star, tw.vel, tw.mass, rho0)]
            pts.append({"major": m, "stats": st,
                        "corr": [sum(r.corrected for r in x) for x in (rd, ro, rt)],
                        "ncomp": [sum(r.n_compute for r in x) for x in (rd, ro, rt)]})
    print(json.dumps({"probe": name, "series": pts}), flush=True)


def probe_argmax(name, scene, kw, majors):
    """Free run of the device and the fp32-state oracle; the particles holding
    the max density error in each, and their state in the other solver."""
    from oracle.sph import OraclePcisph
    dev, orc = pair_pcisph(scene, mode="rts", **kw)
    t32 = OraclePcisph(scene, mode="rts", state_f32=True, **kw)
    t32.pos[:] = orc.pos
    t32.xstar[:] = orc.xstar
    for _ in range(majors):
        dev.advance()
        t32.advance()
        orc.advance()
    rho0 = scene.rest_density
    ed = (dev.host("rho_star") - rho0) / rho0
    et = (t32.rho_star - rho0) / rho0
    eo = (orc.rho_star - rho0) / rho0
    out = {"probe": name}
    for tag, e in (("dev", ed), ("t32", et), ("orc", eo)):
        top = np.argsort(-e)[:5]
        out[tag] = [{"i": int(i), "err_dev": float(ed[i]), "err_t32": float(et[i]),
                     "err_orc": float(eo[i]), "region": [int(dev.host("region")[i]),
                                                         int(t32.region[i]), int(orc.region[i])],
                     "dpos_dev_t32": float(np.abs(dev.host("pos")[i] - t32.pos[i]).max()),
                     "in_se": [bool(dev.host("in_se")[i]), bool(t32.in_se[i])],
                     "in_sob": [bool(dev.host("in_sob")[i]), bool(t32.in_sob[i])]}
                    for i in top]
    out["n_diff_rho_gt_1e-3"] = int((np.abs(ed - et) > 1e-3).sum())
    out["pos_max_diff_dev_t32"] = float(np.abs(dev.host("pos")[:dev.n_fluid]
                                               - t32.pos[:t32.n_fluid]).max())
    print(json.dumps(out), flush=True)


def probe_series(name, scene, kw, majors, every):
    """Free run with the statistics of both solvers every ``every`` majors:
    how far apart the runs drift against how much each statistic moves."""
    dev, orc = pair_pcisph(scene, mode="rts", **kw)
    rho0 = scene.rest_density
    pts = []
    for m in range(1, majors + 1):
        dev.advance()
        orc.advance()
        if m % every == 0:
            rd, ro = dev.host("rho_star"), orc.rho_star
            sd = density_stats(rd, dev.host("vel"), dev.mass, rho0)
            so = density_stats(ro, orc.vel, orc.mass, rho0)
            ed, eo = (rd - rho0) / rho0, (ro - rho0) / rho0
            pts.append({"major": m, "dev": sd, "orc": so,
                        "p999": [float(np.quantile(ed, 0.999)), float(np.quantile(eo, 0.999))],
                        "pos_max_diff": float(np.abs(dev.host("pos")[:dev.n_fluid]
                                                     - orc.pos[:orc.n_fluid]).max())})
    print(json.dumps({"probe": name, "series": pts}), flush=True)


def main():
    import bench
    what = sys.argv[1:] or ["pcisph16k", "adaptive", "pcisph1m", "wcsph1m"]
    for w in what:
        if w == "pcisph16k":
            probe_pcisph("pcisph16k_eta2", scene_cfg1(eta_max=0.02, eta_avg=0.01), {}, 2, 50, 50)
        elif w == "pcisph1m":
            probe_pcisph("pcisph1m_cfg2", bench.scene_cfg2(), {"iteration_cap": 50}, 2, 8, 50)
        elif w == "adaptive":
            from conftest import tiny_tank
            probe_adaptive(tiny_tank(), 40, "adaptive_tiny")
            probe_adaptive(scene_cfg1(eta_max=0.02, eta_avg=0.01), 40, "adaptive16k")
        elif w == "twin16k":
            probe_twin("twin16k", scene_cfg1(eta_max=0.02, eta_avg=0.01), {}, 50, 5)
        elif w == "twin1m":
            probe_twin("twin1m", bench.scene_cfg2(), {"iteration_cap": 50}, 50, 5)
        elif w == "f32twin16k":
            probe_twin("f32twin16k", scene_cfg1(eta_max=0.02, eta_avg=0.01), {}, 50, 5, True)
        elif w == "f32twin1m":
            probe_twin("f32twin1m", bench.scene_cfg2(), {"iteration_cap": 50}, 50, 5, True)
        elif w == "argmax1m":
            probe_argmax("argmax1m", bench.scene_cfg2(), {"iteration_cap": 50}, 50)
        elif w == "series16k":
            probe_series("series16k", scene_cfg1(eta_max=0.02, eta_avg=0.01), {}, 100, 5)
        elif w == "series1m":
            probe_series("series1m", bench.scene_cfg2(), {"iteration_cap": 50}, 50, 5)
        elif w == "wcsph1m":
            probe_wcsph1m(20, 50)


if __name__ == "__main__":
    main()
