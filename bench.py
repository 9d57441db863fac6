#!/usr/bin/env python
"""Benchmark: RTS-PCISPH (BASELINE.json configs[1]) particle-updates/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (configs[1], mapped per SURVEY.md section 0.4 / 8(d)): dam break,
100^3 = 1,000,000 fluid particles at spacing 0.01 m (h = 0.02 m) in a
2.5 x 1.25 x 2.5 m tank with 2 wall layers (510,064 wall samples), +-1 %
seeded lattice jitter (seed 1234), RTS-PCISPH with up to 4 levels, minor
step 1.75e-4 s, iteration cap 50, eta_max = 0.03 / eta_avg = 0.015 (the
literal 1 % diverges on the reference itself).  A bench step
is one ``advance()`` = one major step (4 minor steps); the metric counts
N_fluid x minor steps / second.  Synthetic data; fp32 state, fp64 pair sums.

For N > 1 (torchrun, one rank per GPU) the scene grows along x by 1 m of
fluid per rank (weak scaling) and is cut into x-slabs
(paper_2009_14514_b200/distributed.py): ghost-column exchange and
migration at every major step, ghost x*/p/err exchange and an all-reduce of
the convergence scalars in every correction iteration (NCCL).
Timing: W untimed majors, then K majors bracketed by barrier +
synchronize, CUDA events on the solver stream, max over ranks.

The line also carries: the live roofline of the dominant kernel (CUDA
events around its launches), e2e (same metric through the public API with
pinned host state copied in and out every step), the CPU oracle baseline
on this host (bounded sample), clocks sampled during the timed region, and
the RTS-WCSPH 1M (configs[2]) throughput as an extra.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "particle-updates/s (RTS-PCISPH, 1M dam break, minor steps)"
UNIT = "particle-updates/s"
SEED = 1234


def scene_cfg2(world: int = 1):
    """configs[1] at world = 1; for weak scaling the fluid column and the
    tank grow along x by 1 m per rank (world m of fluid in a world + 1.5 m
    tank), so every rank's x-slab holds ~1 M particles."""
    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0.0, 0.0, 0.0), domain_max=(world + 1.5, 1.25, 2.5),
                 fluid_boxes=(((0.0, 0.0, 0.0), (float(world), 1.0, 1.0)),), spacing=0.01,
                 eta_max=0.03, eta_avg=0.015)


def scene_cfg3():
    import math

    from paper_2009_14514_b200 import Scene
    return Scene(domain_min=(0.0, 0.0, 0.0), domain_max=(2.5, 1.25, 2.5),
                 fluid_boxes=(((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)),), spacing=0.01,
                 sound_speed=10.0 * math.sqrt(2.0 * 9.81 * 1.0))


def jitter_np(n, spacing):
    import numpy as np
    return np.random.default_rng(SEED).uniform(-0.01 * spacing, 0.01 * spacing, (n, 3))


def make_device_solver(kind: str, device):
    import numpy as np
    import torch

    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    if kind == "pcisph":
        s = PcisphSolver(scene_cfg2(), mode="rts", iteration_cap=50, device=device)
    else:
        s = WcsphSolver(scene_cfg3(), mode="rts", device=device)
    nf = s.n_fluid
    x = (s.host("pos")[:nf] + jitter_np(nf, s.scene.spacing)).astype(np.float32)
    s.pos[:nf] = torch.as_tensor(x, device=s.device)
    if kind == "pcisph":
        s.xstar[:] = s.pos[:nf]
    return s


# per-kernel algorithmic bytes (fp32 state, int32 indices, neighbour data
# reused on chip) -- DESIGN.md "Kernels and their rooflines"
def algo_bytes(name: str, solver, c_mean: float, rec: dict, launches: int = 1) -> float:
    """Algorithmic bytes of all recorded launches of one entry point."""
    nf = solver.n_fluid
    # density 24 + 4c per predicted particle plus the
    # pressure accumulation (8 B) of the force set; refresh 56 + 8c per
    # refreshed particle (list build 16 + 4c, external forces 40 + 4c).  The
    # pressure-force pass is the survey's fused force/predict (80 + 4c)
    # without the prediction, which k_motion does (84 B per particle).
    if name == "rts_pci_density":
        return rec["pred"] * (24 + 4 * c_mean) + rec["force"] * 8
    if name == "rts_pci_pforces":
        return rec["force"] * (40 + 4 * c_mean)
    if name == "rts_pci_refresh":
        return rec["refresh"] * (56 + 8 * c_mean) + nf * 1
    if name == "rts_pci_motion":
        return rec["motion"] * 84
    if name == "rts_pci_sets":
        return launches * nf * 9 + 4 * (rec["pred"] + rec["force"])
    if name == "rts_pci_se_reduce":
        return launches * nf * 13
    if name == "rts_pci_integrate":
        return launches * nf * 82
    return 0.0


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"rts_clocks_{os.getpid()}.csv")

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader",
                 "-lms", "20"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                mx.append(float(f[2].split()[0]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        loaded.sort()
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_sample(majors: int = 2, warm: int = 1) -> dict:
    """Time the CPU oracle (fp64 C + numpy restatement of the reference) on
    the same scene: ``warm`` untimed majors, then ``majors`` timed."""
    import numpy as np

    from oracle import sph as O
    sc = scene_cfg2()
    t_setup = time.perf_counter()
    o = O.OraclePcisph(sc, mode="rts", iteration_cap=50)
    nf = o.n_fluid
    x = (o.pos[:nf] + jitter_np(nf, sc.spacing)).astype(np.float32).astype(np.float64)
    o.pos[:nf] = x
    o.xstar[:] = x
    for _ in range(warm):
        o.advance()
    minors = 0
    t0 = time.perf_counter()
    for _ in range(majors):
        minors += len(o.advance())
    dt = time.perf_counter() - t0
    return {"value": nf * minors / dt, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
            "sample": f"{majors} major steps ({minors} minor steps) of the 1M cfg2 scene after "
                      f"{warm} untimed major(s); oracle = fp64 C/OpenMP + numpy restatement",
            "seconds": round(dt, 3), "setup_s": round(t0 - t_setup, 1)}


def run_reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    from oracle import sph as O
    import numpy as np
    sc = scene_cfg2()
    o = O.OraclePcisph(sc, mode="rts", iteration_cap=50)
    nf = o.n_fluid
    x = (o.pos[:nf] + jitter_np(nf, sc.spacing)).astype(np.float32).astype(np.float64)
    o.pos[:nf] = x
    o.xstar[:] = x
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, 6))  # bounded sample: ~3 s CPU per major here
    for _ in range(warm):
        o.advance()
    minors = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        minors += len(o.advance())
    dt = time.perf_counter() - t0
    v = nf * minors / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * dt / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg2: 1M dam break RTS-PCISPH (eta 3%/1.5%, cap 50)",
                   "n_fluid": nf, "minor_steps": minors, "host_threads": O.num_threads()},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
                         "sample": f"{steps} major steps ({minors} minor steps) after {warm} "
                                   "untimed; CPU oracle restating the reference"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=125)  # 125 majors = configs[1]'s 500 steps
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-wcsph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2009_14514_b200 import _native
    local = local % max(1, torch.cuda.device_count())  # ranks > GPUs: 1-GPU path checks
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("RTS_BENCH_BACKEND", "nccl")  # gloo: 1-GPU path checks
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    if world == 1:
        solver = make_device_solver("pcisph", device)
        driver = solver
        n_total = solver.n_fluid
    else:  # x-slab decomposition (paper_2009_14514_b200/distributed.py)
        from paper_2009_14514_b200.distributed import DistributedPcisph
        from paper_2009_14514_b200.scene import seed_particles
        sc = scene_cfg2(world)
        n_total = len(seed_particles(sc)[0])
        driver = DistributedPcisph(sc, device=device, jitter=jitter_np(n_total, sc.spacing),
                                   iteration_cap=50)
        solver = driver.solver
    nf = n_total
    stream = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        driver.advance()
    torch.cuda.synchronize()

    # ---- timed region: K majors, device time --------------------------------
    kernels = ["rts_pci_density", "rts_pci_pforces", "rts_pci_refresh", "rts_pci_motion",
               "rts_pci_sets", "rts_pci_se_reduce", "rts_pci_integrate"]
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = _native.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    minors = 0
    rows = []
    for _ in range(args.steps):
        r = driver.advance()
        rows.extend(r)
        minors += len(r)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    clk = clocks.stop()
    t = ev0.elapsed_time(ev1) * 1e-3
    if world > 1:
        tt = torch.tensor([t, float(minors)], device=device, dtype=torch.float64)
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        t = float(tt[0])
    value = n_total * minors / t  # whole-job particle-updates / s

    # ---- dominant kernel roofline (separate instrumented pass) --------------
    solver.time_kernels(kernels)
    solver.use_graphs = False  # per-kernel CUDA events need individual launches
    solver._force_total = 0
    rec = {"pred": 0, "force": 0, "refresh": 0, "motion": 0}
    prof_rows = []
    for _ in range(max(2, min(args.steps, 8))):
        prof_rows.extend(driver.advance())
    torch.cuda.synchronize()
    totals = {k: sum(solver.kernel_times(k)) for k in kernels}
    counts = {k: len(solver.kernel_times(k)) for k in kernels}
    dom = max(totals, key=totals.get)
    rec["pred"] = sum(r.corrected for r in prof_rows)
    iters = sum(r.iterations for r in prof_rows)
    rec["force"] = rec["pred"]  # force set is a subset; refined by counters below
    if hasattr(solver, "_force_total"):
        rec["force"] = solver._force_total
    rec["refresh"] = sum(r.n_compute for r in prof_rows) * solver.n_fluid // max(1, nf)
    rec["pred"] = rec["pred"] * solver.n_fluid // max(1, nf)
    rec["motion"] = solver.n_fluid * len(prof_rows) + rec["force"]
    c_mean = float(solver.cnt.double().mean())
    solver._ktimes = None
    solver.use_graphs = True
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    alg = algo_bytes(dom, solver, c_mean, rec, counts[dom])
    achieved = alg / totals[dom] / 1e9 if totals[dom] > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(dom)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "launches": counts[dom], "kernel_s": round(totals[dom], 6),
                "algorithmic_bytes": alg,
                "algorithmic_bytes_per_launch": round(alg / max(1, counts[dom])),
                "share_of_step": round(totals[dom] / max(1e-12, sum(totals.values())), 3),
                "kernels": {k: {"s": round(totals[k], 6), "launches": counts[k],
                                "achieved_gbs": round(algo_bytes(k, solver, c_mean, rec,
                                                                 counts[k]) /
                                                      max(totals[k], 1e-12) / 1e9, 1)}
                            for k in kernels if counts[k]},
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
    # live cross-check inside the timed region: the device's %globaltimer
    # stamps around each minor step's refresh (StepStats.t_neighbor: refresh
    # list + search + f_ext on the launching stream) over the K timed majors
    t_live = sum(r.t_neighbor for r in rows)
    alg_live = sum(r.n_compute for r in rows) * solver.n_fluid // max(1, nf) * (56 + 8 * c_mean) \
        + solver.n_fluid * len(rows)
    roofline["live_timed_region"] = {
        "kernel": "rts_pci_refresh", "s": round(t_live, 6), "launches": len(rows),
        "achieved_gbs": round(alg_live / max(t_live, 1e-12) / 1e9, 1),
        "frac": round(alg_live / max(t_live, 1e-12) / 1e9 / peak, 4),
        "share_of_step": round(t_live / max(t, 1e-12), 3),
        "how": "globaltimer stamps in the major-step graph (minor begin -> first prediction)"}

    # ---- e2e through the public API with host-owned state ----------------------
    e2e = None
    if not args.no_e2e:
        # host-owned state: the rank's fluid pos/vel live in pinned host memory,
        # go up before and come back after every advance()
        def dev_state():
            if world == 1:
                return solver.pos[:solver.n_fluid], solver.vel
            return driver.state["pos"], driver.state["vel"]
        k_e2e = max(2, min(args.steps, 10))
        cap = 2 * dev_state()[0].shape[0] + 1024
        hp_all = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        hv_all = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        dp, dv = dev_state()
        hp_all[:dp.shape[0]].copy_(dp)
        hv_all[:dv.shape[0]].copy_(dv)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e_minors = 0
        nbytes = 0
        for _ in range(k_e2e):
            dp, dv = dev_state()
            n = dp.shape[0]
            dp.copy_(hp_all[:n], non_blocking=True)  # step inputs: host -> device
            dv.copy_(hv_all[:n], non_blocking=True)
            e_minors += len(driver.advance())
            dp, dv = dev_state()  # results (ownership may have changed)
            n2 = dp.shape[0]
            hp_all[:n2].copy_(dp, non_blocking=True)
            hv_all[:n2].copy_(dv, non_blocking=True)
            nbytes = (n + n2) * 24
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], device=device, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": n_total * e_minors / te, "unit": UNIT,
               "h2d_bytes_per_step": nbytes // 2, "d2h_bytes_per_step": nbytes // 2,
               "steps": k_e2e, "note": "pinned host pos+vel uploaded before and downloaded "
                                       "after every advance(); wall clock"}

    # ---- WCSPH extra (configs[2] geometry, 1M RTS-WCSPH) ----------------------
    wc = None
    if not args.no_wcsph and world == 1:
        ws = make_device_solver("wcsph", device)
        for _ in range(8):
            ws.step()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        n_w = 40
        a.record(stream)
        fr = 0.0
        for _ in range(n_w):
            fr += ws.step().frac_compute
        b.record(stream)
        b.synchronize()
        tw = a.elapsed_time(b) * 1e-3
        sim_rts = n_w * ws.dt_base
        wc = {"metric": "particle-updates/s (RTS-WCSPH, 1M, base steps)",
              "value": ws.n_fluid * n_w / tw, "ms_per_step": 1e3 * tw / n_w,
              "mean_active_fraction": fr / n_w, "steps": n_w,
              "wall_s_per_simulated_ms": tw / (1e3 * sim_rts)}
        del ws
        # configs[2]'s comparison: the global adaptive baseline (CFL step,
        # dt_cap = 4 dt_base) on the same scene
        from paper_2009_14514_b200 import WcsphSolver
        wb = WcsphSolver(scene_cfg3(), mode="baseline", device=device)
        wb.dt_cap = 4 * wb.dt_base
        nfb = wb.n_fluid
        xb = (wb.host("pos")[:nfb] + jitter_np(nfb, wb.scene.spacing)).astype("float32")
        wb.pos[:nfb] = torch.as_tensor(xb, device=wb.device)
        for _ in range(4):
            wb.step()
        torch.cuda.synchronize()
        sim_b = 0.0
        a.record(stream)
        for _ in range(n_w // 2):
            sim_b += wb.step().dt
        b.record(stream)
        b.synchronize()
        tb = a.elapsed_time(b) * 1e-3
        wc["baseline_adaptive"] = {
            "ms_per_step": 1e3 * tb / (n_w // 2), "mean_dt": sim_b / (n_w // 2),
            "wall_s_per_simulated_ms": tb / (1e3 * sim_b),
            "rts_speedup_per_simulated_time": (tb / sim_b) / (tw / sim_rts)}
        del wb

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_oracle_sample()
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "cfg2: 1M dam break RTS-PCISPH (eta 3%/1.5%, cap 50, "
                                   "dt 1.75e-4, 4 levels)", "n_fluid": nf,
                       "n_boundary": solver.n_bound, "minor_steps": minors,
                       "iterations_per_minor": round(sum(r.iterations for r in rows) /
                                                     max(1, minors), 3),
                       "corrected_per_minor_over_nf": round(sum(r.corrected for r in rows) /
                                                           max(1, minors) / nf, 3),
                       "l2": "working set > L2 (neighbour tables 512 MB + state)",
                       "parallelism": ("single GPU" if world == 1 else
                                       f"x-slabs x{world} (ghost exchange + allreduce)"),
                       "arithmetic": "fp32 state, fp64 pair sums"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "wcsph_rts_1m": wc,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
