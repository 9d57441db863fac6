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


E2E_CHUNKS = int(os.environ.get("RTS_E2E_CHUNKS", "1"))  # scripts/e2e_ab.py: 1-2 best, 0 = back to back


class HostRoundTrip:
    """Host-owned state between steps: after a step, its results (the device
    tensors) go to pinned host buffers, and the next step's inputs come back
    from those buffers.  Each tensor moves in E2E_CHUNKS chunks: the
    device->host copy of chunk c runs on the compute stream and the
    host->device copy of the same chunk, which reads what that copy wrote,
    on a side stream as soon as it landed -- the two PCIe directions overlap
    (full duplex) instead of running back to back.  Every byte of every step
    still crosses PCIe both ways; the next step waits for the last upload."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.side = torch.cuda.Stream(device=device)
        self.ev = [torch.cuda.Event() for _ in range(64)]

    def upload(self, dev_tensors, host_tensors):
        for d, h in zip(dev_tensors, host_tensors):
            d.copy_(h[:d.shape[0]], non_blocking=True)

    def download(self, dev_tensors, host_tensors):
        for d, h in zip(dev_tensors, host_tensors):
            h[:d.shape[0]].copy_(d, non_blocking=True)

    def round_trip(self, dev_tensors, host_tensors, chunks=None):
        torch = self.torch
        main = torch.cuda.current_stream()
        nch = E2E_CHUNKS if chunks is None else chunks
        if nch <= 0:  # back to back on the compute stream
            self.download(dev_tensors, host_tensors)
            self.upload(dev_tensors, host_tensors)
            return
        k = 0
        for d, h in zip(dev_tensors, host_tensors):
            n = d.shape[0]
            for c in range(nch):
                a, b = n * c // nch, n * (c + 1) // nch
                if b <= a:
                    continue
                h[a:b].copy_(d[a:b], non_blocking=True)
                ev = self.ev[k % len(self.ev)]
                ev.record(main)
                self.side.wait_event(ev)
                with torch.cuda.stream(self.side):
                    d[a:b].copy_(h[a:b], non_blocking=True)
                k += 1
        done = torch.cuda.Event()
        done.record(self.side)
        main.wait_event(done)


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


def scene_cfg4():
    """configs[3]: mixed-dynamics tank, z up.  A 4 x 2 x 2 m box; the pool
    (80 %, ~6.4 M) fills z in [0, 2/3]; the falling block (20 %, ~1.6 M) has
    its bottom at z = 5/3 (1 m above the pool), spans x in [1, 3] and the
    full y width and is flattened to 35 layers (0.33 m) so it fits under
    z = 2; spacing (V_pool / 6.4e6)^(1/3)."""
    from paper_2009_14514_b200 import Scene
    s = (4.0 * 2.0 * (2.0 / 3.0) / 6.4e6) ** (1.0 / 3.0)
    z0 = 5.0 / 3.0
    return Scene(domain_min=(0.0, 0.0, 0.0), domain_max=(4.0, 2.0, 2.0),
                 fluid_boxes=(((0.0, 0.0, 0.0), (4.0, 2.0, 2.0 / 3.0)),
                              ((1.0, 0.0, z0), (3.0, 2.0, z0 + 35 * s))),
                 spacing=s, gravity=(0.0, 0.0, -9.81), eta_max=0.03, eta_avg=0.015,
                 name="cfg4_mixed_tank")


def scene_cfg5(world: int = 1, kind: str = "pcisph"):
    """configs[4]: weak-scaling elongated dam-break tank, 4 M fluid particles
    per GPU: an 8 m x 0.5 m x 1 m column per rank (5,000 per lattice layer
    at s = 0.01) in a (8 N + 1) x 1 x 1 m tank."""
    import math

    from paper_2009_14514_b200 import Scene
    kw = {"eta_max": 0.03, "eta_avg": 0.015} if kind == "pcisph" else {
        "sound_speed": 10.0 * math.sqrt(2.0 * 9.81 * 0.5)}
    return Scene(domain_min=(0.0, 0.0, 0.0), domain_max=(8.0 * world + 1.0, 1.0, 1.0),
                 fluid_boxes=(((0.0, 0.0, 0.0), (8.0 * world, 0.5, 1.0)),), spacing=0.01,
                 name=f"cfg5_weak_{kind}", **kw)


WORKLOADS = {
    "cfg2": ("pcisph", "cfg2: 1M dam break RTS-PCISPH (eta 3%/1.5%, cap 50, dt 1.75e-4, "
                       "4 levels)", "weak"),
    "cfg4": ("pcisph", "cfg4: 8M mixed-dynamics tank RTS-PCISPH (z up, pool 80% + block 20% "
                       "at v0 = (0,0,-2), eta 3%/1.5%, cap 50)", "strong"),
    "cfg5-pcisph": ("pcisph", "cfg5: weak scaling, 4M/GPU elongated tank RTS-PCISPH, "
                              "v0 ~ N(0, 0.1 m/s), eta 3%/1.5%, cap 50", "weak"),
    "cfg5-wcsph": ("wcsph", "cfg5: weak scaling, 4M/GPU elongated tank RTS-WCSPH, "
                            "v0 ~ N(0, 0.1 m/s)", "weak"),
}


def workload_scene(workload: str, world: int = 1):
    if workload == "cfg2":
        return scene_cfg2(world)
    if workload == "cfg4":
        return scene_cfg4()
    return scene_cfg5(world, WORKLOADS[workload][0])


def initial_velocity(workload: str, fluid):
    """(n, 3) float32 initial velocities for the seeded fluid, or None."""
    import numpy as np
    if workload == "cfg4":
        v = np.zeros((len(fluid), 3), dtype=np.float32)
        v[fluid[:, 2] > 1.0, 2] = -2.0  # the falling block
        return v
    if workload.startswith("cfg5"):
        return np.random.default_rng(SEED + 1).normal(0.0, 0.1, (len(fluid), 3)).astype(
            np.float32)
    return None


def jitter_np(n, spacing):
    import numpy as np
    return np.random.default_rng(SEED).uniform(-0.01 * spacing, 0.01 * spacing, (n, 3))


def make_device_solver(kind: str, device, workload: str | None = None):
    """One-GPU solver for ``workload`` (default: cfg2 for "pcisph", cfg3 for
    "wcsph"), seeded lattice + jitter (+ the workload's initial velocities)."""
    import numpy as np
    import torch

    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    if workload is None:
        sc = scene_cfg2() if kind == "pcisph" else scene_cfg3()
    else:
        sc = workload_scene(workload, 1)
    if kind == "pcisph":
        s = PcisphSolver(sc, mode="rts", iteration_cap=50, device=device)
    else:
        s = WcsphSolver(sc, mode="rts", device=device)
    from paper_2009_14514_b200.scene import seed_particles
    nf = s.n_fluid
    lattice = seed_particles(sc)[0]  # fp64 seeds: the oracle jitters the same values
    assert len(lattice) == nf
    x = (lattice + jitter_np(nf, s.scene.spacing)).astype(np.float32)
    s.pos[:nf] = torch.as_tensor(x, device=s.device)
    v0 = initial_velocity(workload, lattice) if workload else None
    if v0 is not None:
        s.vel[:nf] = torch.as_tensor(v0, device=s.device)
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
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    thread polling every 2 ms (a 20-major timed region lasts ~50 ms, too short
    for nvidia-smi's loop), falling back to ``nvidia-smi -lms 5``."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.gpu = gpu_index
        self.period = period_s
        self.proc = None
        self.thread = None
        self.samples: list = []
        self.path = os.path.join("/tmp", f"rts_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self._nv, self._h = nv, h
            self._max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._stop = threading.Event()

            def poll():
                get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                                getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
                while not self._stop.is_set():
                    try:
                        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                             get_r(h) if get_r else 0))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader",
                 "-lms", "5"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    @staticmethod
    def _summary(sm, mx, reasons, how) -> dict:
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["no samples"], "how": how}
        loaded = sorted(v for v in sm if v > 0.5 * max(sm)) or sorted(sm)
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "how": how}

    def stop(self) -> dict:
        if self.thread is not None:
            self._stop.set()
            self.thread.join()
            nv = self._nv
            reasons = set()
            for _, r in self.samples:
                for name, attr in self.REASONS:
                    if r & getattr(nv, attr, 0):
                        reasons.add(name)
            return self._summary([c for c, _ in self.samples], self._max, reasons,
                                 f"NVML poll every {self.period * 1e3:g} ms")
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = [n for n, _ in self.REASONS]
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
        return self._summary(sm, max(mx) if mx else None, reasons, "nvidia-smi -lms 5")


METRICS = {
    "cfg2": METRIC,
    "cfg4": "particle-updates/s (RTS-PCISPH, 8M mixed tank, minor steps)",
    "cfg5-pcisph": "particle-updates/s (RTS-PCISPH, 4M/GPU elongated tank, minor steps)",
    "cfg5-wcsph": "particle-updates/s (RTS-WCSPH, 4M/GPU elongated tank, base steps)",
}


def _oracle_for(workload: str, world: int = 1):
    """The CPU oracle on the workload's scene at ``world`` ranks (the whole
    scene the N-GPU run simulates), jittered (and with the workload's initial
    velocities) exactly as the device solver."""
    import numpy as np

    from oracle import sph as O
    kind = WORKLOADS[workload][0]
    sc = workload_scene(workload, world)
    if kind == "pcisph":
        o = O.OraclePcisph(sc, mode="rts", iteration_cap=50)
    else:
        o = O.OracleWcsph(sc, mode="rts")
    nf = o.n_fluid
    lattice = o.pos[:nf].copy()
    x = (lattice + jitter_np(nf, sc.spacing)).astype(np.float32).astype(np.float64)
    o.pos[:nf] = x
    v0 = initial_velocity(workload, lattice) if workload != "cfg2" else None
    if v0 is not None:
        o.vel[:nf] = v0.astype(np.float64)
    if kind == "pcisph":
        o.xstar[:] = x
    return o, O


def _oracle_steps(o, budget_s: float, max_steps: int):
    """Timed steps (advance() = one major for PCISPH, one base step for
    WCSPH) until ``budget_s`` seconds or ``max_steps`` steps."""
    import time as _t
    units, steps = 0, 0
    t0 = _t.perf_counter()
    while steps < max_steps:
        units += len(o.advance())
        steps += 1
        if _t.perf_counter() - t0 > budget_s:
            break
    return units, steps, _t.perf_counter() - t0


def cpu_oracle_sample(majors: int = 2, warm: int = 1, workload: str = "cfg2") -> dict:
    """Time the CPU oracle (fp64 C + numpy restatement of the reference) on
    the same scene: ``warm`` untimed steps, then up to ``majors`` timed
    (bounded to ~20 s of CPU work)."""
    t_setup = time.perf_counter()
    o, O = _oracle_for(workload)
    nf = o.n_fluid
    for _ in range(warm):
        o.advance()
    t0 = time.perf_counter()
    units, steps, dt = _oracle_steps(o, 20.0, majors)
    what = "major steps" if WORKLOADS[workload][0] == "pcisph" else "base steps"
    return {"value": nf * units / dt, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
            "sample": f"{steps} {what} ({units} updates of every particle) of the "
                      f"{workload} one-GPU scene ({nf} fluid) after {warm} untimed; "
                      "oracle = fp64 C/OpenMP + numpy restatement",
            "seconds": round(dt, 3), "setup_s": round(t0 - t_setup, 1)}


def bench_config(workload: str, world: int, n_fluid: int, n_boundary: int) -> dict:
    """The ``config`` of both arms' JSON line: the workload only (scene,
    sizes, step unit), so the two lines compare like for like."""
    kind, wl_name, _ = WORKLOADS[workload]
    return {"workload": wl_name, "n_fluid": n_fluid, "n_boundary": n_boundary,
            "bench_step": ("one major step (advance(): up to 4 minor steps)" if kind == "pcisph"
                           else "4 base steps (step())"),
            "scene_ranks": world, "seed": SEED, "jitter": "+-1% of spacing",
            "l2": "working set > L2 (state, tables) -- no flush needed"}


def run_reference_arm(args, rank: int, world: int) -> None:
    """The reference path on the host: the CPU oracle (fp64 C/OpenMP
    restatement of the reference's numba kernels + numpy bookkeeping, all
    host threads) on the same scene, the same --warmup and --steps (the
    N-rank scenes: as many steps as fit RTS_REF_BUDGET_S seconds)."""
    if rank != 0:
        return
    kind, wl_name, scaling = WORKLOADS[args.workload]
    o, O = _oracle_for(args.workload, world)
    nf = o.n_fluid
    per_step = 1 if kind == "pcisph" else 4  # a WCSPH bench step = 4 base steps
    for _ in range(args.warmup * per_step):
        o.advance()
    # the full --steps when they fit the wall budget (N = 1: ~2 min); the
    # N-rank scenes (N M particles) stop at the budget, a bounded sample
    budget = float(os.environ.get("RTS_REF_BUDGET_S", "240"))
    t0 = time.perf_counter()
    units, steps = 0, 0
    while steps < args.steps and (steps == 0 or time.perf_counter() - t0 < budget):
        for _ in range(per_step):
            units += len(o.advance())
        steps += 1
    dt = time.perf_counter() - t0
    v = nf * units / dt
    what = (f"the full run: {steps} bench steps" if steps == args.steps else
            f"a bounded sample: {steps} of the {args.steps} requested bench steps "
            f"(wall budget {budget:g} s)")
    line = {
        "impl": "reference", "metric": METRICS[args.workload], "value": v, "unit": UNIT,
        "n_gpus": world, "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / max(1, steps),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args.workload, world, nf, len(o.pos) - nf),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
                         "sample": f"{what} ({units} updates of each of {nf} particles) after "
                                   f"{args.warmup} untimed; CPU oracle restating the reference"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_threads": O.num_threads(),
    }
    print(json.dumps(line), flush=True)


def wcsph_algo_bytes(name: str, nf: int, active: int, launches: int) -> float:
    """SURVEY.md section 8(d) RTS-WCSPH bytes: density + Tait 20 per active
    particle, forces + bookkeeping 88 per active, predictor 68 per particle
    + corrector 16 per active, level propagation 15 per particle."""
    if name == "rts_wcsph_density":
        return 20.0 * active
    if name == "rts_wcsph_forces":
        return 88.0 * active
    if name == "rts_wcsph_integrate":
        return 68.0 * nf * launches + 16.0 * active
    if name == "rts_wcsph_propagate":
        return 15.0 * nf * launches
    return 0.0


def wcsph_comparison(world: int, device, stream, barrier) -> dict:
    """configs[2]: RTS-WCSPH on the 1M dam break against the global adaptive
    baseline (CFL step, dt_cap = 4 dt_base), per
    simulated time.  N > 1: the same scene cut into N x-slab ranks (strong
    scaling), device time max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2009_14514_b200 import WcsphSolver

    def make(mode: str):
        sc = scene_cfg3()
        if world == 1:
            if mode == "rts":
                return make_device_solver("wcsph", device), None
            s = WcsphSolver(sc, mode=mode, device=device)
            nf = s.n_fluid
            x = (s.host("pos")[:nf] + jitter_np(nf, sc.spacing)).astype("float32")
            s.pos[:nf] = torch.as_tensor(x, device=s.device)
            return s, s
        from paper_2009_14514_b200.distributed import DistributedWcsph
        from paper_2009_14514_b200.scene import seed_particles
        n = len(seed_particles(sc)[0])
        d = DistributedWcsph(sc, mode=mode, device=device, jitter=jitter_np(n, sc.spacing))
        return d, d.solver

    def timed(drv, steps: int):
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fr, sim = 0.0, 0.0
        for _ in range(steps):
            st = drv.step()
            fr += st.n_compute
            sim += st.dt
        b.record(stream)
        b.synchronize()
        t = a.elapsed_time(b) * 1e-3
        if world > 1:
            v = torch.tensor([t], dtype=torch.float64, device=device)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            t = float(v.item())
            c = torch.tensor([fr], dtype=torch.float64, device=device)
            dist.all_reduce(c)
            fr = float(c.item())
        return t, fr, sim

    n_w = 40
    ws, _ = make("rts")
    for _ in range(8):
        ws.step()
    tw, act, sim_rts = timed(ws, n_w)
    n_total = ws.n_global if world > 1 else ws.n_fluid
    wc = {"metric": "particle-updates/s (RTS-WCSPH, 1M, base steps)",
          "value": n_total * n_w / tw, "ms_per_step": 1e3 * tw / n_w,
          "mean_active_fraction": act / (n_total * n_w), "steps": n_w,
          "wall_s_per_simulated_ms": tw / (1e3 * sim_rts), "n_gpus": world,
          "scaling": "strong" if world > 1 else None}
    del ws
    # the global baseline (wcsph.py:199-233, every particle every step) at both
    # caps BASELINE.md section 2 reports: dt_cap = 4 dt_base (CFL-adaptive,
    # mean dt ~4 dt_base on this calm start) and the reference's default
    # dt_cap = dt_base (wcsph.py:143-144: a constant dt_base step)
    for key, cap in (("baseline_adaptive", 4.0), ("baseline_default_cap", 1.0)):
        wb, solver = make("baseline")
        solver.dt_cap = cap * solver.dt_base
        for _ in range(4):
            wb.step()
        tb, _, sim_b = timed(wb, n_w // 2)
        wc[key] = {
            "dt_cap_over_dt_base": cap,
            "ms_per_step": 1e3 * tb / (n_w // 2), "mean_dt": sim_b / (n_w // 2),
            "wall_s_per_simulated_ms": tb / (1e3 * sim_b),
            "rts_speedup_per_simulated_time": (tb / sim_b) / (tw / sim_rts)}
        del wb, solver
    return wc


def run_wcsph_workload(args, rank: int, world: int, device, barrier) -> None:
    """RTS-WCSPH bench line (cfg5-wcsph): K base steps, device time, max over
    ranks; roofline of the dominant kernel from an instrumented pass."""
    import torch
    import torch.distributed as dist

    from paper_2009_14514_b200 import _native
    _, wl_name, scaling = WORKLOADS[args.workload]
    if world == 1:
        solver = make_device_solver("wcsph", device, args.workload)
        driver = solver
        n_total = solver.n_fluid
        n_bound_total = solver.n_bound
    else:
        from paper_2009_14514_b200.distributed import DistributedWcsph
        from paper_2009_14514_b200.scene import seed_particles
        sc = workload_scene(args.workload, world)
        lattice, walls = seed_particles(sc)
        n_total, n_bound_total = len(lattice), len(walls)
        driver = DistributedWcsph(sc, device=device, jitter=jitter_np(n_total, sc.spacing),
                                  velocity=initial_velocity(args.workload, lattice),
                                  rebalance_every=args.rebalance)
        solver = driver.solver
    stream = torch.cuda.current_stream(device)
    steps = args.steps * 4  # one bench step = 4 base steps (a major's worth)
    for _ in range(args.warmup * 4):
        driver.step()
    torch.cuda.synchronize()
    clocks = ClockSampler(device.index or 0)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = _native.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    rows = [driver.step() for _ in range(steps)]
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    clk = clocks.stop()
    t = ev0.elapsed_time(ev1) * 1e-3
    if world > 1:
        tt = torch.tensor([t], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    value = n_total * steps / t

    kernels = ["rts_wcsph_propagate", "rts_wcsph_density", "rts_wcsph_forces",
               "rts_wcsph_integrate", "rts_block_levels"]
    solver.time_kernels(kernels)
    prof = [driver.step() for _ in range(8)]
    torch.cuda.synchronize()
    totals = {k: sum(solver.kernel_times(k)) for k in kernels}
    counts = {k: len(solver.kernel_times(k)) for k in kernels}
    solver._ktimes = None
    nf_local = solver.n_fluid
    active = sum(int(r.n_compute) for r in prof)
    dom = max(totals, key=totals.get)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    alg = wcsph_algo_bytes(dom, nf_local, active, counts[dom])
    ach = alg / max(totals[dom], 1e-12) / 1e9
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": None, "kernel": dom,
                "launches": counts[dom], "kernel_s": round(totals[dom], 6),
                "algorithmic_bytes": alg,
                "share_of_step": round(totals[dom] / max(1e-12, sum(totals.values())), 3),
                "kernels": {k: {"s": round(totals[k], 6), "launches": counts[k],
                                "achieved_gbs": round(wcsph_algo_bytes(k, nf_local, active,
                                                                       counts[k]) /
                                                      max(totals[k], 1e-12) / 1e9, 1)}
                            for k in kernels if counts[k]},
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}

    e2e = None
    if not args.no_e2e:
        def dev_state():
            if world == 1:
                return solver.pos[:solver.n_fluid], solver.vel
            return driver.state["pos"], driver.state["vel"]
        k_e2e = 16
        cap = 2 * dev_state()[0].shape[0] + 1024
        hp = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        hv = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        dp, dv = dev_state()
        hp[:dp.shape[0]].copy_(dp)
        hv[:dv.shape[0]].copy_(dv)
        nbytes = 0
        rt = HostRoundTrip(device)
        rt.upload(dev_state(), (hp, hv))  # one untimed e2e step first
        driver.step()
        rt.download(dev_state(), (hp, hv))
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        rt.upload(dev_state(), (hp, hv))  # the first step's inputs
        for k in range(k_e2e):
            n = dev_state()[0].shape[0]
            driver.step()
            dp, dv = dev_state()
            n2 = dp.shape[0]
            if k + 1 < k_e2e:  # results down, next step's inputs up (overlapped)
                rt.round_trip((dp, dv), (hp, hv))
            else:
                rt.download((dp, dv), (hp, hv))
            nbytes = (n + n2) * 24
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], device=device, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": n_total * k_e2e / te, "unit": UNIT,
               "h2d_bytes_per_step": nbytes // 2, "d2h_bytes_per_step": nbytes // 2,
               "steps": k_e2e, "note": "pinned host pos+vel uploaded before and downloaded "
                                       "after every step() (chunked, the two PCIe directions "
                                       "overlapped: HostRoundTrip); wall clock"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_oracle_sample(majors=8, warm=1, workload=args.workload)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "error": repr(exc)}
    if rank == 0:
        line = {
            "metric": METRICS[args.workload], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": bench_config(args.workload, world, n_total, n_bound_total),
            "run": {"base_steps": steps,
                    "mean_active_fraction": round(sum(r.frac_compute for r in rows) /
                                                  max(1, len(rows)), 4),
                    "parallelism": ("single GPU" if world == 1 else
                                    f"x-slabs x{world} (ghost exchange + migration)"),
                    "arithmetic": "fp32 particle state; fp64 pair terms and sums"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
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
    ap.add_argument("--rebalance", type=int, default=0,
                    help="x-slab ranks: re-cut by work every K majors (WCSPH: base steps)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="cfg2 (default, the headline) or the BASELINE configs[3..4] "
                         "workloads")
    args = ap.parse_args()
    kind, wl_name, scaling = WORKLOADS[args.workload]

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

    if kind == "wcsph":
        run_wcsph_workload(args, rank, world, device, barrier)
        if world > 1:
            dist.destroy_process_group()
        return

    if world == 1:
        solver = make_device_solver("pcisph", device, args.workload)
        driver = solver
        n_total = solver.n_fluid
        n_bound_total = solver.n_bound
    else:  # x-slab decomposition (paper_2009_14514_b200/distributed.py)
        from paper_2009_14514_b200.distributed import DistributedPcisph
        from paper_2009_14514_b200.scene import seed_particles
        sc = workload_scene(args.workload, world)
        lattice, walls = seed_particles(sc)
        n_total, n_bound_total = len(lattice), len(walls)
        driver = DistributedPcisph(sc, device=device, jitter=jitter_np(n_total, sc.spacing),
                                   velocity=initial_velocity(args.workload, lattice),
                                   iteration_cap=50, rebalance_every=args.rebalance)
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
    traffic = None  # ncu DRAM bytes per launch: captured for the default workload only
    l1 = {}  # ncu L1 LSU data-pipe utilisation (% of peak) per kernel, same capture
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf) and args.workload == "cfg2" and world == 1:
        tj = json.load(open(tf))
        traffic = tj.get(dom)
        l1 = {k: tj[k + "_l1_wavefront_pct"] for k in kernels if k + "_l1_wavefront_pct" in tj}
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
    if l1:  # the gather kernels' own bound: wavefronts of the L1 LSU data pipe
        roofline["l1_wavefront_pct"] = l1.get(dom)
        roofline["l1_wavefront_pct_by_kernel"] = l1
        roofline["l1_note"] = ("ncu l1tex__data_pipe_lsu_wavefronts % of peak (profiles/"
                               "ncu_traffic.json): the neighbour gathers touch ~10 128-byte "
                               "lines per warp request, so these kernels are bound by L1 "
                               "wavefronts, not HBM bytes (DESIGN.md section 4)")
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
        # go up before and come back after every advance().  One GPU: a fresh
        # solver from the same seeded start runs the same W + K majors as the
        # device-timed region (the e2e number covers the same stretch of the
        # simulation as `value` and the reference arm); x-slab ranks: K' =
        # min(K, 10) majors of the running decomposition.
        e_solver = None
        if world == 1:
            e_solver = make_device_solver("pcisph", device, args.workload)
            e_driver = e_solver
        else:
            e_driver = driver

        def dev_state():
            if world == 1:
                return e_solver.pos[:e_solver.n_fluid], e_solver.vel
            return driver.state["pos"], driver.state["vel"]
        k_e2e = args.steps if world == 1 else max(2, min(args.steps, 10))
        w_e2e = args.warmup if world == 1 else 1
        cap = 2 * dev_state()[0].shape[0] + 1024
        hp_all = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        hv_all = torch.empty((cap, 3), dtype=torch.float32).pin_memory()
        dp, dv = dev_state()
        hp_all[:dp.shape[0]].copy_(dp)
        hv_all[:dv.shape[0]].copy_(dv)
        e_minors = 0
        nbytes = 0
        rt = HostRoundTrip(device)
        # untimed e2e warm-up steps first (x-slab ranks: the graphs were last
        # launched before the host-driven instrumented pass above)
        for _ in range(w_e2e):
            rt.upload(dev_state(), (hp_all, hv_all))
            e_driver.advance()
            rt.download(dev_state(), (hp_all, hv_all))
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        rt.upload(dev_state(), (hp_all, hv_all))  # the first step's inputs: host -> device
        for k in range(k_e2e):
            n = dev_state()[0].shape[0]
            e_minors += len(e_driver.advance())
            dp, dv = dev_state()  # results (ownership may have changed)
            n2 = dp.shape[0]
            if k + 1 < k_e2e:  # results down, next step's inputs up (overlapped)
                rt.round_trip((dp, dv), (hp_all, hv_all))
            else:
                rt.download((dp, dv), (hp_all, hv_all))
            nbytes = (n + n2) * 24
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], device=device, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": n_total * e_minors / te, "unit": UNIT,
               "h2d_bytes_per_step": nbytes // 2, "d2h_bytes_per_step": nbytes // 2,
               "steps": k_e2e, "warmup": w_e2e,
               "note": ("pinned host pos+vel uploaded before and downloaded after every "
                        "advance() (the two PCIe directions overlapped: HostRoundTrip); wall "
                        "clock; " + ("a fresh solver over the same W + K majors as `value`"
                                     if world == 1 else "min(K, 10) majors after the timed region"))}
        del e_solver

    # ---- WCSPH extra (configs[2]: the 1M scene, RTS-WCSPH vs the global -------
    # adaptive baseline; one GPU, or the same scene cut into N x-slab ranks)
    wc = None
    if not args.no_wcsph and args.workload == "cfg2":
        wc = wcsph_comparison(world, device, stream, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_oracle_sample(workload=args.workload)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRICS[args.workload], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": bench_config(args.workload, world, nf, n_bound_total),
            "run": {"minor_steps": minors,
                    "iterations_per_minor": round(sum(r.iterations for r in rows) /
                                                  max(1, minors), 3),
                    "corrected_per_minor_over_nf": round(sum(r.corrected for r in rows) /
                                                        max(1, minors) / nf, 3),
                    "parallelism": ("single GPU" if world == 1 else
                                    f"x-slabs x{world} (ghost exchange + allreduce)"),
                    "arithmetic": "fp32 particle state; fp64 x*, p, pair terms and sums"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "wcsph_rts_1m": wc,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
