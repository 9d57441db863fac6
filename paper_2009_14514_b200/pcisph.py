"""RTS-PCISPH on the B200 -- drop-in for ``rts_sph.pcisph.PcisphSolver``
(/root/reference/pkg/src/rts_sph/pcisph.py:279-768; Algorithms 2-3 of
arXiv 2009.14514) and its constant / globally adaptive baselines.

Control flow (major step -> minor steps -> scheduled correction loop with
S_e / S_ob sets, local phases with snapshot/revert, early termination and
the iteration cap) is the reference's, driven from the host; every
particle and block pass is a librtssph kernel (see csrc/pcisph.cu).  The
host reads one small counters block per correction iteration (max err,
sum rho*, any S_e, |pred|) to take the reference's convergence decisions.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from . import _native as N
from ._device import raise_on_errors
from .errors import ConfigError, NumericalError
from .scene import Scene
from .stats import StepStats
from .wcsph import NEIGHBOR_WIDTH, _DeviceSolver

__all__ = ["PcisphSolver", "MajorStepController", "DEFAULT_SCHEDULE", "VALIDITY_PERIOD",
           "validate_schedule", "pci_delta"]

# refresh period in minor steps by region id (pcisph.py:63-66)
VALIDITY_PERIOD = np.array([0, 1, 2, 4, 4], dtype=np.int32)

# one tuple per minor step, one inner tuple of scheduled regions per
# correction iteration (pcisph.py:68-77)
DEFAULT_SCHEDULE = (
    ((1, 2, 3, 4), (1, 2, 3, 4), (1,)),
    ((1, 2, 3, 4), (1,), (1,)),
    ((1, 2, 3, 4), (1, 2), (1,)),
    ((1, 2, 3, 4), (1,), (1,)),
)


def validate_schedule(schedule, n_regions: int = 4) -> None:
    """The five legality rules of pcisph.py:80-117; ConfigError on failure."""
    n_minor = len(schedule)
    tally = np.zeros((n_minor, n_regions + 1), dtype=int)
    for j, rows in enumerate(schedule):
        for row in rows:
            for n in row:
                if not 1 <= n <= n_regions:
                    raise ConfigError(f"schedule names region {n} outside 1..{n_regions}")
                tally[j, n] += 1
    for j in range(n_minor):
        for n in range(1, n_regions + 1):
            if tally[j, n] < 1:
                raise ConfigError(f"region {n} receives no iteration on minor step {j + 1}")
    for n in range(1, n_regions + 1):
        if tally[0, n] < 2:
            raise ConfigError(
                f"region {n} receives fewer than 2 iterations on the first minor step")
    for j in range(n_minor):
        if tally[j, 1] < 3:
            raise ConfigError(f"region 1 receives fewer than 3 iterations on minor step {j + 1}")
    for n in range(1, n_regions + 1):
        window = 2 if n == 2 else min(n, n_minor)
        for j in range(n_minor):
            total = sum(tally[(j + q) % n_minor, n] for q in range(window))
            if total < 3:
                raise ConfigError(f"region {n} receives {total} < 3 iterations in the "
                                  f"{window}-minor window starting at minor step {j + 1}")


def _template_factor(h: float, spacing: float) -> float:
    """|sum grad W|^2 + sum |grad W|^2 over the filled lattice neighbourhood
    (pcisph.py:131-148)."""
    c_spiky = -45.0 / (math.pi * h**6)
    g_sum = np.zeros(3)
    g_dot = 0.0
    reach = int(math.ceil(h / spacing))
    rng = range(-reach, reach + 1)
    for ix in rng:
        for iy in rng:
            for iz in rng:
                if ix == 0 and iy == 0 and iz == 0:
                    continue
                off = np.array([ix, iy, iz]) * spacing
                r = math.sqrt(float(off @ off))
                if r >= h:
                    continue
                d = h - r
                g = (c_spiky * d * d / r) * (-off)
                g_sum += g
                g_dot += float(g @ g)
    return float(g_sum @ g_sum) + g_dot


def pci_delta(scene: Scene, dt: float) -> float:
    """Pressure stiffness per unit density error (pcisph.py:120-128)."""
    f = _template_factor(scene.support_radius, scene.spacing)
    m = scene.particle_mass
    return scene.rest_density**2 / (2.0 * dt * dt * m * m * f)


@dataclasses.dataclass
class MajorStepController:
    """Halves the major step for ten majors after an early termination
    (pcisph.py:151-166)."""

    n_nominal: int = 4
    n_current: int = 4
    recovery_left: int = 0

    def note_major(self, early_terminated: bool) -> None:
        if early_terminated:
            self.n_current = 2
            self.recovery_left = 10
        elif self.recovery_left > 0:
            self.recovery_left -= 1
            if self.recovery_left == 0:
                self.n_current = self.n_nominal


def _row_mask(row) -> int:
    m = 0
    for n in row:
        if 0 <= n < 31:
            m |= 1 << n
    return m


class PcisphSolver(_DeviceSolver):
    """PCISPH with ``mode`` "const", "adaptive" or "rts" (pcisph.py:279)."""

    mode_names = ("const", "adaptive", "rts")

    def __init__(self, scene: Scene, mode: str = "rts", dt: float | None = None,
                 schedule=DEFAULT_SCHEDULE, pin_region: int | None = None,
                 audit_neighbors: bool = False, iteration_cap: int = 24,
                 local_attempts: int = 4, n_regions: int = 4, device="cuda"):
        if mode not in self.mode_names:
            raise ValueError(f"unknown pcisph mode {mode!r}")
        validate_schedule(schedule, n_regions)
        self.mode = mode
        self.schedule = schedule
        self.pin_region = pin_region
        self.audit_neighbors = audit_neighbors
        self.iteration_cap = iteration_cap
        self.local_attempts = local_attempts
        self.n_regions = n_regions
        self._setup_common(scene, "pcisph" if mode == "rts" else "wcsph", device)
        if dt is not None:
            self.dt = dt
        elif mode == "const":
            self.dt = scene.const_dt()
        else:
            self.dt = scene.base_dt("pcisph")
        self.inv_mass = 1.0 / self.mass
        self._set_betas(n_regions, scene.alpha_for("pcisph"))
        self.controller = MajorStepController(scene.minor_steps, scene.minor_steps)
        self._delta_factor = _template_factor(self.kernel.h, scene.spacing)
        nf = self.n_fluid
        n1 = max(nf, 1)
        A = self.arena
        f32 = torch.float32
        self.vel = A.alloc("vel", (n1, 3), f32, 0)[:nf]
        self.f_ext = A.alloc("force", (n1, 3), f32, 0)[:nf]
        self.f_p = A.alloc("f_p", (n1, 3), f32, 0)[:nf]
        self.p = A.alloc("pres", (n1,), f32, 0)[:nf]
        self.rho_star = A.alloc("rho", (n1,), f32, scene.rest_density)[:nf]
        self.err = A.alloc("err", (n1,), torch.float64, 0)[:nf]
        self.xstar = A.alloc("xstar", (n1, 3), f32, 0)[:nf]
        self.xstar.copy_(self.pos[:nf])
        self.region = A.alloc("region", (n1,), torch.int8, 1)[:nf]
        self.validity = A.alloc("validity", (n1,), torch.int32, 0)[:nf]
        self.compute = A.alloc("compute", (n1,), torch.bool, True)[:nf]
        self.in_se = A.alloc("in_se", (n1,), torch.bool, False)[:nf]
        self.in_sob = A.alloc("in_sob", (n1,), torch.bool, False)[:nf]
        self._nbr = A.alloc("nbr", (n1, NEIGHBOR_WIDTH), torch.int32, 0)
        self.cnt = A.alloc("cnt", (n1,), torch.int32, 0)[:nf]
        A.alloc("xs4", (max(nf + self.n_bound, 1), 4), f32, 0)
        A.alloc("pflag", (n1,), torch.uint8, 0)
        A.alloc("partial", (4096,), torch.float64, 0)
        A.alloc("snap_p", (n1,), f32, 0)
        A.alloc("snap_fp", (n1, 3), f32, 0)
        A.alloc("slot_of", (n1,), torch.int32, 0)
        self.local_entered_total = 0
        self.local_reverted_total = 0
        self._force_total = 0
        p = self.params
        p.dt_base = self.dt
        p.use_sound = 0
        p.rts = 1 if mode == "rts" else 0
        stream = torch.cuda.current_stream(self.device)
        N.call("rts_pci_walls", p, A.buf, stream.cuda_stream)

    # -- reference-facing helpers -------------------------------------------
    @property
    def block_region(self) -> torch.Tensor:
        return self.arena["block_field"]

    @property
    def nbr(self) -> torch.Tensor:
        return self._nbr[: self.n_fluid]

    def delta(self, dt: float) -> float:
        rho0 = self.scene.rest_density
        return rho0 * rho0 / (2.0 * dt * dt * self.mass * self.mass * self._delta_factor)

    def particle_regions(self) -> torch.Tensor:
        if self.mode == "rts":
            return self.region
        return torch.ones(self.n_fluid, dtype=torch.int8, device=self.device)

    def advance(self) -> list[StepStats]:
        if self.mode == "rts":
            return self.major_step()
        return [self.sync_step()]

    # -- plumbing -------------------------------------------------------------
    def _stream(self):
        return torch.cuda.current_stream(self.device)

    def _call(self, name, *args):
        self._launch(name, *args)

    def _prepare(self, dt: float) -> None:
        self._sync_params()
        p = self.params
        sc = self.scene
        p.dt = dt
        p.delta = self.delta(dt)
        p.eta_max, p.eta_avg, p.rho_T = sc.eta_max, sc.eta_avg, sc.rho_T
        p.pin_region = int(self.pin_region or 0)

    def _read(self) -> N.RtsCounters:
        c = self.counters.read(self._stream())
        self.grid.n_sorted = int(c.n_sorted)
        self._raise(c)
        return c

    def _raise(self, c) -> None:
        if c.err_flags & N.ERR_NONFINITE and not c.err_flags & (N.ERR_ESCAPED | N.ERR_OVERFLOW):
            raise NumericalError("non-finite predicted density; the simulation has blown up")
        raise_on_errors(c, NEIGHBOR_WIDTH)

    def _avg_from(self, c) -> float:
        if not self.n_fluid:
            return 0.0
        mean = float(c.sum_rho) / self.n_fluid
        return max(0.0, mean / self.scene.rest_density - 1.0)

    def _rebuild(self, want_maxima: bool) -> None:
        self.counters.reset(self._stream())
        self.grid.launch_rebuild(self.params, self._stream(), want_maxima=want_maxima,
                                 add_fp=True)
        self._call("rts_pci_gather")

    def _zero_pressure(self) -> None:
        s = self._stream().cuda_stream
        nf = self.n_fluid
        N.call("rts_memset", self.arena.buf.pres, 0, 4 * nf, s) if nf else None
        N.call("rts_memset", self.arena.buf.f_p, 0, 12 * nf, s) if nf else None

    # -- synchronous baselines (pcisph.py:376-476) ------------------------------
    def sync_step(self) -> StepStats:
        nf = self.n_fluid
        dt = self.dt
        self._prepare(dt)
        tm = self.timer
        st = self._stream()
        self._rebuild(False)
        tm.start(st)
        self._call("rts_pci_refresh", 1, 0)
        tm.mark("neighbor", st)
        self._zero_pressure()
        it = corrected = 0
        while True:
            self._call("rts_pci_motion", 1)
            self._call("rts_pci_sets", 0, 1)
            self._call("rts_pci_density")
            self._call("rts_pci_se_reduce", 0)
            self._call("rts_pci_pforces")
            c = self._read()
            it += 1
            corrected += nf
            max_err = float(c.max_err)
            avg_err = self._avg_from(c)
            if it >= 3 and max_err < self.scene.eta_max and avg_err < self.scene.eta_avg:
                break
            if it > self.iteration_cap + 3:
                raise NumericalError(
                    f"pressure solve did not converge within {it} iterations "
                    f"(max error {max_err:.4%} of rest density)")
        self._call("rts_pci_integrate", 0)
        tm.mark("physics", st)
        c = self._read()
        self.grid.n_sorted = int(c.n_sorted)
        if self.mode == "adaptive":
            self._adapt_dt(it)
        self.step_index += 1
        self.sim_time += dt
        t = tm.totals()
        return StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=nf,
                         frac_compute=1.0, iterations=it, corrected=corrected, iters_r1=it,
                         iters_r2=it, iters_r3=it, iters_r4=it, max_err=max_err,
                         avg_err=avg_err, t_neighbor=t["neighbor"], t_physics=t["physics"],
                         t_rts=t["rts"])

    def _vel_max(self) -> float:
        if not self.n_fluid:
            return 0.0
        st = self._stream()
        self.counters.reset(st)
        self._call("rts_vel_max")
        c = self.counters.read(st)
        return float(np.array([c.fmax_bits], dtype=np.uint64).view(np.float64)[0])

    def _adapt_dt(self, iters: int) -> None:
        """pcisph.py:470-476."""
        v_max = self._vel_max()
        cfl_ok = v_max * self.dt <= 0.4 * self.kernel.h
        if iters <= 5 and cfl_ok:
            self.dt = min(self.dt * 1.002, 2.0 * self.scene.base_dt("pcisph"))
        else:
            self.dt = max(self.dt * 0.8, 0.1 * self.scene.const_dt())

    # -- regional mode (pcisph.py:482-768) -----------------------------------
    def major_step(self) -> list[StepStats]:
        n_minor = self.controller.n_current
        self._prepare(self.dt)
        self._rebuild(True)
        self._assign_major_regions(n_minor, rebuilt=True)
        rows = []
        early = False
        for j in range(n_minor):
            st = self._minor_step(j, self.schedule[j], last=(j == n_minor - 1))
            rows.append(st)
            if st.early_term:
                early = True
                break
        self.controller.note_major(early)
        return rows

    def _assign_major_regions(self, n_minor: int, rebuilt: bool = False) -> None:
        """Block levels at major start (pcisph.py:507-535): maxima of |v| and
        |f_ext + f_p| (from the rebuild pass, or recomputed), assign with
        n_max = min(n_regions, n_minor), smooth, expand regions 1/2."""
        self._prepare(self.dt)
        if not rebuilt:
            self._call("rts_block_maxima", 1)
        p = self.params
        p.n_max = min(self.n_regions, n_minor)
        self._call("rts_block_levels", 1)
        self._call("rts_pci_major_particles")
        self._call("rts_pci_observed", 0)
        self._call("rts_pci_sob")
        if not rebuilt:
            self._raise(self.counters.read(self._stream()))

    def _minor_step(self, j: int, rows, last: bool) -> StepStats:
        nf = self.n_fluid
        dt = self.dt
        self._prepare(dt)
        st = self._stream()
        tm = self.timer
        tm.start(st)
        self._call("rts_pci_refresh", 0, 1)
        tm.mark("neighbor", st)
        missed = 0
        if self.audit_neighbors:
            missed = self._audit_refresh()
            self.missed_neighbors_total += missed
        self._zero_pressure()
        iters, corrected, riters, early, c_last = self._correct_scheduled(dt, rows)
        self._call("rts_pci_integrate", 1)
        tm.mark("physics", st)
        if not last:
            self._mark_timestep_updates(launch_only=True)
        tm.mark("rts", st)
        c = self._read()
        n_refresh = int(self._n_refresh)
        self.step_index += 1
        self.sim_time += dt
        t = tm.totals()
        return StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=n_refresh,
                         frac_compute=n_refresh / max(1, nf), iterations=iters,
                         corrected=corrected, iters_r1=riters[1], iters_r2=riters[2],
                         iters_r3=riters[3], iters_r4=riters[4], max_err=float(c_last.max_err),
                         avg_err=self._avg_from(c_last), early_term=int(early),
                         missed_neighbors=missed, t_neighbor=t["neighbor"],
                         t_physics=t["physics"], t_rts=t["rts"])

    def _correct_scheduled(self, dt: float, rows):
        sc = self.scene
        s = self._stream().cuda_stream
        N.call("rts_memset", self.arena.buf.in_se, 0, self.n_fluid, s) if self.n_fluid else None
        self._call("rts_pci_observed", 0)
        it = g_count = corrected = 0
        riters = [0, 0, 0, 0, 0]
        local_active = local_banned = False
        local_run = 0
        early = False
        motion_all = True
        first = True
        while True:
            if local_active:
                mask = 0
            else:
                row = rows[g_count % len(rows)]
                mask = _row_mask(row)
                for n in row:
                    if n <= self.n_regions:
                        riters[n] += 1
            self._call("rts_pci_motion", int(motion_all))
            self._call("rts_pci_sets", mask, 0)
            self._call("rts_pci_density")
            self._call("rts_pci_se_reduce", 1)
            self._call("rts_pci_observed", 1)
            self._call("rts_pci_pforces")
            c = self._read()
            if first:
                self._n_refresh = int(c.n_compute)
                first = False
            motion_all = False
            it += 1
            corrected += int(c.n_pred)
            self._force_total += int(c.n_force)
            if local_active:
                local_run += 1
            else:
                g_count += 1
            max_err = float(c.max_err)
            avg_err = self._avg_from(c)
            if max_err < sc.eta_max and avg_err < sc.eta_avg:
                if it >= 3:
                    break
                continue
            if it < 3:
                continue
            if local_active:
                if local_run >= self.local_attempts:
                    self._call("rts_pci_snapshot", 1)
                    motion_all = True
                    local_active = False
                    local_banned = True
                    self.local_reverted_total += 1
            elif avg_err * 100.0 < sc.rho_T and not local_banned and c.any_se:
                local_active = True
                local_run = 0
                self._call("rts_pci_snapshot", 0)
                self.local_entered_total += 1
            if g_count > 6:
                early = True
            if g_count > self.iteration_cap:
                raise NumericalError(
                    f"pressure solve used {g_count} global iterations in one minor step "
                    f"(max error {max_err:.4%} of rest density)")
        self._call("rts_pci_sob")
        return it, corrected, riters, early, c

    def _mark_timestep_updates(self, launch_only: bool = False) -> None:
        """Mid-major pre-emption (pcisph.py:718-755)."""
        self._prepare(self.dt)
        p = self.params
        p.n_max = min(self.n_regions, self.controller.n_current)
        self._call("rts_block_maxima", 1)
        self._call("rts_block_levels", 2)
        self._call("rts_pci_mark_updates")
        if not launch_only:
            self._raise(self.counters.read(self._stream()))

    def _audit_refresh(self) -> int:
        raise NotImplementedError("neighbour audit on the B200 path is not implemented yet")
