"""RTS-PCISPH on the B200 -- drop-in for ``rts_sph.pcisph.PcisphSolver``
(/root/reference/pkg/src/rts_sph/pcisph.py:279-768; Algorithms 2-3 of
arXiv 2009.14514) and its constant / globally adaptive baselines.

Control flow (major step -> minor steps -> scheduled correction loop with
S_e / S_ob sets, local phases with snapshot/revert, early termination and
the iteration cap) is the reference's; every particle and block pass is a
librtssph kernel (see csrc/pcisph.cu) and every convergence decision is
taken on the device by ``k_control``.  With ``use_graphs`` (default) a
whole major step -- rebuild, levels, every minor step with its correction
loop as a CUDA-graph conditional while node -- is one graph launch and one
read-back of the control block; ``use_graphs=False`` launches the same
kernels one by one (per-kernel timing, the neighbour audit, x-slab ranks).
"""

from __future__ import annotations

import collections
import ctypes
import dataclasses
import itertools
import math
import os

import numpy as np
import torch

from . import _native as N
from ._device import nvtx_range, raise_on_errors
from .errors import ConfigError, NumericalError
from .scene import Scene
from .stats import StepStats
from .grid import BlockGrid
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


def _violations(tally, n_regions: int):
    """The schedule rules of pcisph.py:80-117, as messages, in the order the
    reference checks them: every region on every minor step; every region
    twice on the first; region 1 three times on each; region n (window 2 for
    region 2) at least 3 times in every cyclic window of its own step."""
    n_minor = len(tally)
    regions = range(1, n_regions + 1)
    yield from (f"region {n} receives no iteration on minor step {j + 1}"
                for j in range(n_minor) for n in regions if tally[j][n] < 1)
    yield from (f"region {n} receives fewer than 2 iterations on the first minor step"
                for n in regions if tally[0][n] < 2)
    yield from (f"region 1 receives fewer than 3 iterations on minor step {j + 1}"
                for j in range(n_minor) if tally[j][1] < 3)
    for n in regions:
        w = 2 if n == 2 else min(n, n_minor)
        for j in range(n_minor):
            got = sum(tally[(j + q) % n_minor][n] for q in range(w))
            if got < 3:
                yield (f"region {n} receives {got} < 3 iterations in the {w}-minor window "
                       f"starting at minor step {j + 1}")


def validate_schedule(schedule, n_regions: int = 4) -> None:
    """ConfigError unless ``schedule`` meets the reference's legality rules."""
    tally = [collections.Counter() for _ in schedule]
    for j, rows in enumerate(schedule):
        for n in itertools.chain.from_iterable(rows):
            if not 1 <= n <= n_regions:
                raise ConfigError(f"schedule names region {n} outside 1..{n_regions}")
            tally[j][n] += 1
    first = next(_violations(tally, n_regions), None)
    if first is not None:
        raise ConfigError(first)


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
        if early_terminated:  # N = 2 for the next ten majors
            self.n_current, self.recovery_left = 2, 10
            return
        if self.recovery_left:
            self.recovery_left -= 1
            if not self.recovery_left:
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
    # x / y / z candidate copies written by the major-start gather only: the
    # full refresh of the first minor step searches them (packed fp32x2);
    # the integrator keeps only cpos current and the later partial refreshes
    # read that (RtsCounters.soa_fresh)
    _soa_candidates = os.environ.get("RTS_PCI_SOA", "1") != "0"

    def __new__(cls, scene=None, *args, comm=None, **kw):
        """``comm`` (the default torch.distributed group): this process is one
        x-slab rank -- a ``DistributedPcisph`` (RTS mode) with the same solver
        keywords (SURVEY.md 8b "extra kwargs: device, comm")."""
        if comm is not None:
            from .distributed import rank_solver
            return rank_solver("pcisph", scene, comm, *args, **kw)
        return super().__new__(cls)
    _FIELDS = (("vel", "vel", 3, torch.float32, 0.0), ("f_ext", "force", 3, torch.float32, 0.0),
               ("f_p", "f_p", 3, torch.float32, 0.0), ("p", "pres", 1, torch.float32, 0.0),
               ("rho_star", "rho", 1, torch.float32, None), ("err", "err", 1, torch.float64, 0.0),
               ("xstar", "xstar", 3, torch.float32, 0.0),
               ("region", "region", 1, torch.int8, 1), ("validity", "validity", 1, torch.int32, 0),
               ("compute", "compute", 1, torch.bool, True), ("in_se", "in_se", 1, torch.bool, False),
               ("in_sob", "in_sob", 1, torch.bool, False))
    _xch = None  # ghost-exchange hooks of a distributed rank (distributed.py)

    def _realloc_extra(self, cap: int, nb: int) -> None:
        A = self.arena
        stride = -(-max(cap, 1) // 32) * 32
        self._nbr = A.alloc("nbr", (NEIGHBOR_WIDTH, stride), torch.int32, 0)
        self.params.nbr_stride = stride
        self._cnt_full = A.alloc("cnt", (cap,), torch.int32, 0)
        A.alloc("xs", (cap + nb, 4), torch.float64, 0)  # 32-byte rows: fp64 x*, p
        A.alloc("pflag", (cap,), torch.uint8, 0)
        A.alloc("snap_p", (cap,), torch.float64, 0)
        A.alloc("snap_fp", (cap, 3), torch.float32, 0)
        A.alloc("slot_of", (cap,), torch.int32, 0)
        A.alloc("ghost", (cap,), torch.uint8, 0)

    def _set_local_particles(self, state, walls, capacity=None, init=False, ghost=None):
        super()._set_local_particles(state, walls, capacity, init)
        nf = self.n_fluid
        self.cnt = self.arena["cnt"][:nf]
        g = self.arena["ghost"]
        g.zero_()
        self.params.n_ghost = 0
        if ghost is not None and nf:
            g[:nf].copy_(ghost.to(torch.uint8))
            self.params.n_ghost = int(ghost.sum())
        self.params.n_fluid = nf
        N.call("rts_pci_walls", self.params, self.arena.buf, self._stream().cuda_stream)

    def _resize_fluid(self, nf: int, n_ghost: int = 0) -> None:
        super()._resize_fluid(nf)
        self.cnt = self.arena["cnt"][:nf]
        g = self.arena["ghost"]
        g.zero_()
        if n_ghost:
            g[nf - n_ghost:nf] = 1
        self.params.n_ghost = n_ghost
        N.call("rts_pci_walls", self.params, self.arena.buf, self._stream().cuda_stream)

    def __init__(self, scene: Scene, mode: str = "rts", dt: float | None = None,
                 schedule=DEFAULT_SCHEDULE, pin_region: int | None = None,
                 audit_neighbors: bool = False, iteration_cap: int = 24,
                 local_attempts: int = 4, n_regions: int = 4, device="cuda",
                 use_graphs: bool = True, comm=None):
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
        stride = -(-n1 // 32) * 32  # column-major table: entry q of particle i at [q, i]
        self._nbr = A.alloc("nbr", (NEIGHBOR_WIDTH, stride), torch.int32, 0)
        self.params.nbr_stride = stride
        self.cnt = A.alloc("cnt", (n1,), torch.int32, 0)[:nf]
        A.alloc("xs", (max(nf + self.n_bound, 1), 4), torch.float64, 0)  # fp64 x*, p
        A.alloc("pflag", (n1,), torch.uint8, 0)
        A.alloc("partial", (4096,), torch.float64, 0)
        A.alloc("snap_p", (n1,), torch.float64, 0)
        A.alloc("snap_fp", (n1, 3), f32, 0)
        A.alloc("slot_of", (n1,), torch.int32, 0)
        A.alloc("se_stamp", (self.grid.n_cells,), torch.int32, 0)
        A.alloc("near_stamp", (self.grid.n_cells,), torch.int32, 0)
        self._ctl = A.alloc("ctl", (ctypes.sizeof(N.RtsControl),), torch.uint8, 0)
        self._ctl_host = torch.zeros(ctypes.sizeof(N.RtsControl), dtype=torch.uint8).pin_memory()
        self.use_graphs = use_graphs
        self._graphs: dict = {}
        self._force_total = 0
        p = self.params
        p.dt_base = self.dt
        p.n_regions = n_regions
        p.use_sound = 0
        p.rts = 1 if mode == "rts" else 0
        stream = torch.cuda.current_stream(self.device)
        N.call("rts_pci_walls", p, A.buf, stream.cuda_stream)
        self._upload_schedule()

    def __del__(self):
        for g in getattr(self, "_graphs", {}).values():
            try:
                N.load().rts_graph_destroy(g)
            except Exception:  # pragma: no cover
                pass

    # -- device loop control ----------------------------------------------------
    def _upload_schedule(self) -> None:
        """Write the schedule's row masks / region multiplicities into the
        control block (its loop state and running totals restart at zero)."""
        c = N.RtsControl()
        if len(self.schedule) > N.MAX_MINOR:
            raise ConfigError(f"at most {N.MAX_MINOR} minor steps are supported")
        for j, rows in enumerate(self.schedule):
            if len(rows) > N.MAX_ROWS:
                raise ConfigError(f"at most {N.MAX_ROWS} iterations per minor step are supported")
            c.n_rows[j] = len(rows)
            for r, row in enumerate(rows):
                c.row_masks[j][r] = _row_mask(row)
                packed = 0
                for n in row:
                    if 1 <= n <= min(self.n_regions, 7):
                        packed += 1 << (4 * n)
                c.row_counts[j][r] = packed
        host = torch.frombuffer(bytearray(bytes(c)), dtype=torch.uint8)
        self._ctl.copy_(host)

    def _read_control(self):
        st = self._stream()
        self._ctl_host.copy_(self._ctl, non_blocking=True)
        c = self.counters.read(st)
        ctl = N.RtsControl.from_buffer_copy(self._ctl_host.numpy().tobytes())
        self._ctl_cache = ctl
        self.grid.n_sorted = int(c.n_sorted)
        return ctl, c

    @property
    def local_entered_total(self) -> int:
        ctl = getattr(self, "_ctl_cache", None)
        return int(ctl.local_entered) if ctl is not None else 0

    @property
    def local_reverted_total(self) -> int:
        ctl = getattr(self, "_ctl_cache", None)
        return int(ctl.local_reverted) if ctl is not None else 0

    def _graph(self, mode: int, n_minor: int):
        key = (mode, n_minor, bytes(self.params), bytes(self.arena.buf), self.local_attempts,
               self.iteration_cap)
        g = self._graphs.get(key)
        if g is None:
            if len(self._graphs) >= 8:
                for old in self._graphs.values():
                    N.load().rts_graph_destroy(old)
                self._graphs.clear()
            err = ctypes.c_int(0)
            g = N.load().rts_pci_graph_create(self.params, self.arena.buf, mode, n_minor,
                                              self.local_attempts, self.iteration_cap,
                                              ctypes.byref(err))
            if not g:
                raise N.NativeError(f"rts_pci_graph_create failed with cudaError {err.value}")
            self._graphs[key] = g
        return g

    def _run_loop_host(self, sync_mode: int) -> None:
        """Correction loop without a graph: enqueue iterations, read `done`.
        With ghost exchanges (x-slab ranks) the first three iterations -- the
        minimum of every minor step (pcisph.py:681) -- are enqueued before the
        first read of `done`, so the exchanges of consecutive iterations are
        queued without a host round trip (iterations after `done` are no-ops
        in every kernel)."""
        x = self._xch
        ahead = 3 if x is not None else 1
        while True:
            if self._ktimes is None and x is None:
                self._call("rts_pci_iteration", sync_mode, 0, self.local_attempts,
                           self.iteration_cap)
            else:  # per-entry-point launches: kernel timing / ghost exchanges
                self._call("rts_pci_motion", -1)
                if x is not None:
                    x.after_motion(self)
                self._call("rts_pci_sets", -1, sync_mode)
                self._call("rts_pci_density")
                if x is not None:
                    x.after_density(self)
                self._call("rts_pci_se_reduce", int(not sync_mode))
                if x is not None:
                    x.reduce(self)
                self._call("rts_pci_pforces")
                self._call("rts_pci_control", sync_mode, 0, self.local_attempts,
                           self.iteration_cap)
            ahead -= 1
            if ahead > 0:
                continue
            ahead = 1
            self._ctl_host[24:28].copy_(self._ctl[24:28], non_blocking=True)  # ctl.done
            self._stream().synchronize()
            if int(self._ctl_host[24:28].view(torch.int32)[0]):
                return

    def _raise_control(self, ctl, c) -> None:
        raise_on_errors(c, NEIGHBOR_WIDTH) if c.err_flags & (N.ERR_ESCAPED | N.ERR_OVERFLOW) else None
        if not ctl.failed:
            return
        if ctl.fail_kind == 1 or c.err_flags & N.ERR_NONFINITE:
            raise NumericalError("non-finite predicted density; the simulation has blown up")
        if ctl.fail_kind == 2:
            raise NumericalError(
                f"pressure solve used {int(ctl.fail_g)} global iterations in one minor step "
                f"(max error {float(ctl.fail_err):.4%} of rest density)")
        if ctl.fail_kind == 3:
            raise NumericalError(
                f"pressure solve did not converge within {int(ctl.fail_g)} iterations "
                f"(max error {float(ctl.fail_err):.4%} of rest density)")
        raise_on_errors(c, NEIGHBOR_WIDTH)

    # -- reference-facing helpers -------------------------------------------
    @property
    def block_region(self) -> torch.Tensor:
        return self.arena["block_field"]

    @property
    def xstar(self) -> torch.Tensor:
        """Predicted positions of the last prediction (pcisph.py:202-213): the
        fp32 view of the fp64 x* the kernels keep in the xs rows, refreshed
        on access after a step (the integrator no longer copies it out)."""
        t = self._xstar_t
        if getattr(self, "_xstar_dirty", False) and self.n_fluid:
            t.copy_(self.arena["xs"][: self.n_fluid, :3])
        self._xstar_dirty = False
        return t

    @xstar.setter
    def xstar(self, t: torch.Tensor) -> None:
        self._xstar_t = t
        self._xstar_dirty = False

    @property
    def vstar(self) -> torch.Tensor:
        """Predicted velocities of the last prediction (pcisph.py:202-213),
        recovered as (x* - pos) / dt from the stored fp32 x* (the kernels keep
        x* only)."""
        nf = self.n_fluid
        return (self.xstar.double() - self.pos[:nf].double()).div_(self.dt).float()

    @property
    def nbr(self) -> torch.Tensor:
        """(n_fluid, 128) view of the column-major device table (rows as in
        the reference, grid.py:146-149)."""
        return self._nbr[:, : self.n_fluid].T

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
        self._xstar_dirty = True  # any pass may have rewritten the xs rows

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
    @nvtx_range("rts_pcisph.sync_step")
    def sync_step(self) -> StepStats:
        """Synchronous baseline step (pcisph.py:376-419): rebuild, full
        search + external forces, the standard correction loop (device
        control, >= 3 iterations until max err < eta_max and avg < eta_avg),
        integrate."""
        nf = self.n_fluid
        dt = self.dt
        self._prepare(dt)
        st = self._stream()
        graph = None
        if self.use_graphs:
            graph = self._graph(1, 1)
            N.call("rts_graph_launch", graph, st.cuda_stream)
        else:
            N.call("rts_counters_reset", self.arena.buf, st.cuda_stream)
            self._call("rts_pci_major_begin")
            self.grid.launch_rebuild(self.params, st, want_maxima=False, add_fp=True)
            self._call("rts_pci_gather")
            self._call("rts_pci_minor_begin", 0, 1)
            self._call("rts_pci_refresh", 1, 0)
            self._call("rts_pci_zero_pressure")
            self._run_loop_host(1)
            self._call("rts_pci_integrate", 0)
            self._call("rts_pci_minor_end", 0)
        ctl, c = self._read_control()
        self._xstar_dirty = True
        if graph is not None:
            n_static, n_body = N.graph_kernel_counts(graph)
            N.note_graph_kernels(n_static + n_body * max(0, ctl.stats[0].iterations))
        self._raise_control(ctl, c)
        ms = ctl.stats[0]
        it = int(ms.iterations)
        self._force_total += int(ms.forced)
        if self.mode == "adaptive":
            self._adapt_dt(it)
        self.step_index += 1
        self.sim_time += dt
        t_nb = max(0, ms.t_refreshed - ms.t_begin) * 1e-9
        t_ph = max(0, ms.t_end - ms.t_refreshed) * 1e-9
        return StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=nf,
                         frac_compute=1.0, iterations=it, corrected=int(ms.corrected),
                         iters_r1=it, iters_r2=it, iters_r3=it, iters_r4=it,
                         max_err=float(ms.max_err), avg_err=float(ms.avg_err),
                         t_neighbor=t_nb, t_physics=t_ph, t_rts=0.0)

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
    @nvtx_range("rts_pcisph.major_step")
    def major_step(self) -> list[StepStats]:
        """One major step of N minor steps (pcisph.py:482-505).  With
        ``use_graphs`` (default) the whole major -- rebuild, region
        assignment, every minor step with its device-controlled correction
        loop -- is one CUDA-graph launch followed by a single read-back."""
        n_minor = self.controller.n_current
        self._prepare(self.dt)
        self.params.n_max = min(self.n_regions, n_minor)
        st = self._stream()
        audit = bool(self.audit_neighbors)
        missed = []
        graph = None
        if self.use_graphs and self._xch is None and not audit:
            graph = self._graph(0, n_minor)
            N.call("rts_graph_launch", graph, st.cuda_stream)
        else:
            N.call("rts_counters_reset", self.arena.buf, st.cuda_stream)
            self._call("rts_pci_major_begin")
            self.grid.launch_rebuild(self.params, st, want_maxima=True, add_fp=True)
            self._call("rts_pci_gather")
            self._call("rts_block_levels", 1)
            self._call("rts_pci_major_particles")
            x = self._xch
            for j in range(n_minor):
                if self._ktimes is None and x is None and not audit:
                    self._call("rts_pci_minor_head", j)
                else:
                    self._call("rts_pci_minor_begin", j, 0)
                    self._call("rts_pci_refresh", 0, 1)
                    if audit:
                        self._audit_refresh()
                        missed.append(self.counters.read(st).missing)
                    self._call("rts_pci_zero_pressure")
                    N.call("rts_memset", self.arena.buf.in_se, 0, self.n_fluid, st.cuda_stream)
                    self._call("rts_pci_observed", 0)
                self._run_loop_host(0)
                if self._ktimes is None and x is None:
                    self._call("rts_pci_minor_tail", j, int(j == n_minor - 1))
                else:
                    self._call("rts_pci_integrate", 1)
                    if x is not None:
                        x.after_integrate(self)
                    if j != n_minor - 1:
                        self._call("rts_block_maxima", 1)
                        self._call("rts_pci_mark_updates")  # required levels included
                    self._call("rts_pci_minor_end", j)
        ctl, c = self._read_control()
        self._xstar_dirty = True
        if graph is not None:  # launch accounting of the graph's kernel nodes
            n_static, n_body = N.graph_kernel_counts(graph)
            its = sum(max(0, ctl.stats[j].iterations) for j in range(n_minor))
            N.note_graph_kernels(n_static + n_body * its)
        rows = []
        early = False
        nf = self.n_fluid
        for j in range(n_minor):
            ms = ctl.stats[j]
            if ms.iterations < 0:
                break
            if ctl.failed and j == int(ctl.minor):
                break
            self.step_index += 1
            self.sim_time += self.dt
            early = early or bool(ms.early)
            self._force_total += int(ms.forced)
            rows.append(StepStats(
                step=self.step_index, time=self.sim_time, dt=self.dt,
                n_compute=int(ms.n_refresh), frac_compute=int(ms.n_refresh) / max(1, nf),
                iterations=int(ms.iterations), corrected=int(ms.corrected),
                iters_r1=int(ms.riters[1]), iters_r2=int(ms.riters[2]),
                iters_r3=int(ms.riters[3]), iters_r4=int(ms.riters[4]),
                max_err=float(ms.max_err), avg_err=float(ms.avg_err), early_term=int(ms.early),
                missed_neighbors=(int(missed[j]) - (int(missed[j - 1]) if j else 0))
                if j < len(missed) else 0,
                t_neighbor=max(0, ms.t_refreshed - ms.t_begin) * 1e-9,
                t_physics=max(0, ms.t_looped - ms.t_refreshed) * 1e-9,
                t_rts=max(0, ms.t_end - ms.t_looped) * 1e-9))
        self.missed_neighbors_total += sum(r.missed_neighbors for r in rows)
        self._raise_control(ctl, c)
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

    def _mark_timestep_updates(self, launch_only: bool = False) -> None:
        """Mid-major pre-emption (pcisph.py:718-755)."""
        self._prepare(self.dt)
        p = self.params
        p.n_max = min(self.n_regions, self.controller.n_current)
        self._call("rts_block_maxima", 1)
        self._call("rts_pci_mark_updates")  # required levels (block_raw) included
        if not launch_only:
            self._raise(self.counters.read(self._stream()))

    def _audit_refresh(self) -> None:
        """count_missing_neighbors (grid.py:353-394) for this minor's refresh
        list: a grid freshly rebuilt at the current positions (block edge
        max(h, block), all wall samples near fluid) is scanned one layer
        around each refreshed particle; true neighbours absent from its new
        table row accumulate in ctr.missing."""
        from ._device import Arena, Counters
        st = self._stream()
        ag = getattr(self, "_audit_grid", None)
        if ag is None:
            g = self.grid
            hi = g.origin + np.asarray(g.dims) * g.block_size
            ag = BlockGrid(g.origin, hi, max(self.kernel.h, g.block_size), device=self.device,
                           arena=Arena(self.device))
            ag.counters = Counters(ag.arena)
            self._audit_grid = ag
        A = ag.arena
        nf, nb = self.n_fluid, self.n_bound
        if getattr(self, "_audit_n", None) != (nf, nb):
            ag._ensure_particles(nf, nf + nb)
            ag.bind_boundary(self.pos[nf:nf + nb].double().cpu().numpy(), nf)
            A.alloc("cpos", (nf + nb + 4, 4), torch.float32, 0)
            A.alloc("slot_of", (max(nf, 1),), torch.int32, 0)
            self._audit_n = (nf, nb)
        A.bind("pos", self._pos)
        pa = ag.params
        pa.n_fluid, pa.n_bound, pa.n_bcells = nf, nb, ag.n_bcells
        pa.h2 = self.kernel.h2
        pa.width = NEIGHBOR_WIDTH
        pa.nbr_stride = self.params.nbr_stride
        ag.counters.reset(st)
        ag.launch_rebuild(pa, st)
        N.call("rts_pci_gather", pa, A.buf, st.cuda_stream)
        N.call("rts_pci_audit", pa, A.buf, self.arena.buf, st.cuda_stream)
