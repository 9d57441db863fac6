"""RTS-WCSPH on the B200 -- drop-in for ``rts_sph.wcsph.WcsphSolver``
(/root/reference/pkg/src/rts_sph/wcsph.py:108-319; Algorithm 1 of
arXiv 2009.14514 with the Serna predictor-corrector).

One ``step()`` enqueues, on the current CUDA stream:

  rts_grid_keys        block keys + domain check + per-block max |v|, |F|
  rts_grid_sort        boundary culling, scan, stable CSR scatter
  rts_block_levels     assign_regions + smooth_regions (RTS mode)
  rts_wcsph_propagate  validity countdown / pre-emption, sorted copies,
                       active-list compaction
  rts_wcsph_density    density + Tait over the 3x3x3 block neighbourhood
  rts_wcsph_forces     pressure + viscosity + gravity, corrector bookkeeping
  rts_wcsph_integrate  predictor (all), corrector (active), clamp

and synchronises once at the end to read the counters block (errors,
n_compute) for the returned StepStats.  State attributes are fp32 CUDA
tensors in the reference's particle order, writable in place
(``solver.vel[i] = ...`` works as with the numpy reference).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from ._device import (Arena, Counters, PhaseTimer, device_index, nvtx_range, raise_on_errors,
                      raw_stream, require_cuda)
from .grid import BlockGrid
from .kernels import KernelSet
from .scene import TAIT_GAMMA, Scene, seed_particles
from .stats import StepStats

__all__ = ["WcsphSolver", "tait_pressure", "NEIGHBOR_WIDTH"]

NEIGHBOR_WIDTH = 128
HIT_CAP = 64  # wcsph.cu kHitCap: per-particle list of the density pass


def tait_pressure(rho: float, rest_density: float, sound_speed: float) -> float:
    """Host form of the clamped Tait EOS (wcsph.py:38-42)."""
    b = rest_density * sound_speed * sound_speed / TAIT_GAMMA
    p = b * ((rho / rest_density) ** TAIT_GAMMA - 1.0)
    return p if p > 0.0 else 0.0


class _DeviceSolver:
    # PCISPH: no SoA candidate copies -- the integrator would have to scatter
    # three more arrays every minor step, which costs what the search saves
    _soa_candidates = False
    """Shared construction: seeding, device buffers, grid, RtsParams."""

    def _setup_common(self, scene: Scene, grid_mode: str, device):
        self.scene = scene
        self.device = require_cuda(device)
        self._dev_idx = device_index(self.device)
        self.kernel = KernelSet(scene.support_radius)
        self.mass = scene.particle_mass
        self.mu = scene.viscosity * scene.rest_density
        fluid, wall = seed_particles(scene)
        nf = self.n_fluid = len(fluid)
        self.n_bound = len(wall)
        A = self.arena = Arena(self.device)
        init = np.concatenate([fluid, wall]) if len(wall) else fluid
        self._pos = A.alloc("pos", (max(nf + self.n_bound, 1), 3), torch.float32, 0)
        self._pos[: nf + self.n_bound].copy_(torch.as_tensor(init, dtype=torch.float32))
        self.counters = Counters(A)
        self.grid = BlockGrid.for_scene(scene, grid_mode, device=self.device, arena=A)
        self.grid.counters = self.counters
        self.grid._ensure_particles(nf, nf + self.n_bound)
        self.grid.bind_boundary(self._pos[nf:nf + self.n_bound].cpu().numpy(), nf)
        self.grid.n_fluid = nf
        self.gravity = np.asarray(scene.gravity, dtype=np.float64)
        self._clamp_lo = np.asarray(scene.domain_min) + 0.1 * scene.spacing
        self._clamp_hi = np.asarray(scene.domain_max) - 0.1 * scene.spacing
        p = self.params = N.RtsParams()
        self.grid.fill_params(p)
        k = self.kernel
        p.h, p.h2, p.c_poly6, p.c_spiky, p.c_visc = k.h, k.h2, k.c_poly6, k.c_spiky, k.c_visc
        p.mass = self.mass
        p.inv_mass = 1.0 / self.mass
        p.rho0 = scene.rest_density
        p.mu = self.mu
        for a in range(3):
            p.clamp_lo[a] = float(self._clamp_lo[a])
            p.clamp_hi[a] = float(self._clamp_hi[a])
        p.n_fluid = nf
        p.n_bound = self.n_bound
        p.n_bcells = self.grid.n_bcells
        p.width = NEIGHBOR_WIDTH
        p.lambda_v = scene.lambda_v
        p.lambda_f = scene.lambda_f
        p.sound_speed = scene.sound_speed
        p.eta_max, p.eta_avg, p.rho_T = scene.eta_max, scene.eta_avg, scene.rho_T
        sms = N.load().rts_device_sms()
        p.n_sms = sms if sms > 0 else 148
        A.alloc("cpos", (nf + self.n_bound + 4, 4), torch.float32, 0)
        A.alloc("cvel", (max(nf + self.n_bound, 1), 4), torch.float32, 0)
        A.alloc("cterm", (max(nf + self.n_bound, 1), 4), torch.float64, 0)
        A.alloc("cwall", (max(nf + self.n_bound, 1),), torch.float64, 0)
        if self._soa_candidates:  # SoA candidate positions (+8: padded quads)
            for name in ("cx", "cy", "cz"):
                A.alloc(name, (nf + self.n_bound + 8,), torch.float32, 0)
        A.alloc("active", (max(nf, 1),), torch.int32, 0)
        A.alloc("list2", (max(nf, 1),), torch.int32, 0)
        A.alloc("list3", (max(nf, 1),), torch.int32, 0)
        self.step_index = 0
        self.sim_time = 0.0
        self.missed_neighbors_total = 0
        self._timers = {"neighbor": 0.0, "physics": 0.0, "rts": 0.0}
        self.timer = PhaseTimer(True)

    def _set_betas(self, n_regions: int, alpha: float):
        betas = self.scene.betas(n_regions)
        p = self.params
        for q in range(8):
            p.betas[q] = float(betas[q]) if q < len(betas) else math.nan
        p.alpha = alpha
        self.betas = betas
        self.alpha = alpha

    def _sync_params(self):
        p = self.params
        g = np.asarray(self.gravity, dtype=np.float64).reshape(3)
        for a in range(3):
            p.gravity[a] = float(g[a])

    # -- kernel launch with optional CUDA-event timing (bench roofline) -----
    _ktimes: dict | None = None

    def time_kernels(self, names) -> None:
        """Record CUDA events around every launch of the named entry points
        (used by bench.py for the live roofline of the dominant kernel)."""
        self._ktimes = {n: [] for n in names}

    def kernel_times(self, name: str) -> list[float]:
        """Durations (s) of the recorded launches of ``name`` (syncs)."""
        return [a.elapsed_time(b) * 1e-3 for a, b in (self._ktimes or {}).get(name, [])]

    def _launch(self, name: str, *args) -> None:
        kt = self._ktimes
        if kt is not None and name in kt:
            stream = torch.cuda.current_stream(self.device)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            N.call(name, self.params, self.arena.buf, *args, stream.cuda_stream)
            b.record(stream)
            kt[name].append((a, b))
        else:
            N.call(name, self.params, self.arena.buf, *args, raw_stream(self._dev_idx))

    @property
    def pos(self) -> torch.Tensor:
        return self._pos[: self.n_fluid + self.n_bound]

    # -- local particle sets (distributed ranks, distributed.py) ---------------
    # (attribute, arena buffer, width, dtype, initial value; None = rest density)
    _FIELDS: tuple = ()

    def _fresh_state(self, pos: torch.Tensor) -> dict:
        n = pos.shape[0]
        out = {"pos": pos.to(torch.float32)}
        for name, _, w, dt, fill in self._FIELDS:
            fill = self.scene.rest_density if fill is None else fill
            shape = (n, w) if w > 1 else (n,)
            out[name] = torch.full(shape, fill, dtype=dt, device=self.device)
        return out

    def _cast_state(self, state: dict) -> dict:
        out = {"pos": state["pos"].to(torch.float32).reshape(-1, 3)}
        for name, _, w, dt, _f in self._FIELDS:
            v = state[name]
            if dt == torch.bool:
                v = v != 0
            out[name] = v.to(dt).reshape((-1, w) if w > 1 else (-1,))
        return out

    def _get_local_state(self) -> dict:
        nf = self.n_fluid
        out = {"pos": self._pos[:nf]}
        for name, *_ in self._FIELDS:
            out[name] = getattr(self, name)
        return out

    def _set_local_particles(self, state, walls, capacity=None, init=False) -> None:
        """Replace the fluid rows (and optionally the static wall set) of this
        solver: the distributed driver loads owned + ghost particles every
        step.  Buffers grow geometrically; wall rows follow the fluid rows."""
        A = self.arena
        if walls is not None:
            self._walls = torch.as_tensor(np.asarray(walls, dtype=np.float32),
                                          device=self.device).reshape(-1, 3)
        nb = self._walls.shape[0]
        nf = 0 if state is None else int(state["pos"].shape[0])
        cap = getattr(self, "_cap", -1)
        if init or nf > cap or nf + nb > self._pos.shape[0] or (capacity or 0) > cap:
            cap = max(nf, int(1.25 * nf) + 1024, capacity or 0)
            self._cap = cap
            self._pos = A.alloc("pos", (cap + nb, 3), torch.float32, 0)
            for _, arena, w, dt, fill in self._FIELDS:
                fill = self.scene.rest_density if fill is None else fill
                A.alloc(arena, (cap, w) if w > 1 else (cap,), dt, fill)
            for name in ("cpos", "cvel"):
                A.alloc(name, (cap + nb + 4, 4), torch.float32, 0)  # +4: padded candidate reads
            A.alloc("cterm", (cap + nb + 4, 4), torch.float64, 0)
            A.alloc("cwall", (cap + nb + 4,), torch.float64, 0)
            if self._soa_candidates:
                for name in ("cx", "cy", "cz"):
                    A.alloc(name, (cap + nb + 8,), torch.float32, 0)
            for name in ("active", "list2", "list3"):
                A.alloc(name, (cap,), torch.int32, 0)
            self._realloc_extra(cap, nb)
            self.grid._ensure_particles(cap, cap + nb)
            if walls is not None or init:
                self.grid.bind_boundary(self._walls.double().cpu().numpy(), nf)
        if walls is not None and not init:
            self.grid.bind_boundary(self._walls.double().cpu().numpy(), nf)
        if nf:
            self._pos[:nf].copy_(state["pos"])
            for name, arena, w, dt, _ in self._FIELDS:
                A[arena][:nf].copy_(state[name].reshape(A[arena][:nf].shape))
        self._pos[nf:nf + nb].copy_(self._walls)
        self.n_fluid = nf
        self.n_bound = nb
        for name, arena, *_ in self._FIELDS:
            setattr(self, name, A[arena][:nf])
        self.grid.n_fluid = nf
        self.grid.shift_boundary(nf)
        p = self.params
        p.n_fluid = nf
        p.n_bound = nb
        p.n_bcells = self.grid.n_bcells

    def _resize_fluid(self, nf: int, n_ghost: int = 0) -> None:
        """Resident x-slab ranks (distributed.py): n_fluid = nf with the rows
        [0, nf) left where they are (no copy); the wall rows move behind
        them.  The caller fills any new rows."""
        if nf > self._cap:
            raise ValueError(f"{nf} fluid rows exceed the capacity {self._cap}")
        nb = self.n_bound
        self._pos[nf:nf + nb].copy_(self._walls)
        A = self.arena
        self.n_fluid = nf
        for name, arena, *_ in self._FIELDS:
            setattr(self, name, A[arena][:nf])
        self.grid.n_fluid = nf
        self.grid.shift_boundary(nf)
        self.params.n_fluid = nf

    def _realloc_extra(self, cap: int, nb: int) -> None:
        """Solver-specific buffers sized by the particle capacity."""

    def host(self, name: str) -> np.ndarray:
        """fp64 numpy snapshot of a state attribute (for parity checks)."""
        t = getattr(self, name)
        t = t.detach().cpu()
        return t.numpy().astype(np.float64) if t.is_floating_point() else t.numpy()


class WcsphSolver(_DeviceSolver):
    """Weakly compressible SPH, ``mode`` "baseline" or "rts" (wcsph.py:108)."""

    # the density pass's search reads x / y / z candidate copies (written by
    # the propagate pass in slot order: free); -8 % on the search
    _soa_candidates = True

    mode_names = ("baseline", "rts")

    def __new__(cls, scene=None, *args, comm=None, **kw):
        """``comm`` (the default torch.distributed group): this process is one
        x-slab rank of a multi-GPU run -- a ``DistributedWcsph`` with the same
        solver keywords (SURVEY.md 8b "extra kwargs: device, comm")."""
        if comm is not None:
            from .distributed import rank_solver
            return rank_solver("wcsph", scene, comm, *args, **kw)
        return super().__new__(cls)

    def _realloc_extra(self, cap: int, nb: int) -> None:
        # the density pass's neighbour lists (slots), reused by the force pass
        stride = -(-max(cap, 1) // 32) * 32
        self.arena.alloc("nbr", (HIT_CAP, stride), torch.int32, 0)
        self.arena.alloc("cnt", (max(cap, 1),), torch.int32, 0)
        self.params.nbr_stride = stride
    _FIELDS = (("vel", "vel", 3, torch.float32, 0.0), ("acc", "acc", 3, torch.float32, 0.0),
               ("acc_prev", "acc_prev", 3, torch.float32, 0.0),
               ("force", "force", 3, torch.float32, 0.0), ("rho", "rho", 1, torch.float32, None),
               ("pres", "pres", 1, torch.float32, 0.0),
               ("dt_since", "dt_since", 1, torch.float64, 0.0),
               ("dt_corr", "dt_corr", 1, torch.float64, 0.0),
               ("validity", "validity", 1, torch.int32, 0), ("region", "region", 1, torch.int8, 1),
               ("compute", "compute", 1, torch.bool, True))

    def __init__(self, scene: Scene, mode: str = "rts", dt_cap: float | None = None,
                 pin_region: int | None = None, apply_correction: bool = True,
                 track_rho_variance: bool = False, audit_neighbors: bool = False,
                 n_regions: int = 4, device="cuda", use_graphs: bool = True, comm=None):
        if mode not in self.mode_names:
            raise ValueError(f"unknown wcsph mode {mode!r}")
        self.mode = mode
        self.pin_region = pin_region
        self.apply_correction = apply_correction
        self.track_rho_variance = track_rho_variance
        self.audit_neighbors = audit_neighbors
        self.n_regions = n_regions
        self._setup_common(scene, "wcsph", device)
        self._var_out = torch.zeros(1, dtype=torch.float64, device=self.device)
        if "partial" not in self.arena.t:
            self.arena.alloc("partial", (4096,), torch.float64, 0)
        self.dt_base = scene.base_dt("wcsph")
        self.dt_cap = self.dt_base if dt_cap is None else dt_cap
        self.b_stiff = scene.rest_density * scene.sound_speed**2 / TAIT_GAMMA
        self._set_betas(n_regions, scene.alpha_for("wcsph"))
        p = self.params
        p.b_stiff = self.b_stiff
        p.dt_base = self.dt_base
        p.n_max = n_regions
        p.use_sound = 1
        p.rts = 1 if mode == "rts" else 0
        nf = self.n_fluid
        A = self.arena
        f32 = torch.float32
        self.vel = A.alloc("vel", (max(nf, 1), 3), f32, 0)[:nf]
        self.acc = A.alloc("acc", (max(nf, 1), 3), f32, 0)[:nf]
        self.acc_prev = A.alloc("acc_prev", (max(nf, 1), 3), f32, 0)[:nf]
        self.force = A.alloc("force", (max(nf, 1), 3), f32, 0)[:nf]
        self.rho = A.alloc("rho", (max(nf, 1),), f32, scene.rest_density)[:nf]
        self.pres = A.alloc("pres", (max(nf, 1),), f32, 0)[:nf]
        self.dt_since = A.alloc("dt_since", (max(nf, 1),), torch.float64, 0)[:nf]
        self.dt_corr = A.alloc("dt_corr", (max(nf, 1),), torch.float64, 0)[:nf]
        self.validity = A.alloc("validity", (max(nf, 1),), torch.int32, 0)[:nf]
        self.region = A.alloc("region", (max(nf, 1),), torch.int8, 1)[:nf]
        self.compute = A.alloc("compute", (max(nf, 1),), torch.bool, True)[:nf]
        self._realloc_extra(max(nf, 1), self.n_bound)
        self._missed_last = 0
        self.use_graphs = use_graphs
        self._graphs: dict = {}

    def __del__(self):
        for g in getattr(self, "_graphs", {}).values():
            try:
                N.load().rts_graph_destroy(g)
            except Exception:  # pragma: no cover
                pass

    def _graph(self):
        import ctypes
        key = bytes(self.params) + bytes(self.arena.buf)  # values and buffer addresses
        g = self._graphs.get(key)
        if g is None:
            if len(self._graphs) >= 8:
                for old in self._graphs.values():
                    N.load().rts_graph_destroy(old)
                self._graphs.clear()
            err = ctypes.c_int(0)
            g = N.load().rts_wcsph_graph_create(self.params, self.arena.buf, ctypes.byref(err))
            if not g:
                raise N.NativeError(f"rts_wcsph_graph_create failed with cudaError {err.value}")
            self._graphs[key] = g
        return g

    # ------------------------------------------------------------------
    def cfl_bound(self) -> float:
        """Global step bound from max |F| (wcsph.py:182-189)."""
        sc = self.scene
        r = self.grid.block_size
        eq1 = sc.lambda_v * r / sc.sound_speed
        f_max = self._force_max()
        eq2 = sc.lambda_f * math.sqrt(r * self.mass / f_max) if f_max > 0.0 else math.inf
        return min(eq1, eq2)

    _reduce_max = None  # x-slab ranks: all-reduce MAX across ranks (distributed.py)

    def _force_max(self) -> float:
        if not self.n_fluid:
            return self._reduce_max(0.0) if self._reduce_max is not None else 0.0
        stream = torch.cuda.current_stream(self.device)
        self.counters.reset(stream)
        N.call("rts_force_max", self.params, self.arena.buf, stream.cuda_stream)
        c = self.counters.read(stream)
        f = float(np.array([c.fmax_bits], dtype=np.uint64).view(np.float64)[0])
        return self._reduce_max(f) if self._reduce_max is not None else f

    def particle_regions(self) -> torch.Tensor:
        if self.mode == "rts":
            return self.region
        return torch.ones(self.n_fluid, dtype=torch.int8, device=self.device)

    def advance(self) -> list[StepStats]:
        return [self.step()]

    @nvtx_range("rts_wcsph.step")
    def step(self) -> StepStats:
        if self.mode == "rts":
            dt = self.dt_base
        else:
            dt = min(self.cfl_bound(), self.dt_cap)
        c = self._enqueue_step(dt)
        raise_on_errors(c, NEIGHBOR_WIDTH)
        n_compute = int(c.n_compute)
        self.step_index += 1
        self.sim_time += dt
        if self._graph_step:  # device %globaltimer stamps inside the step graph
            t0, t1, t2, t3 = (int(x) for x in c.stamps)
            self._timers = {"neighbor": max(0, t1 - t0) * 1e-9, "rts": max(0, t2 - t1) * 1e-9,
                            "physics": max(0, t3 - t2) * 1e-9}
        else:
            self._timers = self.timer.totals()
        st = StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=n_compute,
                       frac_compute=n_compute / max(1, self.n_fluid),
                       missed_neighbors=self._missed_last,
                       t_neighbor=self._timers["neighbor"], t_physics=self._timers["physics"],
                       t_rts=self._timers["rts"])
        if self.track_rho_variance:  # np.var(rho), wcsph.py:231-232 (device reduction)
            out = self._var_out
            N.call("rts_rho_variance", self.params, self.arena.buf, out.data_ptr(),
                   torch.cuda.current_stream(self.device).cuda_stream)
            st.rho_var = float(out.item())
        return st

    def _enqueue_step(self, dt: float, read: bool = True):
        """Enqueue one step (no host sync unless ``read``)."""
        self._sync_params()
        p = self.params
        p.dt = dt
        p.pin_region = int(self.pin_region or 0)
        p.apply_correction = int(bool(self.apply_correction))
        stream = torch.cuda.current_stream(self.device)
        tm = self.timer
        rts = self.mode == "rts"
        self._graph_step = self.use_graphs and rts and self._ktimes is None
        if self._graph_step:  # baseline dt varies per step
            tm.start(stream)
            graph = self._graph()
            N.call("rts_graph_launch", graph, stream.cuda_stream)
            N.note_graph_kernels(N.graph_kernel_counts(graph)[0])
            tm.mark("physics", stream)
            if not read:
                return None
            c = self.counters.read(stream)
            self.grid.n_sorted = int(c.n_sorted)
            return c
        self.counters.reset(stream)
        tm.start(stream)
        self.grid.launch_rebuild(p, stream, want_maxima=rts)
        tm.mark("neighbor", stream)
        if rts:
            self._launch("rts_block_levels", 0)
        self._launch("rts_wcsph_propagate")
        tm.mark("rts", stream)
        self._launch("rts_wcsph_density")
        self._launch("rts_wcsph_forces")
        self._launch("rts_wcsph_integrate")
        tm.mark("physics", stream)
        if not read:
            return None
        c = self.counters.read(stream)
        self.grid.n_sorted = int(c.n_sorted)
        return c
