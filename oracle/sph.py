"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the RTS-SPH hot path.

A float64 restatement of the reference package ``rts_sph`` (arXiv
2009.14514; ``/root/reference/pkg/src/rts_sph``): the block grid, the region
fields, RTS-WCSPH (Algorithm 1) and RTS-PCISPH (Algorithms 2-3) with their
global-stepping baselines.  The particle loops are plain C
(``oracle_kernels.c``, built by ``oracle/Makefile``); bookkeeping is numpy,
written so every array expression evaluates the same float operations in the
same order as the reference, which makes oracle trajectories bit-identical to
the reference's (pinned by ``tests/test_oracle_golden.py`` against fixtures
generated from the reference itself, ``tests/golden/make_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline
leg and ``--impl reference`` arm) may import this module.  The product
package never does.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_2009_14514_b200.errors import ConfigError, NumericalError
from paper_2009_14514_b200.scene import TAIT_GAMMA, Scene, seed_particles
from paper_2009_14514_b200.stats import StepStats

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_rts.so")
_lib = None
_lib_lock = threading.Lock()

NEIGHBOR_WIDTH = 128  # wcsph.py:35
EMPTY = 127           # regions.py:35
VALIDITY_PERIOD = np.array([0, 1, 2, 4, 4], dtype=np.int32)  # pcisph.py:66
DEFAULT_SCHEDULE = (  # pcisph.py:72-77
    ((1, 2, 3, 4), (1, 2, 3, 4), (1,)),
    ((1, 2, 3, 4), (1,), (1,)),
    ((1, 2, 3, 4), (1, 2), (1,)),
    ((1, 2, 3, 4), (1,), (1,)),
)


def build_oracle() -> str:
    """Compile the C oracle (idempotent); returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build_oracle()
            L = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            I = ctypes.c_int64
            D = ctypes.c_double
            L.oracle_search_neighbors.restype = I
            L.oracle_search_neighbors.argtypes = [P, P, P, I, I, I, P, D, D, P, I, P, P, I, P]
            L.oracle_count_missing.restype = I
            L.oracle_count_missing.argtypes = [P, P, P, I, I, I, P, D, D, P, I, P, I, P]
            L.oracle_counting_sort.argtypes = [P, I, I, P, P]
            L.oracle_reduce_max.argtypes = [P, P, I, P]
            L.oracle_density_pressure.argtypes = [P, P, I, P, P, I, D, D, D, D, D, P, P]
            L.oracle_forces.argtypes = [P, P, P, I, P, P, I, D, D, D, D, D, D, I, P, P, P, P]
            L.oracle_ext_forces.argtypes = [P, P, P, I, P, P, I, D, D, D, D, D, I, P, P]
            L.oracle_predict_motion.argtypes = [P, P, P, P, I, D, D, P, P]
            L.oracle_predict_density.argtypes = [P, P, P, I, P, P, I, D, D, D, D, I, P, P]
            L.oracle_pressure_forces.argtypes = [P, P, P, I, P, P, I, D, D, D, D, I, P, P]
            L.oracle_pairwise_sum.restype = D
            L.oracle_pairwise_sum.argtypes = [P, I]
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_set_threads.argtypes = [ctypes.c_int]
            _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle kernels need contiguous arrays"
    return a.ctypes.data


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().oracle_pairwise_sum(_p(a), a.size))


# ----------------------------------------------------------------------
# kernel constants (kernels.py:58-80)
# ----------------------------------------------------------------------

class Kernels:
    def __init__(self, h: float):
        if h <= 0.0:
            raise ValueError("kernel support radius must be positive")
        self.h = float(h)
        self.h2 = self.h * self.h
        self.c_poly6 = 315.0 / (64.0 * np.pi * self.h**9)
        self.c_spiky = -45.0 / (np.pi * self.h**6)
        self.c_visc = 45.0 / (np.pi * self.h**6)


# ----------------------------------------------------------------------
# dense stencils (grid.py:33-62)
# ----------------------------------------------------------------------

_OFFSETS = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a, b, c) != (0, 0, 0)]


def _shifted(padded, d, shape):
    nx, ny, nz = shape
    return padded[1 + d[0]:1 + d[0] + nx, 1 + d[1]:1 + d[1] + ny, 1 + d[2]:1 + d[2] + nz]


def neighbor_min(field: np.ndarray, pad_value) -> np.ndarray:
    """min over the 26 adjacent cells (self excluded), pad outside."""
    padded = np.pad(field, 1, constant_values=pad_value)
    out = np.full_like(field, pad_value)
    for d in _OFFSETS:
        np.minimum(out, _shifted(padded, d, field.shape), out=out)
    return out


def dilate_mask(mask: np.ndarray, layers: int = 1) -> np.ndarray:
    """Chebyshev dilation by ``layers`` blocks."""
    cur = mask
    for _ in range(layers):
        padded = np.pad(cur, 1, constant_values=False)
        nxt = cur.copy()
        for d in _OFFSETS:
            nxt |= _shifted(padded, d, cur.shape)
        cur = nxt
    return cur


# ----------------------------------------------------------------------
# block grid (grid.py:220-394)
# ----------------------------------------------------------------------

class OracleGrid:
    def __init__(self, domain_min, domain_max, block_size: float, pad: float = 0.0):
        lo = np.asarray(domain_min, dtype=np.float64) - pad
        hi = np.asarray(domain_max, dtype=np.float64) + pad
        self.block_size = float(block_size)
        self.inv_block = 1.0 / self.block_size
        self.origin = lo
        self.dims = tuple(max(1, int(math.ceil((b - a) / self.block_size - 1e-12)))
                          for a, b in zip(lo, hi))
        self.n_cells = int(np.prod(self.dims))
        self.n_fluid = 0
        self.fluid_cells = self.starts = self.order = None
        self.occupancy = self.boundary_active = None

    @classmethod
    def for_scene(cls, scene: Scene, mode: str) -> "OracleGrid":
        return cls(scene.domain_min, scene.domain_max, scene.block_size(mode),
                   pad=scene.boundary_layers * scene.spacing)

    def cell_coords(self, x: np.ndarray) -> np.ndarray:
        c = np.floor((x - self.origin) * self.inv_block).astype(np.int64)
        return np.clip(c, 0, np.asarray(self.dims) - 1)

    def cell_ids(self, x: np.ndarray) -> np.ndarray:
        c = self.cell_coords(x)
        _, ny, nz = self.dims
        return (c[:, 0] * ny + c[:, 1]) * nz + c[:, 2]

    def rebuild(self, pos: np.ndarray, n_fluid: int) -> None:
        fluid = pos[:n_fluid]
        lo = self.origin
        hi = self.origin + np.asarray(self.dims) * self.block_size
        bad = ~np.all((fluid >= lo) & (fluid <= hi), axis=1) | ~np.isfinite(fluid).all(axis=1)
        if bad.any():
            raise NumericalError(
                f"{int(bad.sum())} fluid particle(s) left the simulation domain "
                f"(first index {int(np.flatnonzero(bad)[0])})")
        self.n_fluid = n_fluid
        self.fluid_cells = self.cell_ids(fluid)
        self.occupancy = (np.bincount(self.fluid_cells, minlength=self.n_cells) > 0
                          ).reshape(self.dims)
        if len(pos) > n_fluid:
            bcells = self.cell_ids(pos[n_fluid:])
            self.boundary_active = dilate_mask(self.occupancy, 1).ravel()[bcells]
            members = np.concatenate([np.arange(n_fluid),
                                      n_fluid + np.flatnonzero(self.boundary_active)])
            keys = np.concatenate([self.fluid_cells, bcells[self.boundary_active]])
        else:
            self.boundary_active = np.zeros(0, dtype=bool)
            members = np.arange(n_fluid)
            keys = self.fluid_cells
        self.starts, local = counting_sort(keys, self.n_cells)
        self.order = members[local]

    def search_into(self, pos, refresh, layers, h, nbr, cnt) -> None:
        if self.starts is None:
            raise RuntimeError("grid not built; call rebuild() first")
        if refresh.size == 0:
            return
        nx, ny, nz = self.dims
        refresh = _i64(refresh)
        layers = _i64(layers)
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        lost = lib().oracle_search_neighbors(
            _p(pos), _p(self.starts), _p(self.order), nx, ny, nz, _p(self.origin),
            self.inv_block, h * h, _p(refresh), refresh.size, _p(layers), _p(nbr),
            nbr.shape[1], _p(cnt))
        if lost:
            raise NumericalError(
                f"neighbor table overflow: {int(lost)} entries dropped "
                f"(table width {nbr.shape[1]}); the particle distribution has collapsed")

    def reduce_fluid_max(self, values: np.ndarray) -> np.ndarray:
        out = np.zeros(self.n_cells)
        v = np.ascontiguousarray(values, dtype=np.float64)
        lib().oracle_reduce_max(_p(v), _p(self.fluid_cells), v.size, _p(out))
        return out

    def count_missing_neighbors(self, pos, n_fluid, refresh, h, nbr, cnt) -> int:
        if refresh.size == 0:
            return 0
        audit = OracleGrid(self.origin, self.origin + np.asarray(self.dims) * self.block_size,
                           max(h, self.block_size))
        audit.rebuild(pos[:n_fluid], n_fluid)
        if len(pos) > n_fluid:
            keys = np.concatenate([audit.fluid_cells, audit.cell_ids(pos[n_fluid:])])
            audit.starts, audit.order = counting_sort(keys, audit.n_cells)
        nx, ny, nz = audit.dims
        refresh = _i64(refresh)
        return int(lib().oracle_count_missing(
            _p(pos), _p(audit.starts), _p(audit.order), nx, ny, nz, _p(audit.origin),
            audit.inv_block, h * h, _p(refresh), refresh.size, _p(nbr), nbr.shape[1],
            _p(cnt)))


def counting_sort(keys: np.ndarray, n_cells: int):
    keys = _i64(keys)
    starts = np.zeros(n_cells + 1, dtype=np.int64)
    order = np.empty(keys.size, dtype=np.int64)
    lib().oracle_counting_sort(_p(keys), keys.size, n_cells, _p(starts), _p(order))
    return starts, order


# ----------------------------------------------------------------------
# region fields (regions.py:38-125)
# ----------------------------------------------------------------------

def assign_regions(v_max, f_max, occupied, *, dt_base, block_size, particle_mass,
                   sound_speed, lambda_v, lambda_f, alpha, betas, n_max,
                   use_sound_criterion):
    region = np.where(occupied, np.int8(1), np.int8(0))
    r = block_size
    for n in range(2, n_max + 1):
        dt_n = n * dt_base
        ok = occupied & (region == n - 1)
        if use_sound_criterion and not dt_n <= lambda_v * r / sound_speed:
            break
        with np.errstate(divide="ignore", over="ignore"):
            fb = lambda_f * np.sqrt(r * particle_mass / f_max)
        ok = ok & ((f_max == 0.0) | (dt_n <= fb))
        if math.isfinite(betas[n]):
            ok = ok & (dt_n * v_max / r <= alpha * betas[n])
        region[ok] = n
    return region


def smooth_regions(region, dims):
    f = region.reshape(dims)
    nm = neighbor_min(np.where(f > 0, f, np.int8(EMPTY)), np.int8(EMPTY))
    new = np.minimum(f, nm)
    new[f == 0] = 0
    return new.ravel(), (new < f).ravel()


def expand_fast_regions(region, dims, layers: int = 4):
    f = region.reshape(dims)
    new = f.copy()
    new[(f > 2) & dilate_mask(f == 2, layers)] = 2
    new[(f > 1) & dilate_mask(f == 1, layers)] = 1
    return new.ravel()


def derive_observed(region, dims, error_blocks):
    f = region.reshape(dims)
    occ = f > 0
    nm = neighbor_min(np.where(occ, f, np.int8(EMPTY)), np.int8(EMPTY))
    obs = occ & (nm < f)
    e = error_blocks.reshape(dims)
    if e.any():
        obs |= occ & dilate_mask(e, 1) & ~e
    return obs.ravel()


# ----------------------------------------------------------------------
# RTS-WCSPH (wcsph.py:108-319)
# ----------------------------------------------------------------------

class OracleWcsph:
    mode_names = ("baseline", "rts")

    def __init__(self, scene: Scene, mode="rts", dt_cap=None, pin_region=None,
                 apply_correction=True, track_rho_variance=False, audit_neighbors=False,
                 n_regions=4):
        if mode not in self.mode_names:
            raise ValueError(f"unknown wcsph mode {mode!r}")
        self.scene, self.mode = scene, mode
        self.pin_region = pin_region
        self.apply_correction = apply_correction
        self.track_rho_variance = track_rho_variance
        self.audit_neighbors = audit_neighbors
        self.n_regions = n_regions
        self.kernel = Kernels(scene.support_radius)
        self.dt_base = scene.base_dt("wcsph")
        self.dt_cap = self.dt_base if dt_cap is None else dt_cap
        self.mass = scene.particle_mass
        self.mu = scene.viscosity * scene.rest_density
        self.b_stiff = scene.rest_density * scene.sound_speed**2 / TAIT_GAMMA
        self.betas = scene.betas(n_regions)
        self.alpha = scene.alpha_for("wcsph")
        fluid, wall = seed_particles(scene)
        nf = self.n_fluid = len(fluid)
        self.pos = np.concatenate([fluid, wall]) if len(wall) else fluid.copy()
        z3 = lambda: np.zeros((nf, 3))  # noqa: E731
        self.vel, self.acc, self.acc_prev, self.force = z3(), z3(), z3(), z3()
        self.rho = np.full(nf, scene.rest_density)
        self.pres = np.zeros(nf)
        self.dt_since = np.zeros(nf)
        self.dt_corr = np.zeros(nf)
        self.validity = np.zeros(nf, dtype=np.int32)
        self.region = np.ones(nf, dtype=np.int8)
        self.compute = np.ones(nf, dtype=bool)
        self.nbr = np.zeros((nf, NEIGHBOR_WIDTH), dtype=np.int64)
        self.cnt = np.zeros(nf, dtype=np.int64)
        self.grid = OracleGrid.for_scene(scene, "wcsph")
        self.gravity = np.asarray(scene.gravity)
        self._lo = np.asarray(scene.domain_min) + 0.1 * scene.spacing
        self._hi = np.asarray(scene.domain_max) - 0.1 * scene.spacing
        self.step_index = 0
        self.sim_time = 0.0
        self.missed_neighbors_total = 0
        self._missed_last = 0
        self._timers = {"neighbor": 0.0, "physics": 0.0, "rts": 0.0}

    def cfl_bound(self) -> float:
        sc = self.scene
        r = self.grid.block_size
        eq1 = sc.lambda_v * r / sc.sound_speed
        f_max = float(np.max(np.linalg.norm(self.force, axis=1))) if self.n_fluid else 0.0
        eq2 = sc.lambda_f * math.sqrt(r * self.mass / f_max) if f_max > 0.0 else math.inf
        return min(eq1, eq2)

    def particle_regions(self):
        return self.region if self.mode == "rts" else np.ones(self.n_fluid, dtype=np.int8)

    def advance(self):
        return [self.step()]

    def step(self) -> StepStats:
        for k in self._timers:
            self._timers[k] = 0.0
        t0 = time.perf_counter()
        self.grid.rebuild(self.pos, self.n_fluid)
        self._timers["neighbor"] += time.perf_counter() - t0
        if self.mode == "rts":
            t0 = time.perf_counter()
            self._assign_and_propagate()
            self._timers["rts"] += time.perf_counter() - t0
            dt = self.dt_base
            idx = np.flatnonzero(self.compute)
        else:
            dt = min(self.cfl_bound(), self.dt_cap)
            idx = np.arange(self.n_fluid)
        self._advance(dt, idx)
        self.step_index += 1
        self.sim_time += dt
        st = StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=int(idx.size),
                       frac_compute=idx.size / max(1, self.n_fluid),
                       missed_neighbors=self._missed_last,
                       t_neighbor=self._timers["neighbor"], t_physics=self._timers["physics"],
                       t_rts=self._timers["rts"])
        if self.track_rho_variance:
            st.rho_var = float(np.var(self.rho))
        return st

    def _assign_and_propagate(self):
        sc = self.scene
        v_max = self.grid.reduce_fluid_max(np.linalg.norm(self.vel, axis=1))
        f_max = self.grid.reduce_fluid_max(np.linalg.norm(self.force, axis=1))
        occ = self.grid.occupancy.ravel()
        raw = assign_regions(v_max, f_max, occ, dt_base=self.dt_base,
                             block_size=self.grid.block_size, particle_mass=self.mass,
                             sound_speed=sc.sound_speed, lambda_v=sc.lambda_v,
                             lambda_f=sc.lambda_f, alpha=self.alpha, betas=self.betas,
                             n_max=self.n_regions, use_sound_criterion=True)
        field, _ = smooth_regions(raw, self.grid.dims)
        if self.pin_region is not None:
            field = np.where(occ, np.int8(self.pin_region), np.int8(0))
        self.block_field = field
        block_n = field[self.grid.fluid_cells]
        self.validity -= 1
        renew = (self.validity <= 0) | (block_n != self.region)
        self.compute = renew
        self.region = np.where(renew, block_n, self.region)
        self.validity = np.where(renew, block_n.astype(np.int32), self.validity)

    def _advance(self, dt, idx):
        k = self.kernel
        nf = self.n_fluid
        self._missed_last = 0
        if idx.size:
            idx = _i64(idx)
            t0 = time.perf_counter()
            self.grid.search_into(self.pos, idx, np.ones(idx.size, dtype=np.int64), k.h,
                                  self.nbr, self.cnt)
            self._timers["neighbor"] += time.perf_counter() - t0
            if self.audit_neighbors:
                self._missed_last = self.grid.count_missing_neighbors(
                    self.pos, nf, idx, k.h, self.nbr, self.cnt)
                self.missed_neighbors_total += self._missed_last
            t0 = time.perf_counter()
            lib().oracle_density_pressure(
                _p(self.pos), _p(self.nbr), NEIGHBOR_WIDTH, _p(self.cnt), _p(idx), idx.size,
                self.mass, k.h2, k.c_poly6, self.b_stiff, self.scene.rest_density,
                _p(self.rho), _p(self.pres))
            if not math.isfinite(float(np.sum(self.rho[idx]))):
                raise NumericalError("non-finite density; the simulation has blown up")
            self.dt_corr[idx] = self.dt_since[idx]
            self.dt_since[idx] = 0.0
            self.acc_prev[idx] = self.acc[idx]
            grav = np.ascontiguousarray(self.gravity, dtype=np.float64)
            lib().oracle_forces(
                _p(self.pos), _p(self.vel), _p(self.nbr), NEIGHBOR_WIDTH, _p(self.cnt), _p(idx),
                idx.size, self.mass, k.h, k.c_spiky, k.c_visc, self.mu,
                self.scene.rest_density, nf, _p(self.rho), _p(self.pres), _p(grav),
                _p(self.force))
            self.acc[idx] = self.force[idx] / self.mass
            self._timers["physics"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        fl = self.pos[:nf]
        fl += self.vel * dt + self.acc * (0.5 * dt * dt)
        self.vel += self.acc * dt
        self.dt_since += dt
        if self.apply_correction and idx.size:
            da = self.acc[idx] - self.acc_prev[idx]
            dtc = self.dt_corr[idx][:, None]
            self.pos[idx] += da * (dtc * dtc / 6.0)
            self.vel[idx] += da * (dtc / 2.0)
        _clamp(self.pos[:nf], self.vel, self._lo, self._hi)
        self._timers["physics"] += time.perf_counter() - t0


def _clamp(fluid, vel, lo, hi):
    breached = (fluid < lo) | (fluid > hi)
    if breached.any():
        vel[breached] = 0.0
        np.clip(fluid, lo, hi, out=fluid)


# ----------------------------------------------------------------------
# RTS-PCISPH (pcisph.py:80-768)
# ----------------------------------------------------------------------

def validate_schedule(schedule, n_regions: int = 4) -> None:
    n_minor = len(schedule)
    cnt = np.zeros((n_minor, n_regions + 1), dtype=int)
    for j, rows in enumerate(schedule):
        for row in rows:
            for n in row:
                if not 1 <= n <= n_regions:
                    raise ConfigError(f"schedule names region {n} outside 1..{n_regions}")
                cnt[j, n] += 1
    for j in range(n_minor):
        for n in range(1, n_regions + 1):
            if cnt[j, n] < 1:
                raise ConfigError(f"region {n} receives no iteration on minor step {j + 1}")
    for n in range(1, n_regions + 1):
        if cnt[0, n] < 2:
            raise ConfigError(f"region {n} receives fewer than 2 iterations on the first minor step")
    for j in range(n_minor):
        if cnt[j, 1] < 3:
            raise ConfigError(f"region 1 receives fewer than 3 iterations on minor step {j + 1}")
    for n in range(1, n_regions + 1):
        w = 2 if n == 2 else min(n, n_minor)
        for j in range(n_minor):
            tot = sum(cnt[(j + q) % n_minor, n] for q in range(w))
            if tot < 3:
                raise ConfigError(f"region {n} receives {tot} < 3 iterations in the "
                                  f"{w}-minor window starting at minor step {j + 1}")


def template_factor(h: float, spacing: float) -> float:
    """|sum grad W|^2 + sum |grad W|^2 over the filled lattice (pcisph.py:131-148)."""
    c_spiky = -45.0 / (math.pi * h**6)
    sg = np.zeros(3)
    sd = 0.0
    reach = int(math.ceil(h / spacing))
    for ix in range(-reach, reach + 1):
        for iy in range(-reach, reach + 1):
            for iz in range(-reach, reach + 1):
                if ix == iy == iz == 0:
                    continue
                off = np.array([ix, iy, iz]) * spacing
                r = math.sqrt(float(off @ off))
                if r >= h:
                    continue
                s = 0.0 if r <= 0.0 else c_spiky * (h - r) * (h - r) / r
                g = s * (-off)
                sg += g
                sd += float(g @ g)
    return float(sg @ sg) + sd


class Controller:
    def __init__(self, n_nominal=4, n_current=4, recovery_left=0):
        self.n_nominal, self.n_current, self.recovery_left = n_nominal, n_current, recovery_left

    def note_major(self, early: bool) -> None:
        if early:
            self.n_current, self.recovery_left = 2, 10
        elif self.recovery_left > 0:
            self.recovery_left -= 1
            if self.recovery_left == 0:
                self.n_current = self.n_nominal


class OraclePcisph:
    mode_names = ("const", "adaptive", "rts")

    def __init__(self, scene: Scene, mode="rts", dt=None, schedule=DEFAULT_SCHEDULE,
                 pin_region=None, audit_neighbors=False, iteration_cap=24, local_attempts=4,
                 n_regions=4, state_f32=False):
        """``state_f32``: not the reference -- the reference algorithm with its
        particle state (pos, vel, f_ext, f_p, rho*) rounded to fp32 wherever
        the B200 solver stores it as fp32 (BASELINE.json's fp32 state).  The
        parity tests use it as the noise floor of fp32 state: how far the
        reference itself moves when its state is stored at that precision."""
        if mode not in self.mode_names:
            raise ValueError(f"unknown pcisph mode {mode!r}")
        validate_schedule(schedule, n_regions)
        self.state_f32 = state_f32
        self.scene, self.mode, self.schedule = scene, mode, schedule
        self.pin_region = pin_region
        self.audit_neighbors = audit_neighbors
        self.iteration_cap = iteration_cap
        self.local_attempts = local_attempts
        self.n_regions = n_regions
        self.kernel = Kernels(scene.support_radius)
        if dt is not None:
            self.dt = dt
        elif mode == "const":
            self.dt = scene.const_dt()
        else:
            self.dt = scene.base_dt("pcisph")
        self.mass = scene.particle_mass
        self.inv_mass = 1.0 / self.mass
        self.mu = scene.viscosity * scene.rest_density
        self.betas = scene.betas(n_regions)
        self.alpha = scene.alpha_for("pcisph")
        self.controller = Controller(scene.minor_steps, scene.minor_steps)
        self._delta_factor = template_factor(self.kernel.h, scene.spacing)
        fluid, wall = seed_particles(scene)
        nf = self.n_fluid = len(fluid)
        self.pos = np.concatenate([fluid, wall]) if len(wall) else fluid.copy()
        self.vel = np.zeros((nf, 3))
        self.f_ext = np.zeros((nf, 3))
        self.f_p = np.zeros((nf, 3))
        self.p = np.zeros(nf)
        self.rho_star = np.full(nf, scene.rest_density)
        self.err = np.zeros(nf)
        self.xstar = fluid.copy()
        self.vstar = np.zeros((nf, 3))
        self.region = np.ones(nf, dtype=np.int8)
        self.validity = np.zeros(nf, dtype=np.int32)
        self.compute = np.ones(nf, dtype=bool)
        self.in_se = np.zeros(nf, dtype=bool)
        self.in_sob = np.zeros(nf, dtype=bool)
        self.nbr = np.zeros((nf, NEIGHBOR_WIDTH), dtype=np.int64)
        self.cnt = np.zeros(nf, dtype=np.int64)
        self.grid = OracleGrid.for_scene(scene, "pcisph" if mode == "rts" else "wcsph")
        self.block_region = np.zeros(self.grid.n_cells, dtype=np.int8)
        self.gravity = np.asarray(scene.gravity)
        self._lo = np.asarray(scene.domain_min) + 0.1 * scene.spacing
        self._hi = np.asarray(scene.domain_max) - 0.1 * scene.spacing
        self.step_index = 0
        self.sim_time = 0.0
        self.missed_neighbors_total = 0
        self.local_entered_total = 0
        self.local_reverted_total = 0
        self._timers = {"neighbor": 0.0, "physics": 0.0, "rts": 0.0}

    # -- kernels ---------------------------------------------------------
    def _f32(self, *arrays):
        if self.state_f32:
            for a in arrays:
                a[...] = a.astype(np.float32)

    def delta(self, dt):
        rho0 = self.scene.rest_density
        return rho0 * rho0 / (2.0 * dt * dt * self.mass * self.mass * self._delta_factor)

    def particle_regions(self):
        return self.region if self.mode == "rts" else np.ones(self.n_fluid, dtype=np.int8)

    def advance(self):
        return self.major_step() if self.mode == "rts" else [self.sync_step()]

    def _ext(self, idx):
        k = self.kernel
        grav = np.ascontiguousarray(self.gravity, dtype=np.float64)
        lib().oracle_ext_forces(_p(self.pos), _p(self.vel), _p(self.nbr), NEIGHBOR_WIDTH,
                                _p(self.cnt), _p(idx), idx.size, self.mass, k.h, k.c_visc,
                                self.mu, self.scene.rest_density, self.n_fluid, _p(grav),
                                _p(self.f_ext))

    def _motion(self, dt):
        lib().oracle_predict_motion(_p(self.pos), _p(self.vel), _p(self.f_ext), _p(self.f_p),
                                    self.n_fluid, dt, self.inv_mass, _p(self.xstar),
                                    _p(self.vstar))

    def _density(self, idx):
        k = self.kernel
        lib().oracle_predict_density(_p(self.xstar), _p(self.pos), _p(self.nbr), NEIGHBOR_WIDTH,
                                     _p(self.cnt), _p(idx), idx.size, self.mass, k.h2,
                                     k.c_poly6, self.scene.rest_density, self.n_fluid,
                                     _p(self.rho_star), _p(self.err))

    def _pforces(self, idx):
        k = self.kernel
        lib().oracle_pressure_forces(_p(self.xstar), _p(self.pos), _p(self.nbr), NEIGHBOR_WIDTH,
                                     _p(self.cnt), _p(idx), idx.size, self.mass, k.h,
                                     k.c_spiky, self.scene.rest_density, self.n_fluid,
                                     _p(self.p), _p(self.f_p))

    def _avg_err(self):
        if not self.n_fluid:
            return 0.0
        mean = pairwise_sum(self.rho_star) / self.n_fluid
        return max(0.0, mean / self.scene.rest_density - 1.0)

    def _accumulate_pressure(self, idx, delta):
        pi = self.p[idx] + delta * (self.rho_star[idx] - self.scene.rest_density)
        np.maximum(pi, 0.0, out=pi)
        self.p[idx] = pi

    # -- synchronous baselines (pcisph.py:376-476) -------------------------
    def sync_step(self):
        for k in self._timers:
            self._timers[k] = 0.0
        nf = self.n_fluid
        dt = self.dt
        all_idx = np.arange(nf, dtype=np.int64)
        t0 = time.perf_counter()
        self.grid.rebuild(self.pos, nf)
        self.grid.search_into(self.pos, all_idx, np.ones(nf, dtype=np.int64), self.kernel.h,
                              self.nbr, self.cnt)
        self._timers["neighbor"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        self._ext(all_idx)
        self.p[:] = 0.0
        self.f_p[:] = 0.0
        iters, corrected = self._correct_all(dt, all_idx)
        self._integrate(dt)
        self._timers["physics"] += time.perf_counter() - t0
        max_err = float(self.err.max()) if nf else 0.0
        avg_err = self._avg_err()
        if self.mode == "adaptive":
            self._adapt_dt(iters)
        self.step_index += 1
        self.sim_time += dt
        return StepStats(step=self.step_index, time=self.sim_time, dt=dt, n_compute=nf,
                         frac_compute=1.0, iterations=iters, corrected=corrected,
                         iters_r1=iters, iters_r2=iters, iters_r3=iters, iters_r4=iters,
                         max_err=max_err, avg_err=avg_err,
                         t_neighbor=self._timers["neighbor"], t_physics=self._timers["physics"],
                         t_rts=self._timers["rts"])

    def _correct_all(self, dt, all_idx):
        sc = self.scene
        delta = self.delta(dt)
        it = corrected = 0
        while True:
            self._motion(dt)
            self._density(all_idx)
            self._accumulate_pressure(all_idx, delta)
            self._pforces(all_idx)
            it += 1
            corrected += self.n_fluid
            if not math.isfinite(float(self.rho_star.max())):
                raise NumericalError("non-finite predicted density; the simulation has blown up")
            conv = self.err.max() < sc.eta_max and self._avg_err() < sc.eta_avg
            if it >= 3 and conv:
                return it, corrected
            if it > self.iteration_cap + 3:
                raise NumericalError(
                    f"pressure solve did not converge within {it} iterations "
                    f"(max error {self.err.max():.4%} of rest density)")

    def _adapt_dt(self, iters):
        v_max = float(np.max(np.linalg.norm(self.vel, axis=1))) if self.n_fluid else 0.0
        if iters <= 5 and v_max * self.dt <= 0.4 * self.kernel.h:
            self.dt = min(self.dt * 1.002, 2.0 * self.scene.base_dt("pcisph"))
        else:
            self.dt = max(self.dt * 0.8, 0.1 * self.scene.const_dt())

    # -- regional mode (pcisph.py:482-768) ---------------------------------
    def major_step(self):
        n_minor = self.controller.n_current
        for k in self._timers:
            self._timers[k] = 0.0
        t0 = time.perf_counter()
        self.grid.rebuild(self.pos, self.n_fluid)
        self._timers["neighbor"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        self._assign_major_regions(n_minor)
        self._timers["rts"] += time.perf_counter() - t0
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

    def _levels(self, n_max):
        sc = self.scene
        occ = self.grid.occupancy.ravel()
        v_max = self.grid.reduce_fluid_max(np.linalg.norm(self.vel, axis=1))
        f_max = self.grid.reduce_fluid_max(np.linalg.norm(self.f_ext + self.f_p, axis=1))
        return occ, assign_regions(v_max, f_max, occ, dt_base=self.dt,
                                   block_size=self.grid.block_size, particle_mass=self.mass,
                                   sound_speed=sc.sound_speed, lambda_v=sc.lambda_v,
                                   lambda_f=sc.lambda_f, alpha=self.alpha, betas=self.betas,
                                   n_max=n_max, use_sound_criterion=False)

    def _assign_major_regions(self, n_minor):
        occ, raw = self._levels(min(self.n_regions, n_minor))
        field, _ = smooth_regions(raw, self.grid.dims)
        field = expand_fast_regions(field, self.grid.dims)
        if self.pin_region is not None:
            field = np.where(occ, np.int8(self.pin_region), np.int8(0))
        self.block_region = field
        self.region = field[self.grid.fluid_cells]
        self.validity = VALIDITY_PERIOD[self.region]
        self.compute[:] = True
        self.in_se[:] = False
        self._refresh_observed()

    def _refresh_observed(self):
        se = np.zeros(self.grid.n_cells, dtype=bool)
        if self.in_se.any():
            se[self.grid.fluid_cells[self.in_se]] = True
        self.in_sob = derive_observed(self.block_region, self.grid.dims, se)[self.grid.fluid_cells]

    def _minor_step(self, j, rows, last):
        k = self.kernel
        nf = self.n_fluid
        dt = self.dt
        missed = 0
        base = dict(self._timers)
        refresh = np.flatnonzero(self.compute).astype(np.int64)
        t0 = time.perf_counter()
        if refresh.size:
            layers = np.where(self.region[refresh] == 1, 2, 1).astype(np.int64)
            self.grid.search_into(self.pos, refresh, layers, k.h, self.nbr, self.cnt)
        self._timers["neighbor"] += time.perf_counter() - t0
        if self.audit_neighbors and refresh.size:
            missed = self.grid.count_missing_neighbors(self.pos, nf, refresh, k.h, self.nbr,
                                                       self.cnt)
            self.missed_neighbors_total += missed
        t0 = time.perf_counter()
        if refresh.size:
            self._ext(refresh)
            self._f32(self.f_ext)
        self.p[:] = 0.0
        self.f_p[:] = 0.0
        self._timers["physics"] += time.perf_counter() - t0
        iters, corrected, riters, g_count, early = self._correct_scheduled(dt, rows)
        t0 = time.perf_counter()
        self._integrate(dt)
        self._timers["physics"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        self.validity -= 1
        expired = self.validity <= 0
        self.compute = expired
        self.validity[expired] = VALIDITY_PERIOD[self.region[expired]]
        if not last:
            self._mark_timestep_updates()
        self._timers["rts"] += time.perf_counter() - t0
        self.step_index += 1
        self.sim_time += dt
        return StepStats(step=self.step_index, time=self.sim_time, dt=dt,
                         n_compute=int(refresh.size), frac_compute=refresh.size / max(1, nf),
                         iterations=iters, corrected=corrected, iters_r1=riters[1],
                         iters_r2=riters[2], iters_r3=riters[3], iters_r4=riters[4],
                         max_err=float(self.err.max()), avg_err=self._avg_err(),
                         early_term=int(early), missed_neighbors=missed,
                         t_neighbor=self._timers["neighbor"] - base["neighbor"],
                         t_physics=self._timers["physics"] - base["physics"],
                         t_rts=self._timers["rts"] - base["rts"])

    def _correct_scheduled(self, dt, rows):
        sc = self.scene
        nf = self.n_fluid
        delta = self.delta(dt)
        self.in_se[:] = False
        self._refresh_observed()
        it = g_count = corrected = 0
        riters = [0, 0, 0, 0, 0]
        local_active = local_banned = False
        local_run = 0
        snap_p = snap_fp = None
        early = False
        while True:
            if local_active:
                turn = np.zeros(nf, dtype=bool)
            else:
                row = rows[g_count % len(rows)]
                turn = np.isin(self.region, row)
                for n in row:
                    if n <= self.n_regions:
                        riters[n] += 1
            pred = np.flatnonzero(turn | self.in_se | self.in_sob).astype(np.int64)
            force = np.flatnonzero(turn | self.in_se).astype(np.int64)
            self._motion(dt)
            self._density(pred)
            self._accumulate_pressure(force, delta)
            self._f32(self.rho_star)
            self.in_se = self.err > 0.5 * sc.eta_max
            self._refresh_observed()
            self._pforces(force)
            self._f32(self.f_p)
            it += 1
            corrected += int(pred.size)
            if local_active:
                local_run += 1
            else:
                g_count += 1
            if not math.isfinite(float(self.rho_star[pred].max() if pred.size else 0.0)):
                raise NumericalError("non-finite predicted density; the simulation has blown up")
            max_err = float(self.err.max())
            avg_err = self._avg_err()
            if max_err < sc.eta_max and avg_err < sc.eta_avg:
                if it >= 3:
                    break
                continue
            if it < 3:
                continue
            if local_active:
                if local_run >= self.local_attempts:
                    self.p[:] = snap_p
                    self.f_p[:] = snap_fp
                    local_active = False
                    local_banned = True
                    self.local_reverted_total += 1
            elif avg_err * 100.0 < sc.rho_T and not local_banned and self.in_se.any():
                local_active = True
                local_run = 0
                snap_p = self.p.copy()
                snap_fp = self.f_p.copy()
                self.local_entered_total += 1
            if g_count > 6:
                early = True
            if g_count > self.iteration_cap:
                raise NumericalError(
                    f"pressure solve used {g_count} global iterations in one minor step "
                    f"(max error {max_err:.4%} of rest density)")
        return it, corrected, riters, g_count, early

    def _mark_timestep_updates(self):
        occ, required = self._levels(min(self.n_regions, self.controller.n_current))
        cur = self.block_region
        violating = occ & (required < cur) & (cur > 0)
        if not violating.any():
            return
        dims = self.grid.dims
        vf = np.where(violating, required, np.int8(EMPTY)).reshape(dims)
        spread = np.minimum(vf, neighbor_min(vf, np.int8(EMPTY)))
        new = np.where(occ, np.minimum(cur, spread.ravel()), np.int8(0))
        changed = new < cur
        self.block_region = new
        pm = changed[self.grid.fluid_cells]
        if pm.any():
            self.region[pm] = new[self.grid.fluid_cells[pm]]
            self.compute[pm] = True
            self.validity[pm] = VALIDITY_PERIOD[self.region[pm]]

    def _integrate(self, dt):
        self.vel += (self.f_ext + self.f_p) * (dt * self.inv_mass)
        fl = self.pos[:self.n_fluid]
        fl += self.vel * dt
        _clamp(fl, self.vel, self._lo, self._hi)
        self._f32(fl, self.vel)


def make_oracle(scene: Scene, name: str, **kw):
    """Factory mirroring ``rts_sph.bench.make_solver`` (bench.py:50-61)."""
    table = {"wcsph": (OracleWcsph, "baseline"), "wcsph-rts": (OracleWcsph, "rts"),
             "pcisph-const": (OraclePcisph, "const"),
             "pcisph-adaptive": (OraclePcisph, "adaptive"), "pcisph-rts": (OraclePcisph, "rts")}
    if name not in table:
        raise ConfigError(f"unknown solver {name!r}")
    cls, mode = table[name]
    return cls(scene, mode=mode, **kw)
