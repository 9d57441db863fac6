"""SPH kernel constants and host reference forms (``rts_sph.kernels``,
/root/reference/pkg/src/rts_sph/kernels.py:23-108).

The device evaluates the same three formulas inside the librtssph pair
kernels (csrc/common.cuh: poly6, spiky, visc_lap) in fp64 with the same
operation order; the constants below are what the host passes in RtsParams.
"""

from __future__ import annotations

import dataclasses

import numpy as np

__all__ = ["KernelSet", "poly6_w", "spiky_grad_scale", "viscosity_lap"]


def poly6_w(r2, h2, c_poly6):
    d = h2 - r2
    return 0.0 if d <= 0.0 else c_poly6 * d * d * d


def spiky_grad_scale(r, h, c_spiky):
    if r <= 0.0 or r >= h:
        return 0.0
    d = h - r
    return c_spiky * d * d / r


def viscosity_lap(r, h, c_visc):
    d = h - r
    return 0.0 if d <= 0.0 else c_visc * d


@dataclasses.dataclass
class KernelSet:
    """Kernel constants for support radius ``h``: poly6 315/(64 pi h^9),
    spiky gradient -45/(pi h^6), viscosity Laplacian 45/(pi h^6)."""

    h: float
    h2: float = dataclasses.field(init=False)
    c_poly6: float = dataclasses.field(init=False)
    c_spiky: float = dataclasses.field(init=False)
    c_visc: float = dataclasses.field(init=False)

    def __post_init__(self):
        if self.h <= 0.0:
            raise ValueError("kernel support radius must be positive")
        h = float(self.h)
        self.h = h
        self.h2 = h * h
        self.c_poly6 = 315.0 / (64.0 * np.pi * h**9)
        self.c_spiky = -45.0 / (np.pi * h**6)
        self.c_visc = 45.0 / (np.pi * h**6)

    def density(self, r):
        r = np.asarray(r, dtype=np.float64)
        d = np.clip(self.h2 - r * r, 0.0, None)
        return self.c_poly6 * d**3

    def grad_pressure(self, offsets):
        x = np.asarray(offsets, dtype=np.float64)
        r = np.linalg.norm(x, axis=-1)
        d = np.where((r > 0.0) & (r < self.h), self.h - r, 0.0)
        return (self.c_spiky * d * d / np.maximum(r, 1e-300))[..., None] * x

    def laplacian_viscosity(self, r):
        r = np.asarray(r, dtype=np.float64)
        return np.where(r < self.h, self.c_visc * np.clip(self.h - r, 0.0, None), 0.0)
