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
