"""Region fields -- the public functions of the reference's ``rts_sph.regions``
(/root/reference/pkg/src/rts_sph/regions.py:38-125), same signatures and
results (bit-exact), evaluated by the librtssph kernels the solvers use
(``rts_block_levels`` for assign_regions, ``rts_region_op`` for the others).

Inputs and outputs are numpy arrays over the grid cells, as in the
reference; the arrays go to the CUDA device (``device``, default ``cuda``)
and back.  There is no CPU path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["assign_regions", "smooth_regions", "expand_fast_regions", "derive_observed",
           "neighbor_min", "dilate_mask"]


def _setup(n_cells: int, dims, device):
    import torch

    from . import _native as N
    from ._device import Arena, Counters, require_cuda
    dev = require_cuda(device)
    A = Arena(dev)
    for name, dt in (("cell_count", torch.int32), ("vmax", torch.float64),
                     ("fmax", torch.float64), ("block_raw", torch.int8),
                     ("block_field", torch.int8), ("block_tmp", torch.int8),
                     ("block_flag", torch.uint8)):
        A.alloc(name, (max(n_cells, 1),), dt, 0)
    Counters(A)
    p = N.RtsParams()
    p.n_cells = int(n_cells)
    d = tuple(int(x) for x in dims) if dims is not None else (int(n_cells), 1, 1)
    p.dims[0], p.dims[1], p.dims[2] = d
    return A, p, torch.cuda.current_stream(dev)


def _put(A, name, values):
    import torch
    t = A[name]
    t.copy_(torch.as_tensor(np.ascontiguousarray(values).reshape(-1)).to(t.dtype))


def _get(A, name, dtype):
    return A[name].cpu().numpy().astype(dtype, copy=False)


def _call(name, *args):
    from . import _native as N
    N.call(name, *args)


def assign_regions(v_max, f_max, occupied, *, dt_base: float, block_size: float,
                   particle_mass: float, sound_speed: float, lambda_v: float, lambda_f: float,
                   alpha: float, betas, n_max: int, use_sound_criterion: bool,
                   device="cuda") -> np.ndarray:
    """Per-block region ids from per-block maxima (regions.py:38-75):
    int8, 0 for empty blocks."""
    v = np.asarray(v_max, dtype=np.float64).reshape(-1)
    A, p, st = _setup(v.size, None, device)
    _put(A, "vmax", v)
    _put(A, "fmax", np.asarray(f_max, dtype=np.float64))
    _put(A, "cell_count", np.asarray(occupied).astype(np.int32))
    p.dt_base, p.block_size, p.mass = float(dt_base), float(block_size), float(particle_mass)
    p.sound_speed, p.lambda_v, p.lambda_f = float(sound_speed), float(lambda_v), float(lambda_f)
    p.alpha, p.n_max, p.use_sound = float(alpha), int(n_max), int(bool(use_sound_criterion))
    for n in range(8):
        p.betas[n] = float(betas[n]) if n < len(betas) else float("inf")
    _call("rts_block_levels", p, A.buf, 2, st.cuda_stream)  # assign only
    return _get(A, "block_raw", np.int8)


def smooth_regions(region, dims) -> tuple[np.ndarray, np.ndarray]:
    """One min-with-neighbours pass (regions.py:78-91): (new field, mask of
    blocks whose region dropped)."""
    r = np.asarray(region, dtype=np.int8).reshape(-1)
    A, p, st = _setup(r.size, dims, device="cuda")
    _put(A, "block_raw", r)
    _call("rts_region_op", p, A.buf, 0, 0, st.cuda_stream)
    new = _get(A, "block_field", np.int8)
    return new, new < r


def expand_fast_regions(region, dims, layers: int = 4) -> np.ndarray:
    """Grow regions 1 and 2 by ``layers`` blocks (regions.py:94-107)."""
    r = np.asarray(region, dtype=np.int8).reshape(-1)
    A, p, st = _setup(r.size, dims, device="cuda")
    _put(A, "block_tmp", r)
    _call("rts_region_op", p, A.buf, 1, int(layers), st.cuda_stream)
    return _get(A, "block_field", np.int8)


def derive_observed(region, dims, error_blocks) -> np.ndarray:
    """Observed-block mask for the final field (regions.py:110-125)."""
    r = np.asarray(region, dtype=np.int8).reshape(-1)
    A, p, st = _setup(r.size, dims, device="cuda")
    _put(A, "block_field", r)
    _put(A, "block_flag", np.asarray(error_blocks).reshape(-1).astype(np.uint8))
    _call("rts_region_op", p, A.buf, 2, 0, st.cuda_stream)
    return _get(A, "block_tmp", np.int8).astype(bool)


def dilate_mask(mask, layers: int = 1) -> np.ndarray:
    """Chebyshev dilation of a boolean 3-D mask by ``layers`` blocks
    (grid.py:48-62), via the expansion pass (a mask of 2s grown over 1s)."""
    m = np.asarray(mask, dtype=bool)
    field = np.where(m, 2, 3).astype(np.int8)
    grown = expand_fast_regions(field.reshape(-1), m.shape, layers).reshape(m.shape)
    return grown == 2


def neighbor_min(field, pad_value) -> np.ndarray:
    """Minimum over each cell's 26 neighbours, self excluded, cells outside
    the grid counting as ``pad_value`` (grid.py:33-45), for int8 fields."""
    f = np.asarray(field)
    if f.dtype != np.int8:
        raise TypeError("neighbor_min: int8 fields (the region stencils)")
    A, p, st = _setup(f.size, f.shape, device="cuda")
    _put(A, "block_raw", f.reshape(-1))
    _call("rts_region_op", p, A.buf, 3, int(pad_value), st.cuda_stream)
    return _get(A, "block_field", np.int8).reshape(f.shape)
