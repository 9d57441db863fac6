"""Uniform block grid on the B200 -- drop-in for ``rts_sph.grid.BlockGrid``
(/root/reference/pkg/src/rts_sph/grid.py:220-394).

Geometry (origin, dims, inv_block) is computed on the host with the
reference's expressions (grid.py:223-244).  ``rebuild`` runs the librtssph
kernels: fp64 block keys with the domain check, occupancy counts, boundary
culling by the 1-dilated occupancy, a tile scan, and the stable counting
sort into ``starts``/``order`` (bit-identical to the reference's CSR:
fluid ascending, then active boundary ascending, inside every block).

All per-particle and per-block arrays are device tensors (int32 indices,
bool masks); ``order`` holds reference particle indices (fluid first,
boundary as ``n_fluid + b``).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from ._device import Arena, Counters, as_device_f32, raise_on_errors, require_cuda

__all__ = ["BlockGrid", "neighbor_min", "dilate_mask"]


def neighbor_min(field, pad_value):
    """grid.py:33-45 of the reference (26-neighbour minimum, ``pad_value``
    outside), evaluated on the device: ``regions.neighbor_min``."""
    from .regions import neighbor_min as _nm
    return _nm(field, pad_value)


def dilate_mask(mask, layers: int = 1):
    """grid.py:48-62 of the reference (Chebyshev dilation by ``layers``),
    evaluated on the device: ``regions.dilate_mask``."""
    from .regions import dilate_mask as _dm
    return _dm(mask, layers)


class BlockGrid:
    """Block decomposition of the padded domain at a fixed block edge."""

    def __init__(self, domain_min, domain_max, block_size: float, pad: float = 0.0,
                 device="cuda", arena: Arena | None = None):
        lo = np.asarray(domain_min, dtype=np.float64) - pad
        hi = np.asarray(domain_max, dtype=np.float64) + pad
        self.block_size = float(block_size)
        self.inv_block = 1.0 / self.block_size
        self.origin = lo
        self.dims = tuple(max(1, int(math.ceil((b - a) / self.block_size - 1e-12)))
                          for a, b in zip(lo, hi))
        self.n_cells = int(np.prod(self.dims))
        if self.n_cells >= 2**31 - 1:
            raise ValueError("grid has more than 2^31 blocks")
        self.device = require_cuda(device)
        self.arena = arena if arena is not None else Arena(self.device)
        self._own_counters = arena is None
        self.counters = Counters(self.arena) if arena is None else None
        self.n_fluid = 0
        self.n_bound = -1
        self.n_sorted = 0
        self._alloc_cells()
        self.params = N.RtsParams()
        self.fill_params(self.params)

    @classmethod
    def for_scene(cls, scene, mode: str, device="cuda", arena=None) -> "BlockGrid":
        return cls(scene.domain_min, scene.domain_max, scene.block_size(mode),
                   pad=scene.boundary_layers * scene.spacing, device=device, arena=arena)

    # -- geometry -----------------------------------------------------------
    def fill_params(self, p: N.RtsParams) -> None:
        hi = self.origin + np.asarray(self.dims) * self.block_size
        for a in range(3):
            p.origin[a] = float(self.origin[a])
            p.grid_hi[a] = float(hi[a])
            p.dims[a] = int(self.dims[a])
        p.block_size = self.block_size
        p.inv_block = self.inv_block
        p.n_cells = self.n_cells

    def cell_coords(self, positions) -> np.ndarray:
        x = np.asarray(positions, dtype=np.float64)
        c = np.floor((x - self.origin) * self.inv_block).astype(np.int64)
        return np.clip(c, 0, np.asarray(self.dims) - 1)

    def cell_ids(self, positions) -> np.ndarray:
        c = self.cell_coords(positions)
        _, ny, nz = self.dims
        return (c[:, 0] * ny + c[:, 1]) * nz + c[:, 2]

    # -- buffers ------------------------------------------------------------
    def _alloc_cells(self) -> None:
        A, nc = self.arena, self.n_cells
        i32, i8, u8 = torch.int32, torch.int8, torch.uint8
        A.alloc("cell_count", (nc,), i32, 0)
        A.alloc("cell_bcount", (nc,), i32, 0)
        A.alloc("starts", (nc + 1,), i32, 0)
        A.alloc("fill", (nc,), i32, 0)
        tiles = -(-nc // 1024)  # grid.cu k_scan_lookback: counter + one 64-bit status per tile
        A.alloc("scan_tmp", (2 * tiles + 64,), i32, 0)
        A.alloc("vmax", (nc,), torch.float64, 0)
        A.alloc("fmax", (nc,), torch.float64, 0)
        A.alloc("block_raw", (nc,), i8, 0)
        A.alloc("block_field", (nc,), i8, 0)
        A.alloc("block_tmp", (nc,), i8, 0)
        A.alloc("block_flag", (nc,), u8, 0)

    def _ensure_particles(self, n_fluid: int, n_total: int) -> None:
        A = self.arena
        if "fluid_cells" not in A.t or A["fluid_cells"].numel() < max(n_fluid, 1):
            A.alloc("fluid_cells", (max(n_fluid, 1),), torch.int32, 0)
        self.n_fluid = n_fluid
        if "order" not in A.t or A["order"].numel() < max(n_total, 1):
            A.alloc("order", (max(n_total, 1),), torch.int32, 0)

    def bind_boundary(self, boundary_pos, n_fluid: int) -> None:
        """Static binning of the wall shell (done once per solver): blocks
        holding wall samples, their CSR of wall indices (ascending), so each
        rebuild only decides which wall blocks are active (grid.py:279-290)."""
        A = self.arena
        bpos = np.asarray(boundary_pos, dtype=np.float64).reshape(-1, 3)
        nb = len(bpos)
        self.n_bound = nb
        A["cell_bcount"].zero_()
        if nb == 0:
            self.n_bcells = 0
            for name in ("bcell_ids", "bcell_start", "bidx", "bcell_of", "bcell_active"):
                A.alloc(name, (1,), torch.int32 if name != "bcell_active" else torch.uint8, 0)
            self._bslot = torch.zeros(0, dtype=torch.int64, device=self.device)
            return
        cells = self.cell_ids(bpos)
        srt = np.argsort(cells, kind="stable")
        ids, first = np.unique(cells[srt], return_index=True)
        starts = np.append(first, nb).astype(np.int32)
        slot = np.searchsorted(ids, cells)
        self.n_bcells = len(ids)
        dev = self.device
        A.bind("bcell_ids", torch.as_tensor(ids.astype(np.int32), device=dev))
        A.bind("bcell_start", torch.as_tensor(starts, device=dev))
        self._bsrt = torch.as_tensor(srt.astype(np.int32), device=dev)
        self._bidx_base = n_fluid
        A.bind("bidx", self._bsrt + n_fluid)
        # block index (into bcell_ids) of every member of the wall CSR, for the
        # member-parallel scatter (grid.cu k_scatter)
        member_t = np.repeat(np.arange(len(ids), dtype=np.int32), np.diff(starts))
        A.bind("bcell_of", torch.as_tensor(member_t, device=dev))
        A.alloc("bcell_active", (self.n_bcells,), torch.uint8, 0)
        self._bslot = torch.as_tensor(slot.astype(np.int64), device=dev)

    def shift_boundary(self, n_fluid: int) -> None:
        """Wall rows follow the fluid rows: re-offset the static wall CSR when
        the fluid count changes (distributed ranks)."""
        if self.n_bound > 0 and n_fluid != self._bidx_base:
            self.arena.bind("bidx", self._bsrt + n_fluid)
            self._bidx_base = n_fluid

    # -- device passes (async, used by the solvers) -----------------------------
    def launch_rebuild(self, p, stream, want_maxima=False, add_fp=False) -> None:
        s = stream.cuda_stream
        N.call("rts_grid_keys", p, self.arena.buf, int(want_maxima), int(add_fp), s)
        N.call("rts_grid_sort", p, self.arena.buf, s)

    # -- reference-facing API -------------------------------------------------
    def rebuild(self, pos, n_fluid: int) -> None:
        """Re-bin ``pos`` (fluid rows first, boundary after); raises
        NumericalError if fluid left the padded grid or is non-finite."""
        x = as_device_f32(pos, self.device).reshape(-1, 3)
        n_total = x.shape[0]
        nb = n_total - n_fluid
        self._ensure_particles(n_fluid, n_total)
        self.bind_boundary(x[n_fluid:].cpu().numpy(), n_fluid)
        self.arena.bind("pos", x)
        self._pos_ref = x
        p = self.params
        p.n_fluid = n_fluid
        p.n_bound = nb
        p.n_bcells = self.n_bcells
        stream = torch.cuda.current_stream(self.device)
        ctr = self.counters
        ctr.reset(stream)
        self.launch_rebuild(p, stream)
        c = ctr.read(stream)
        raise_on_errors(c)
        self.n_sorted = int(c.n_sorted)

    @property
    def fluid_cells(self) -> torch.Tensor:
        return self.arena["fluid_cells"][: self.n_fluid]

    @property
    def starts(self) -> torch.Tensor:
        return self.arena["starts"]

    @property
    def order(self) -> torch.Tensor:
        return self.arena["order"][: self.n_sorted]

    @property
    def occupancy(self) -> torch.Tensor:
        return (self.arena["cell_count"] > 0).reshape(self.dims)

    @property
    def boundary_active(self) -> torch.Tensor:
        if self.n_bound <= 0:
            return torch.zeros(0, dtype=torch.bool, device=self.device)
        return self.arena["bcell_active"][self._bslot].bool()

    def _table_buffers(self, n_total: int, width: int, n_refresh: int) -> None:
        A = self.arena
        stride = -(-max(n_total, 1) // 32) * 32
        if getattr(self, "_tbl", None) != (n_total, width, n_refresh):
            A.alloc("cpos", (n_total + 4, 4), torch.float32, 0)
            A.alloc("slot_of", (max(self.n_fluid, 1),), torch.int32, 0)
            A.alloc("nbr", (width, stride), torch.int32, 0)
            A.alloc("cnt", (max(n_total, 1),), torch.int32, 0)
            A.alloc("active", (max(n_refresh, 1),), torch.int32, 0)
            self._tbl = (n_total, width, n_refresh)
        self.params.nbr_stride = stride
        self.params.width = width

    def search_into(self, pos, refresh, layers, h: float, nbr, cnt) -> None:
        """Neighbour tables of the particles in ``refresh`` at positions
        ``pos`` on this (possibly stale) grid, ``layers[t]`` block layers
        around refresh[t] (grid.py:297-331): rows nbr[i, :cnt[i]] in the
        reference's fill order; NumericalError on table overflow.  ``nbr`` /
        ``cnt`` are numpy arrays or tensors, written in place."""
        from .errors import NumericalError
        if getattr(self, "n_sorted", None) is None:
            raise RuntimeError("grid not built; call rebuild() first")
        ref = torch.as_tensor(np.asarray(refresh), device=self.device).to(torch.int32).reshape(-1)
        n = int(ref.numel())
        if n == 0:
            return
        x = as_device_f32(pos, self.device).reshape(-1, 3)
        width = int(nbr.shape[1])
        self._table_buffers(x.shape[0], width, n)
        A, p = self.arena, self.params
        A.bind("pos", x)
        A["active"][:n].copy_(ref)
        lay = torch.as_tensor(np.asarray(layers), device=self.device).to(torch.int8).reshape(-1)
        p.h2 = float(h) * float(h)
        p.n_fluid = self.n_fluid
        stream = torch.cuda.current_stream(self.device)
        self.counters.reset(stream)  # clears the overflow count; restore the CSR size
        off = N.RtsCounters.n_sorted.offset
        self.counters.dev[off:off + 4].view(torch.int32).fill_(int(self.n_sorted))
        N.call("rts_pci_gather", p, A.buf, stream.cuda_stream)  # candidates at `pos`
        N.call("rts_grid_search", p, A.buf, lay.data_ptr(), n, stream.cuda_stream)
        c = self.counters.read(stream)
        idx = ref.long()
        rows = A["nbr"][:, idx].T.contiguous()  # (n, width)
        counts = A["cnt"][idx]
        self._write_rows(nbr, cnt, idx, rows, counts)
        if c.overflow:
            raise NumericalError(
                f"neighbor table overflow: {int(c.overflow)} entries dropped "
                f"(table width {width}); the particle distribution has collapsed")

    @staticmethod
    def _write_rows(nbr, cnt, idx, rows, counts) -> None:
        q = torch.arange(rows.shape[1], device=rows.device)
        keep = q[None, :] < counts[:, None].long()
        if isinstance(nbr, torch.Tensor):
            i = idx.to(nbr.device)
            cur = nbr[i]
            nbr[i] = torch.where(keep.to(nbr.device), rows.to(nbr.device, nbr.dtype), cur)
            cnt[i] = counts.to(cnt.device, cnt.dtype)
        else:
            i = idx.cpu().numpy()
            r, k = rows.cpu().numpy(), keep.cpu().numpy()
            cur = nbr[i]
            nbr[i] = np.where(k, r.astype(nbr.dtype), cur)
            cnt[i] = counts.cpu().numpy().astype(cnt.dtype)

    def neighbors(self, pos, point_index: int, layers: int = 1) -> np.ndarray:
        """Candidate indices around one particle: every member of the
        (2 layers + 1)^3 blocks around its current block (grid.py:333-345)."""
        if getattr(self, "n_sorted", None) is None:
            raise RuntimeError("grid not built; call rebuild() first")
        x = np.asarray(pos if not isinstance(pos, torch.Tensor) else pos.cpu().numpy())
        cx, cy, cz = self.cell_coords(x[point_index:point_index + 1])[0]
        nx, ny, nz = self.dims
        starts = self.arena["starts"].cpu().numpy()
        order = self.order.cpu().numpy()
        out = []
        for ax in range(max(0, cx - layers), min(nx, cx + layers + 1)):
            for ay in range(max(0, cy - layers), min(ny, cy + layers + 1)):
                base = (ax * ny + ay) * nz
                z0, z1 = max(0, cz - layers), min(nz, cz + layers + 1)
                out.append(order[starts[base + z0]:starts[base + z1]])
        return np.concatenate(out).astype(np.int64) if out else np.zeros(0, dtype=np.int64)

    def count_missing_neighbors(self, pos, n_fluid: int, refresh, h: float, nbr, cnt) -> int:
        """True neighbours (fresh exhaustive search) absent from the tables of
        ``refresh`` (grid.py:353-394)."""
        ref = torch.as_tensor(np.asarray(refresh), device=self.device).to(torch.int32).reshape(-1)
        n = int(ref.numel())
        if n == 0:
            return 0
        x = as_device_f32(pos, self.device).reshape(-1, 3)
        audit = BlockGrid(self.origin, self.origin + np.asarray(self.dims) * self.block_size,
                          max(float(h), self.block_size), device=self.device)
        audit.rebuild(x, n_fluid)
        audit._table_buffers(x.shape[0], int(nbr.shape[1]), 1)
        pa = audit.params
        pa.h2 = float(h) * float(h)
        stream = torch.cuda.current_stream(self.device)
        N.call("rts_pci_gather", pa, audit.arena.buf, stream.cuda_stream)
        # the tables under audit, column-major, with the refresh list
        tb = Arena(self.device)
        width = int(nbr.shape[1])
        stride = -(-max(x.shape[0], 1) // 32) * 32
        t_nbr = torch.as_tensor(np.asarray(nbr) if not isinstance(nbr, torch.Tensor) else nbr,
                                device=self.device).to(torch.int32)
        tb.alloc("nbr", (width, stride), torch.int32, 0)
        tb["nbr"][:, : t_nbr.shape[0]].copy_(t_nbr.T)
        t_cnt = torch.as_tensor(np.asarray(cnt) if not isinstance(cnt, torch.Tensor) else cnt,
                                device=self.device).to(torch.int32).reshape(-1)
        tb.bind("cnt", t_cnt.contiguous())
        tb.alloc("active", (n,), torch.int32, 0)
        tb["active"].copy_(ref)
        tb.bind("pos", x)
        ctr = Counters(tb)
        ctr.reset(stream)
        n_view = ctr.dev[N.RtsCounters.n_compute.offset:N.RtsCounters.n_compute.offset + 4]
        n_view.view(torch.int32).fill_(n)
        pa.nbr_stride = stride
        N.call("rts_pci_audit", pa, audit.arena.buf, tb.buf, stream.cuda_stream)
        return int(ctr.read(stream).missing)

    def reduce_fluid_max(self, values) -> torch.Tensor:
        """Per-block max of a fluid scalar, zeros in empty blocks (grid.py:347-351)."""
        v = torch.as_tensor(values, device=self.device).to(torch.float64).reshape(-1)
        out = torch.zeros(self.n_cells, dtype=torch.float64, device=self.device)
        idx = self.fluid_cells.to(torch.int64)
        return out.scatter_reduce(0, idx, v, reduce="amax", include_self=True)
