"""Device-memory plumbing shared by the solvers: torch-owned buffers, the
``RtsBuffers`` pointer table, the per-step counters block and phase timers.

torch is used only as the allocator / stream owner; every computation on
these buffers is a librtssph kernel.
"""

from __future__ import annotations

import ctypes
import functools
import os

import numpy as np
import torch

from . import _native as N
from .errors import NumericalError

INT32_MAX = 2**31 - 1

_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def raw_stream(index: int) -> int:
    """cudaStream_t of the current stream of device ``index``: the cheap
    query (torch.cuda.current_stream builds a Stream object per call, ~7 us,
    which the host-driven paths pay on every launch)."""
    if _raw_stream is not None:
        return _raw_stream(index)
    return torch.cuda.current_stream(index).cuda_stream


NVTX = os.environ.get("RTS_SPH_NVTX", "0") not in ("", "0")


def nvtx_range(name: str):
    """Decorator: an NVTX range around a host-side phase (major step, base
    step, slab exchange) when RTS_SPH_NVTX=1, so a timeline capture shows the
    solver's phases over its kernels; the undecorated function otherwise."""
    def wrap(fn):
        if not NVTX:
            return fn

        @functools.wraps(fn)
        def inner(*a, **kw):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **kw)
            finally:
                torch.cuda.nvtx.range_pop()
        return inner
    return wrap


def device_index(device: torch.device) -> int:
    return device.index if device.index is not None else torch.cuda.current_device()


def require_cuda(device) -> torch.device:
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError("the B200 solvers run on CUDA devices only (no CPU fallback)")
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible; the B200 solvers have no CPU fallback")
    N.load()
    return dev


class Arena:
    """Named device tensors + the RtsBuffers table that points at them."""

    def __init__(self, device: torch.device):
        self.device = device
        self.t: dict[str, torch.Tensor] = {}
        self.buf = N.RtsBuffers()

    def alloc(self, name: str, shape, dtype, fill=None) -> torch.Tensor:
        if fill is None:
            x = torch.empty(shape, dtype=dtype, device=self.device)
        else:
            x = torch.full(shape, fill, dtype=dtype, device=self.device)
        self.bind(name, x)
        return x

    def bind(self, name: str, x: torch.Tensor) -> None:
        self.t[name] = x
        if name in N.BUFFER_FIELDS:
            setattr(self.buf, name, x.data_ptr() if x.numel() else None)

    def __getitem__(self, name):
        return self.t[name]


class Counters:
    """The RtsCounters block: reset before a step, read back after it."""

    SIZE = ctypes.sizeof(N.RtsCounters)

    def __init__(self, arena: Arena):
        self.dev = arena.alloc("ctr", (self.SIZE,), torch.uint8, 0)
        self.host = torch.zeros(self.SIZE, dtype=torch.uint8).pin_memory()
        init = N.RtsCounters()
        init.first_escaped = INT32_MAX
        self.template = torch.frombuffer(bytearray(bytes(init)), dtype=torch.uint8).pin_memory()

    def reset(self, stream) -> None:
        with torch.cuda.stream(stream):
            self.dev.copy_(self.template, non_blocking=True)

    def read(self, stream) -> N.RtsCounters:
        with torch.cuda.stream(stream):
            self.host.copy_(self.dev, non_blocking=True)
        stream.synchronize()
        return N.RtsCounters.from_buffer_copy(self.host.numpy().tobytes())


def raise_on_errors(c: N.RtsCounters, width: int = 128) -> None:
    """Turn device error bits into the reference's exceptions and messages
    (grid.py:268-273, grid.py:327-331, wcsph.py:286-287)."""
    f = c.err_flags
    if f & N.ERR_ESCAPED:
        raise NumericalError(
            f"{int(c.n_escaped)} fluid particle(s) left the simulation domain "
            f"(first index {int(c.first_escaped)})")
    if f & N.ERR_OVERFLOW:
        raise NumericalError(
            f"neighbor table overflow: {int(c.overflow)} entries dropped "
            f"(table width {width}); the particle distribution has collapsed")
    if f & N.ERR_NONFINITE:
        raise NumericalError("non-finite density; the simulation has blown up")
    if f & N.ERR_CHECK:
        raise N.NativeError(f"device bounds check failed at site {int(c.check_site)} "
                            "(checked build)")


class PhaseTimer:
    """CUDA-event time per bucket (neighbor / physics / rts), read after the
    end-of-step synchronisation so timing never adds a sync of its own."""

    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self._marks: list = []

    def start(self, stream):
        self._marks = []
        self._last = self._event(stream)

    def _event(self, stream):
        if not self.enabled:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def mark(self, bucket: str, stream):
        if not self.enabled:
            return
        e = self._event(stream)
        self._marks.append((bucket, self._last, e))
        self._last = e

    def totals(self) -> dict:
        out = {"neighbor": 0.0, "physics": 0.0, "rts": 0.0}
        for bucket, a, b in self._marks:
            out[bucket] += a.elapsed_time(b) * 1e-3
        return out


def as_device_f32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float32).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device=device).contiguous()
