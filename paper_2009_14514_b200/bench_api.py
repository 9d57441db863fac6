"""Solver factory of the drop-in (``rts_sph.bench.make_solver``, bench.py:50-61)."""

from __future__ import annotations

from .errors import ConfigError

SOLVER_NAMES = ("wcsph", "wcsph-rts", "pcisph-const", "pcisph-adaptive", "pcisph-rts")


def make_solver(scene, name: str, **kwargs):
    from .pcisph import PcisphSolver
    from .wcsph import WcsphSolver

    table = {
        "wcsph": (WcsphSolver, "baseline"),
        "wcsph-rts": (WcsphSolver, "rts"),
        "pcisph-const": (PcisphSolver, "const"),
        "pcisph-adaptive": (PcisphSolver, "adaptive"),
        "pcisph-rts": (PcisphSolver, "rts"),
    }
    if name not in table:
        raise ConfigError(f"unknown solver {name!r}; expected one of {', '.join(SOLVER_NAMES)}")
    cls, mode = table[name]
    return cls(scene, mode=mode, **kwargs)
