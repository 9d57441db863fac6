"""B200-native regional-time-stepping SPH (arXiv 2009.14514).

Drop-in for the hot path of the reference package ``rts_sph``: the same
public names (``Scene``, ``WcsphSolver``, ``PcisphSolver``, ``BlockGrid``,
``StepStats``, ``NumericalError`` ...), constructor arguments and step
semantics, with state held as fp32 CUDA tensors and every particle/block
pass executed by hand-written sm_100a kernels in ``librtssph.so``
(C ABI: ``include/rts_sph.h``).  There is no CPU fallback: constructing a
solver without the library or without a CUDA device raises.
"""

from .errors import ConfigError, NumericalError
from .kernels import KernelSet
from .scene import PRESET_NAMES, Scene, load_scene, parse_scene_text, preset_scene, seed_particles
from .stats import StepStats, read_stats, write_stats

__version__ = "0.1.0"


def __getattr__(name):
    # device-backed classes import torch lazily so the host-only parts of the
    # package (scene parsing, stats I/O) stay importable without CUDA
    if name in ("WcsphSolver", "tait_pressure", "NEIGHBOR_WIDTH"):
        from . import wcsph
        return getattr(wcsph, name)
    if name in ("PcisphSolver", "MajorStepController", "DEFAULT_SCHEDULE", "VALIDITY_PERIOD",
                "validate_schedule", "pci_delta"):
        from . import pcisph
        return getattr(pcisph, name)
    if name in ("BlockGrid",):
        from . import grid
        return grid.BlockGrid
    if name in ("make_solver", "SOLVER_NAMES"):
        from . import bench_api
        return getattr(bench_api, name)
    if name in ("run_simulation", "compare"):
        from . import run
        return getattr(run, name)
    if name in ("assign_regions", "smooth_regions", "expand_fast_regions", "derive_observed"):
        from . import regions
        return getattr(regions, name)
    raise AttributeError(name)


__all__ = [
    "BlockGrid", "ConfigError", "DEFAULT_SCHEDULE", "KernelSet", "MajorStepController",
    "NumericalError", "PRESET_NAMES", "PcisphSolver", "SOLVER_NAMES", "Scene", "StepStats",
    "WcsphSolver", "assign_regions", "compare", "derive_observed", "expand_fast_regions",
    "load_scene", "make_solver", "parse_scene_text", "pci_delta", "preset_scene", "read_stats",
    "run_simulation", "seed_particles", "smooth_regions", "tait_pressure", "validate_schedule",
    "write_stats", "__version__",
]
