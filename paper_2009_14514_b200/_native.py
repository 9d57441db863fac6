"""ctypes binding of ``librtssph.so`` (C ABI in ``include/rts_sph.h``).

The library is the only compute path of this package: if it is missing or
there is no CUDA device, constructing a solver raises -- there is no CPU
fallback.  Structures mirror the header field for field.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtssph.so")
ABI_VERSION = 28

_c = ctypes
_D = _c.c_double
_I = _c.c_int32
_P = _c.c_void_p


class RtsParams(_c.Structure):
    _fields_ = [
        ("origin", _D * 3), ("grid_hi", _D * 3), ("block_size", _D), ("inv_block", _D),
        ("h", _D), ("h2", _D), ("c_poly6", _D), ("c_spiky", _D), ("c_visc", _D),
        ("mass", _D), ("inv_mass", _D), ("rho0", _D), ("b_stiff", _D), ("mu", _D),
        ("clamp_lo", _D * 3), ("clamp_hi", _D * 3), ("gravity", _D * 3), ("dt", _D),
        ("dt_base", _D), ("lambda_v", _D), ("lambda_f", _D), ("sound_speed", _D), ("alpha", _D),
        ("betas", _D * 8), ("eta_max", _D), ("eta_avg", _D), ("rho_T", _D), ("delta", _D),
        ("dims", _I * 3), ("n_cells", _I), ("n_fluid", _I), ("n_bound", _I), ("n_bcells", _I),
        ("width", _I), ("n_max", _I), ("use_sound", _I), ("pin_region", _I),
        ("apply_correction", _I), ("rts", _I), ("n_sms", _I), ("n_regions", _I), ("n_global", _I), ("nbr_stride", _I), ("n_ghost", _I),
    ]


class RtsCounters(_c.Structure):
    _fields_ = [
        ("err_flags", _c.c_uint32), ("n_escaped", _I), ("first_escaped", _I), ("n_compute", _I),
        ("overflow", _c.c_int64), ("n_sorted", _I), ("n_pred", _I), ("n_force", _I),
        ("n_list", _I), ("fmax_bits", _c.c_uint64), ("sum_rho", _D), ("max_err", _D),
        ("any_se", _I), ("lists_all", _I), ("missing", _c.c_int64),
        ("blocks_done", _c.c_uint32), ("check_site", _I), ("stamps", _c.c_int64 * 4),
        ("disp_cur", _c.c_float), ("disp_total", _c.c_float), ("soa_fresh", _c.c_int32), ("reserved1", _c.c_int32),
    ]


class RtsMinorStats(_c.Structure):
    _fields_ = [
        ("iterations", _I), ("n_refresh", _I), ("early", _I), ("riters", _I * 5),
        ("corrected", _c.c_int64), ("forced", _c.c_int64), ("max_err", _D), ("avg_err", _D),
        ("t_begin", _c.c_int64), ("t_refreshed", _c.c_int64), ("t_looped", _c.c_int64),
        ("t_end", _c.c_int64),
    ]


MAX_MINOR = 8
MAX_ROWS = 8


class RtsControl(_c.Structure):
    _fields_ = [
        ("it", _I), ("g_count", _I), ("local_active", _I), ("local_banned", _I),
        ("local_run", _I), ("early", _I), ("done", _I), ("failed", _I), ("motion_all", _I),
        ("row_mask", _I), ("snap_op", _I), ("minor", _I), ("stop_major", _I),
        ("local_entered", _I), ("local_reverted", _I), ("fail_kind", _I), ("fail_g", _I),
        ("stamp", _I), ("prev_force", _I),
        ("n_rows", _I * MAX_MINOR), ("row_masks", (_I * MAX_ROWS) * MAX_MINOR),
        ("row_counts", (_I * MAX_ROWS) * MAX_MINOR), ("riters", _I * 5), ("skipped", _I),
        ("corrected", _c.c_int64), ("forced", _c.c_int64), ("last_max_err", _D),
        ("last_avg_err", _D), ("fail_err", _D),
        ("stats", RtsMinorStats * MAX_MINOR),
    ]


BUFFER_FIELDS = (
    "pos", "vel", "acc", "acc_prev", "force", "f_p", "rho", "pres", "err", "xstar", "dt_since",
    "dt_corr", "validity", "region", "compute", "in_se", "in_sob", "fluid_cells", "cell_count",
    "cell_bcount", "starts", "order", "fill", "scan_tmp", "bcell_ids", "bcell_start", "bidx",
    "bcell_of", "bcell_active", "vmax", "fmax", "block_raw", "block_field", "block_tmp",
    "block_flag", "cpos", "cvel", "cterm", "cwall", "cx", "cy", "cz", "active", "list2", "list3", "nbr", "cnt", "xs", "pflag", "partial",
    "snap_p", "snap_fp", "slot_of", "ctl", "se_stamp", "near_stamp", "ghost", "sort_key", "ctr",
)


class RtsBuffers(_c.Structure):
    _fields_ = [(name, _P) for name in BUFFER_FIELDS]


HALO_MAX_FIELDS = 16
CTL_WORDS = 5  # RTS_CTL_WORDS: rts_ctl_publish row (fp64 words)


class RtsHaloField(_c.Structure):
    _fields_ = [("ptr", _P), ("remap", _P), ("words", _I), ("stride", _I), ("msg_off", _I),
                ("esize", _I)]


class RtsSlabGeom(_c.Structure):
    _fields_ = [("origin_x", _D), ("inv_block", _D), ("nx", _I), ("lo", _I), ("hi", _I),
                ("halo", _I), ("has_left", _I), ("has_right", _I), ("left_lo", _I),
                ("right_hi", _I)]


class RtsHaloSpec(_c.Structure):
    _fields_ = [("n_fields", _I), ("row_words", _I), ("msg_words", _I), ("pad", _I),
                ("f", RtsHaloField * HALO_MAX_FIELDS)]


ERR_ESCAPED, ERR_OVERFLOW, ERR_NONFINITE, ERR_ITERCAP, ERR_CHECK = 0x1, 0x2, 0x4, 0x8, 0x10

# entry points: name -> argtypes (all return int)
_PP = _c.POINTER(RtsParams)
_PB = _c.POINTER(RtsBuffers)
SIGNATURES = {
    "rts_abi_version": [],
    "rts_device_sms": [],
    "rts_memset": [_P, _c.c_int, _c.c_int64, _P],
    "rts_grid_keys": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_grid_sort": [_PP, _PB, _P],
    "rts_block_maxima": [_PP, _PB, _c.c_int, _P],
    "rts_force_max": [_PP, _PB, _P],
    "rts_block_levels": [_PP, _PB, _c.c_int, _P],
    "rts_wcsph_propagate": [_PP, _PB, _P],
    "rts_pci_walls": [_PP, _PB, _P],
    "rts_pci_gather": [_PP, _PB, _P],
    "rts_pci_major_particles": [_PP, _PB, _P],
    "rts_pci_refresh": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_pci_motion": [_PP, _PB, _c.c_int, _P],
    "rts_pci_sets": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_pci_density": [_PP, _PB, _P],
    "rts_pci_se_reduce": [_PP, _PB, _c.c_int, _P],
    "rts_pci_observed": [_PP, _PB, _c.c_int, _P],
    "rts_pci_sob": [_PP, _PB, _P],
    "rts_pci_pforces": [_PP, _PB, _P],
    "rts_pci_integrate": [_PP, _PB, _c.c_int, _P],
    "rts_pci_mark_updates": [_PP, _PB, _P],
    "rts_pci_snapshot": [_PP, _PB, _c.c_int, _P],
    "rts_vel_max": [_PP, _PB, _P],
    "rts_counters_reset": [_PB, _P],
    "rts_stamp": [_PB, _c.c_int, _P],
    "rts_region_op": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_grid_search": [_PP, _PB, _P, _c.c_int, _P],
    "rts_pci_zero_pressure": [_PP, _PB, _P],
    "rts_pci_major_begin": [_PP, _PB, _P],
    "rts_pci_minor_begin": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_pci_minor_end": [_PP, _PB, _c.c_int, _P],
    "rts_pci_iteration": [_PP, _PB, _c.c_int, _c.c_ulonglong, _c.c_int, _c.c_int, _P],
    "rts_pci_control": [_PP, _PB, _c.c_int, _c.c_ulonglong, _c.c_int, _c.c_int, _P],
    "rts_pci_minor_head": [_PP, _PB, _c.c_int, _P],
    "rts_pci_minor_tail": [_PP, _PB, _c.c_int, _c.c_int, _P],
    "rts_graph_launch": [_P, _P],
    "rts_pci_audit": [_PP, _PB, _PB, _P],
    "rts_wcsph_density": [_PP, _PB, _P],
    "rts_wcsph_forces": [_PP, _PB, _P],
    "rts_wcsph_integrate": [_PP, _PB, _P],
    "rts_halo_pack": [_c.POINTER(RtsHaloSpec), _P, _c.c_int64, _P, _P],
    "rts_halo_unpack": [_c.POINTER(RtsHaloSpec), _P, _c.c_int64, _P, _P],
    "rts_ctl_publish": [_PB, _P, _P],
    "rts_rho_variance": [_PP, _PB, _P, _P],
    "rts_slab_classify": [_c.POINTER(RtsSlabGeom), _P, _c.c_int, _P, _c.c_int64, _P, _P, _P],
    "rts_slab_holes": [_P, _c.c_int, _c.c_int, _c.c_int, _P, _P, _P, _P],
    "rts_ctl_fold": [_PB, _P, _c.c_int, _P],
}

_lib = None


class NativeError(RuntimeError):
    pass


def load(path: str | None = None):
    """Load the library (no CUDA call is made); raises if it is missing.
    ``RTS_SPH_LIB`` selects another build of it (e.g. the bounds-checked
    ``-DRTS_CHECKED=1`` variant, scripts/checked_build.sh)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("RTS_SPH_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise NativeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = _c.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _c.c_int
    lib.rts_launch_count.argtypes = []
    lib.rts_launch_count.restype = _c.c_longlong
    lib.rts_pci_graph_create.argtypes = [_PP, _PB, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                         _c.POINTER(_c.c_int)]
    lib.rts_pci_graph_create.restype = _c.c_void_p
    lib.rts_wcsph_graph_create.argtypes = [_PP, _PB, _c.POINTER(_c.c_int)]
    lib.rts_wcsph_graph_create.restype = _c.c_void_p
    lib.rts_graph_kernel_counts.argtypes = [_P, _c.POINTER(_c.c_longlong), _c.POINTER(_c.c_longlong)]
    lib.rts_graph_kernel_counts.restype = _c.c_int
    lib.rts_graph_destroy.argtypes = [_P]
    lib.rts_graph_destroy.restype = None
    if lib.rts_abi_version() != ABI_VERSION:
        raise NativeError(f"librtssph ABI {lib.rts_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


_graph_launched = 0  # kernels executed inside graph launches (counted by the host)


def launch_count() -> int:
    """librtssph kernels launched directly plus those executed by graphs."""
    return int(load().rts_launch_count()) + _graph_launched


def graph_kernel_counts(graph) -> tuple[int, int]:
    a, b = _c.c_longlong(0), _c.c_longlong(0)
    load().rts_graph_kernel_counts(graph, _c.byref(a), _c.byref(b))
    return int(a.value), int(b.value)


def note_graph_kernels(n: int) -> None:
    global _graph_launched
    _graph_launched += int(n)


_fns: dict = {}


def call(name: str, *args) -> None:
    f = _fns.get(name)
    if f is None:
        f = _fns[name] = getattr(load(), name)
    rc = f(*args)
    if rc != 0:
        raise NativeError(f"{name} failed with cudaError {rc}")
