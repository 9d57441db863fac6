"""Import the reference package ``rts_sph`` from /root/reference for fixture
generation (this container only; /root/reference does not exist on the GPU
box).  numba 0.65's parfor pass recurses forever on two reference kernels
(SURVEY.md section 0.3), so those two are re-jitted serially from their
Python source -- same per-row arithmetic, no reference file is modified."""

import os
import sys

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "rts_sph"))


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_rts")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from numba import njit

    import rts_sph
    import rts_sph.grid as g

    for name in ("_search_neighbors", "_count_missing"):
        fn = getattr(g, name)
        if hasattr(fn, "py_func"):
            setattr(g, name, njit(cache=False, parallel=False)(fn.py_func))
    return rts_sph
