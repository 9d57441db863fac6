"""pytest plugin: make ``import rts_sph`` resolve to this package, so the
reference's own host-side test files can run against the drop-in
(tests/test_reference_suite_cpu.py).  Nothing here is reference code."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2009_14514_b200 as pkg  # noqa: E402

sys.modules["rts_sph"] = pkg
for sub in ("scene", "stats", "errors", "kernels", "run", "cli", "bench_api", "regions"):
    sys.modules[f"rts_sph.{sub}"] = __import__(f"paper_2009_14514_b200.{sub}", fromlist=["_"])
sys.modules["rts_sph.bench"] = sys.modules["rts_sph.run"]
