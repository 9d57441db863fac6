"""Small workload for compute-sanitizer (scripts/sanitize.sh): both solvers on
the tiny tank, graph and host-driven paths, the neighbour audit, and the
x-slab halo pack / unpack primitives.  Exits non-zero on any Python error."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from conftest import tiny_tank  # noqa: E402


def main(which):
    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    from paper_2009_14514_b200 import _native as N
    if which in ("all", "wcsph"):
        for mode in ("rts", "baseline"):
            s = WcsphSolver(tiny_tank(), mode=mode, track_rho_variance=True)
            for _ in range(3):
                s.step()
    if which in ("all", "pcisph"):
        for graphs in (False, True):
            s = PcisphSolver(tiny_tank(), mode="rts", use_graphs=graphs)
            s.advance()
            s.advance()
        s = PcisphSolver(tiny_tank(), mode="rts", audit_neighbors=True)
        s.advance()
        for mode in ("const", "adaptive"):
            s = PcisphSolver(tiny_tank(), mode=mode, use_graphs=False)
            s.advance()
    if which in ("all", "halo"):
        N.load()
        dev = torch.device("cuda:0")
        n = 4096
        pos = torch.randn(n, 3, device=dev)
        rows = torch.arange(0, n, 3, dtype=torch.int32, device=dev)
        s = N.RtsHaloSpec()
        s.n_fields, s.msg_words, s.row_words = 1, 3, 3
        s.f[0].ptr = pos.data_ptr()
        s.f[0].remap = None
        s.f[0].words, s.f[0].stride, s.f[0].msg_off = 3, 3, 0
        msg = torch.empty((rows.numel(), 3), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        N.call("rts_halo_pack", ctypes.byref(s), rows.data_ptr(), rows.numel(), msg.data_ptr(), st)
        pos2 = torch.zeros_like(pos)
        s.f[0].ptr = pos2.data_ptr()
        N.call("rts_halo_unpack", ctypes.byref(s), rows.data_ptr(), rows.numel(), msg.data_ptr(),
               st)
        torch.cuda.synchronize()
        assert torch.equal(pos2[rows.long()], pos[rows.long()])
    torch.cuda.synchronize()
    print("sanitize drive ok", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
