"""C6 at desk scale: per-call wall time of RTS-PCISPH majors vs constant-step
PCISPH steps on the double dam break, and the kernels each graph holds."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2009_14514_b200 import preset_scene, make_solver
from paper_2009_14514_b200 import _native as N

sc = preset_scene("double_dam_break")
res = {}
for name in ("pcisph-const", "pcisph-rts"):
    s = make_solver(sc, name, device="cuda")
    for _ in range(20):
        s.advance()
    torch.cuda.synchronize()
    k0 = N.launch_count()
    rows = []
    n = 0
    dt = 0.0
    win, wt, wit = [], 0.0, 0
    edge = 0.25
    while s.sim_time < 1.0:
        t0 = time.perf_counter()
        r = s.advance()
        dt1 = time.perf_counter() - t0
        rows += r
        dt += dt1
        wt += dt1
        wit += sum(x.iterations for x in r)
        n += 1
        if s.sim_time >= edge - 1e-9:
            win.append((round(wt * 1e3, 1), wit))
            wt, wit, edge = 0.0, 0, edge + 0.25
    print(name, "per 0.25 s window (ms, iterations):", win)
    kl = N.launch_count() - k0
    it = sum(r.iterations for r in rows)
    res[name] = dt
    print(f"{name}: {n} calls, {len(rows)} steps, {dt*1e3:.1f} ms, {dt/n*1e6:.1f} us/call, "
          f"{dt/len(rows)*1e6:.1f} us/step, iterations {it} ({dt/it*1e6:.1f} us/iter), "
          f"kernels {kl} ({kl/len(rows):.1f}/step), n_fluid {s.n_fluid}")
print("speedup (same simulated time)", res["pcisph-const"] / res["pcisph-rts"])
