"""Desk-scale acceptance runs of the reference (tests/test_acceptance.py C3,
C6, C7, C9, C10, C11) on the B200 solvers: prints the measured numbers."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from pathlib import Path
from paper_2009_14514_b200 import preset_scene
from paper_2009_14514_b200.run import run_simulation, compare
from paper_2009_14514_b200.stats import read_stats

out = Path(tempfile.mkdtemp())
t0 = time.time()
ddb = preset_scene("double_dam_break")
m = {}
for name in ("pcisph-const", "pcisph-rts"):
    m[name] = run_simulation(ddb, name, 1.0, 30, out / f"ddb_{name}")
rep = compare(out / "ddb_pcisph-const", out / "ddb_pcisph-rts")
print("C6 work ratio", rep["work_ratio"], "speedup", rep["speedup"],
      "walls", m["pcisph-const"]["wall_time"], m["pcisph-rts"]["wall_time"], time.time() - t0)
for name in ("wcsph", "wcsph-rts"):
    m[name] = run_simulation(ddb, name, 0.4, 30, out / f"ddb_{name}")
print("C7 wall ratio", m["wcsph-rts"]["wall_time"] / m["wcsph"]["wall_time"], time.time() - t0)
for n in ("pcisph-rts", "wcsph-rts"):
    print("C9", n, m[n]["t_rts"] / m[n]["wall_time"])
dam = preset_scene("dam_break")
md = run_simulation(dam, "pcisph-rts", 2.0, 30, out / "dam_pcisph-rts",
                    solver_kwargs={"audit_neighbors": True})
rows = [r for r in read_stats(out / "dam_pcisph-rts" / "stats.csv") if r.time <= 1.0 + 1e-9]
print("C3", len(rows), max(r.max_err for r in rows), max(r.avg_err for r in rows),
      dam.eta_max, dam.eta_avg, "missed", md["missed_neighbors"], time.time() - t0)
mw = run_simulation(dam, "wcsph-rts", 2.0, 30, out / "dam_wcsph-rts",
                    solver_kwargs={"audit_neighbors": True})
print("C11 wcsph missed", mw["missed_neighbors"], time.time() - t0)
var = {}
for tag, corr in (("corr", True), ("uncorr", False)):
    run_simulation(ddb, "wcsph-rts", 0.3, 30, out / f"var_{tag}",
                   solver_kwargs={"track_rho_variance": True, "apply_correction": corr,
                                  "audit_neighbors": True})
    var[tag] = read_stats(out / f"var_{tag}" / "stats.csv")
n = min(len(var["corr"]), len(var["uncorr"]))
vc = np.array([r.rho_var for r in var["corr"][:n]]); vu = np.array([r.rho_var for r in var["uncorr"][:n]])
print("C10", n, float(np.mean(vu > vc)), vu.mean(), vc.mean(), time.time() - t0)
