"""Per-launch key metrics from an ncu --set full report (details page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "Executed Ipc Active",
        "Grid Size"]
rows = {}
for row in r[1:]:
    if row[mi] in want:
        key = (int(row[ii]), row[ki].split("(")[0].split("::")[-1])
        rows.setdefault(key, {})[row[mi]] = (row[vi] + " " + row[ui]).strip()
for (i, k), d in sorted(rows.items()):
    print(f"{i:3d} {k:16s} " + " | ".join(f"{m.split()[0][:8]}={d.get(m, '-')}" for m in want))
