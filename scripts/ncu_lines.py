"""Warp-stall samples and executed warp instructions per CUDA source line of
one kernel, from `ncu -i REP --page source --csv --print-source sass,cuda`.

    python scripts/ncu_lines.py REP [kernel-substring] [top=30]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
path = fn = None
hdr = None
line = None
agg = defaultdict(lambda: [0, 0, 0])  # samples, warp instrs, thread instrs
src = {}
stalls = defaultdict(lambda: defaultdict(int))
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or (want and want not in (fn or "")):
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        line = (path, int(r[0]))
        src[line] = r[1].strip()
    if len(r) < 5 or not r[2]:
        continue
    d = {k: (v if v not in ("-", "") else "0") for k, v in zip(hdr[2:], r[2:])}
    try:
        n = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        wi = int(d.get("Instructions Executed") or 0)
        th = int(d.get("Thread Instructions Executed") or 0)
    except ValueError:  # a source row whose quoting ncu did not escape
        continue
    a = agg[line]
    a[0] += n
    a[1] += wi
    a[2] += th
    for k, v in d.items():
        if k.startswith("stall_") and v and v != "0":
            try:
                stalls[line][k] += int(float(v))
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot}, warp instructions {ti}")
for ln, (n, wi, th) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
    top = sorted(stalls[ln].items(), key=lambda kv: -kv[1])[:3]
    st = " ".join(f"{k[6:]}={v}" for k, v in top)
    print(f"{100 * n / tot:5.1f}% smp {100 * wi / ti:5.1f}% ins  eff {th / max(wi, 1):4.1f}  "
          f"{ln[0]}:{ln[1]:<5d} {src.get(ln, '')[:70]:70s} {st}")
