"""Top SASS instructions by warp-stall samples per kernel from `ncu --page source --csv`."""
import csv, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
secs = []; cur = None; hdr = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "ins": []}; secs.append(cur); continue
    if r and r[0] == "Address":
        hdr = r; continue
    if cur is not None and hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); cur["ins"].append(d)
seen = set()
for s in secs:
    if s["name"] in seen: continue
    seen.add(s["name"])
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in s["ins"])
    print("==", s["name"], "samples", tot, "instructions", len(s["ins"]))
    top = sorted(s["ins"], key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:topn]
    for d in top:
        n = int(d["Warp Stall Sampling (All Samples)"] or 0)
        print(f"  {100*n/max(tot,1):5.1f}%  {d['Source'].strip()[:90]}")
