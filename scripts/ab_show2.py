"""Summarise scripts/gpu_ab.sh logs: python scripts/ab_show2.py TAG"""
import collections
import glob
import json
import re
import sys

res = collections.defaultdict(list)
kern = collections.defaultdict(lambda: collections.defaultdict(list))
for path in sorted(glob.glob(f"gpurun_out/ab_{sys.argv[1]}_*.log")):
    m = re.match(rf"gpurun_out/ab_{sys.argv[1]}_(.+)_(cfg[^_]+)_(\d+)\.log", path)
    if not m:
        continue
    lib, wl, _ = m.groups()
    js = [l for l in open(path) if l.startswith("{")]
    if not js:
        res[(lib, wl)].append(None)
        continue
    d = json.loads(js[-1])
    res[(lib, wl)].append(d["ms_per_step"])
    for k, v in d["roofline"]["kernels"].items():
        kern[(lib, wl)][k].append(v["s"] * 1e6 / v["launches"])
for (lib, wl), v in sorted(res.items(), key=lambda x: (x[0][1], x[0][0])):
    ks = {k.replace("rts_", ""): round(sum(x) / len(x), 1) for k, x in kern[(lib, wl)].items()}
    print(f"{wl:12s} {lib:14s} ms/step {v}  {ks}")
