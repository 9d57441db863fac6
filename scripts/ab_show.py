"""Summarise scripts/ab_env.sh logs: python scripts/ab_show.py TAG"""
import glob
import json
import sys

for path in sorted(glob.glob(f"gpurun_out/ab_{sys.argv[1]}_*.log")):
    lines = open(path).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    cfg = [l for l in lines if l.startswith("exit")]
    if not js:
        print(path, cfg, lines[-5:])
        continue
    d = json.loads(js[-1])
    ks = {k: round(v["s"] * 1e6 / v["launches"], 1) for k, v in d["roofline"]["kernels"].items()}
    w = (d.get("wcsph_rts_1m") or {}).get("ms_per_step")
    print(cfg, f"{d['value']:.3e}", round(d["ms_per_step"], 3), "wcsph", w and round(w, 3))
    print("   us/launch", ks)
