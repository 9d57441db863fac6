"""profiles/ncu_traffic.json from an ncu --csv capture of
dram__bytes_read.sum, dram__bytes_write.sum, lts__t_bytes.sum, gpu__time_duration.sum and
l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed: mean DRAM (and L2)
bytes per launch of each PCISPH entry point's main kernel, and the launch-time-weighted
utilisation of the L1 LSU data pipe (the bound of the gather kernels).
usage: python scripts/make_traffic.py gpurun_out/traffic_TAG.csv > profiles/ncu_traffic.json"""
import collections
import csv
import json
import sys

KERNELS = {"k_refresh": "rts_pci_refresh", "k_motion": "rts_pci_motion", "k_sets": "rts_pci_sets",
           "k_density": "rts_pci_density", "k_se_reduce": "rts_pci_se_reduce",
           "k_pforces": "rts_pci_pforces", "k_integrate": "rts_pci_integrate"}
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
per = collections.defaultdict(lambda: collections.defaultdict(float))
for d in data:
    name = d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].strip()
    if name not in KERNELS:
        continue
    per[(name, d["ID"])][d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
out = {"_how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,"
               "gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_"
               "elapsed --clock-control none on bench.py --steps 2 --warmup 1 "
               "(cfg2 1M); mean bytes per launch over all launches of the kernel (cold-cache, "
               "serialised)"}
agg = collections.defaultdict(list)
for (name, _), m in per.items():
    agg[name].append(m)
for name, ms in agg.items():
    e = KERNELS[name]
    out[e] = round(sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms) / len(ms))
    out[e + "_l2_bytes"] = round(sum(m["lts__t_bytes.sum"] for m in ms) / len(ms))
    out[e + "_launches"] = len(ms)
    w = [(m.get("gpu__time_duration.sum", 0.0),
          m.get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed")) for m in ms]
    w = [(t, x) for t, x in w if x is not None]
    if w and sum(t for t, _ in w) > 0:
        out[e + "_l1_wavefront_pct"] = round(sum(t * x for t, x in w) / sum(t for t, _ in w), 1)
print(json.dumps(out, indent=1))
