"""Summarise an ncu --csv gpu__time_duration launch list: per-kernel totals and shares."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot = collections.defaultdict(float); cnt = collections.Counter(); units = set()
for d in data:
    if d['Metric Name'] != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0]; units.add(d['Metric Unit'])
    tot[name] += float(d['Metric Value'].replace(',', '')); cnt[name] += 1
T = sum(tot.values())
print(f"# unit {units}; total {T:.0f}")
print(f"{'kernel':60s} {'launches':>8s} {'total':>12s} {'share':>6s} {'avg':>10s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:12.0f} {100*v/T:5.1f}% {v/cnt[k]:10.0f}")
