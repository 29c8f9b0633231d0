"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    nm = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
    agg.setdefault(nm, []).append(v)
skip = [a for a in sys.argv[2:]]
tot = sum(sum(v) for k, v in agg.items() if not any(s in k for s in skip))
print(f"{'kernel':60s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    if any(s in k for s in skip):
        continue
    print(f"{k:60s} {len(v):5d} {sum(v)/len(v):10.1f} {sum(v):11.1f} {sum(v)/tot*100:5.1f}%")
