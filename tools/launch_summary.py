"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[ki] == "Kernel Name" or (mi is not None and r[mi] != "gpu__time_duration.sum"):
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':34s} {'n':>4s} {'total_us':>10s} {'share':>6s} {'mean_us':>9s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:34s} {len(v):4d} {sum(v):10.1f} {sum(v) / tot * 100:5.1f}% {sum(v) / len(v):9.1f}")
