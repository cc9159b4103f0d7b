#!/bin/bash
# Warm per-kernel GPU times of one C1 (and one C2) batch: ncu launch list with caches NOT flushed
# between kernels (--cache-control none), the last batch of a few.
for w in c1 c2; do
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv python tools/${w}_run.py 6 > gpurun_out/${w}_warm.csv 2>/dev/null
  python3 - "$w" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/{sys.argv[1]}_warm.csv")))
hdr = None; out = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr): out.append(dict(zip(hdr, r)))
ids = sorted(set(int(d["ID"]) for d in out))
tot = 0.0
for i in ids[-10:]:
    d = [x for x in out if int(x["ID"]) == i][0]
    us = float(d["Metric Value"]) / 1000.0
    tot += us
    print(f"{sys.argv[1]} {d['Kernel Name'][:40]:40s} {us:8.1f} us")
print(sys.argv[1], "sum", round(tot, 1), "us")
PY
done
