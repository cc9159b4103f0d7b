"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump per CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
agg = {}
cur_file = ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue  # keep only the per-line summary rows (no SASS address)
    key = (cur_file, r[0], r[1].strip()[:100])
    ws = float(r[4] or 0)
    ie = float(r[7] or 0)
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += ws
    a[1] += ie
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for (f, ln, src), (ws, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ws / tw * 100:5.1f}% stall {ie / ti * 100:5.1f}% inst  {f}:{ln}  {src}")
