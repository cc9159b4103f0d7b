"""Basic-block view of an ncu source-page CSV (one kernel): runs of consecutive SASS lines with
the same execution count, their size, warp instructions executed and stall samples.
    python tools/ncu_blocks.py DUMP.csv [min_share_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    lines.append((int(r[0], 16), r[1].strip(), float(r[hdr.index("Instructions Executed")] or 0),
                  float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
base = lines[0][0]
tot = sum(l[2] for l in lines) or 1
tots = sum(l[3] for l in lines) or 1
blocks = []
cur = None
for a, s, ie, ws in lines:
    if cur and abs(ie - cur[2]) <= 0.01 * max(ie, 1) and not cur[5]:
        cur[1] = a
        cur[3] += ie
        cur[4] += ws
        cur[6] += 1
    else:
        if cur:
            blocks.append(cur)
        cur = [a, a, ie, ie, ws, False, 1]
    if s.split()[0].startswith(("BRA", "@")) and "BRA" in s:
        cur[5] = True
blocks.append(cur)
print(f"{'start':>7} {'end':>7} {'n':>4} {'exec/inst':>10} {'inst%':>6} {'stall%':>6}")
for b0, b1, ie, sie, ws, _, n in blocks:
    if sie / tot * 100 >= minp or ws / tots * 100 >= minp:
        print(f"{b0 - base:7x} {b1 - base:7x} {n:4d} {ie / 1e6:9.3f}M {sie / tot * 100:6.1f} {ws / tots * 100:6.1f}")
