"""Per-opcode totals from `ncu --page source --csv --print-source cuda,sass` (one kernel):
warp instructions executed, stall samples, and the top stall reasons.
    python tools/ncu_sass.py DUMP.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
inst = collections.Counter()
stall = collections.Counter()
reasons = collections.Counter()
seen = set()
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])
    op = r[3].strip().split()
    op = [t for t in op if not t.startswith("@")]
    name = op[0].split(".")[0] if op else "?"
    ie = float(r[hdr.index("Instructions Executed")] or 0)
    ws = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    inst[name] += ie
    stall[name] += ws
    for k, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                reasons[h] += float(r[k] or 0)
            except ValueError:
                pass
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print(f"total warp instructions {ti / 1e6:.1f} M")
for k, v in inst.most_common(top):
    print(f"  {k:12s} {v / 1e6:9.2f} M  {v / ti * 100:5.1f}% inst  {stall[k] / ts * 100:5.1f}% stall")
tr = sum(reasons.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {v / tr * 100:.0f}%" for k, v in reasons.most_common(8)))
