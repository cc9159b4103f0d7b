"""Per-opcode totals from `ncu --page source --csv --print-source sass` (one kernel): warp
instructions executed, stall samples and top stall reasons; with --ranges, per address range.
    python tools/ncu_sass.py DUMP.csv [top] [--dump]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
dump = "--dump" in sys.argv
hdr = None
inst = collections.Counter()
stall = collections.Counter()
reasons = collections.Counter()
lines = []
for r in rows:
    if r and r[0] in ("Address", "Line No"):
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    ai = hdr.index("Address")
    if not r[ai].startswith("0x"):
        continue
    op = r[hdr.index("Source")].strip().split()
    op = [t for t in op if not t.startswith("@")]
    name = op[0].split(".")[0] if op else "?"
    ie = float(r[hdr.index("Instructions Executed")] or 0)
    ws = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    inst[name] += ie
    stall[name] += ws
    rs = {}
    for k, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = float(r[k] or 0)
            except ValueError:
                continue
            reasons[h] += v
            rs[h[6:]] = v
    lines.append((r[ai], r[hdr.index("Source")].strip(), ie, ws, rs))
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print(f"total warp instructions {ti / 1e6:.1f} M, stall samples {ts:.0f}")
for k, v in inst.most_common(top):
    print(f"  {k:12s} {v / 1e6:9.2f} M  {v / ti * 100:5.1f}% inst  {stall[k] / ts * 100:5.1f}% stall")
tr = sum(reasons.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {v / tr * 100:.0f}%" for k, v in reasons.most_common(8)))
if dump:
    for a, s, ie, ws, rs in lines:
        top3 = ",".join(f"{k}:{v:.0f}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3] if v > 0)
        print(f"{a} {ie / 1e6:8.2f}M {ws:7.0f}  {s[:60]:60s} {top3}")
