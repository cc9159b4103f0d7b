"""Opcode histogram of SASS lines 'ADDR OPCODE ...' within address ranges.
    python tools/sass_hist.py FILE 0x1160-0x37f0 0x5350-0x56c0"""
import collections
import sys

rng = [tuple(int(x, 16) for x in a.split("-")) for a in sys.argv[2:]]
c = collections.Counter()
for line in open(sys.argv[1]):
    t = line.split()
    if len(t) < 2:
        continue
    a = int(t[0], 16)
    if rng and not any(lo <= a < hi for lo, hi in rng):
        continue
    op = t[2] if t[1].startswith("@") else t[1]
    c[op.split(".")[0].rstrip(";")] += 1
n = sum(c.values())
print(n, "instructions")
for k, v in c.most_common(40):
    print(f"{v:5d} {k}")
