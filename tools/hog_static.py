"""Static size of k_hog3<F64, vec>'s row loop: the instructions of the largest branch-free
block plus the loop tail, from a compiled object (experiment bookkeeping before GPU time).
    python tools/hog_static.py build/bl_hog.o"""
import collections
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "build/bl_hog.o"
fn = "_ZN3blb6k_hog3ILi1ELb1EEEvPKNS_8PlanDescENS_9HogLaunchEPKvPdS7_"
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# basic blocks split at branches and branch targets
targets = set()
for a, s in ins:
    m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", s)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, s in ins:
    if a in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append((a, s))
    if "BRA" in s or "EXIT" in s:
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
big = max(blocks, key=len)
c = collections.Counter()
for a, s in big:
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    c[op.split(".")[0]] += 1
print(f"largest block {len(big)} instructions at {big[0][0]:#x}")
print(" ".join(f"{k}:{v}" for k, v in c.most_common(24)))
