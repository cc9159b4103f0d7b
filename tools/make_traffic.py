"""profiles/traffic.json from an ncu launch list with dram bytes (tools/ncu_all.sh):
per-stage DRAM read+write bytes per frame.
    python tools/make_traffic.py LAUNCHES.csv FRAMES_PROCESSED SOURCE_TAG"""
import collections
import csv
import json
import os
import sys

STAGE = [("k_resample", "pyramid"), ("k_hog", "gradhist"), ("k_features", "features"), ("k_screen", "screen"),
         ("k_rescore", "rescore"), ("k_nms", "nms"), ("k_flatten", "nms"), ("k_ert", "ert")]
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = collections.Counter()
for r in rows[1:]:
    if r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    name = r[ki].replace("void ", "")
    st = next((s for k, s in STAGE if name.startswith(k) or ("blb::" + k) in name or k in name.split("(")[0]), None)
    if st:
        tot[st] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
frames = float(sys.argv[2])
out = {"bytes_per_frame": {k: round(v / frames, 1) for k, v in tot.items()},
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, {sys.argv[3]}, {int(frames)} frames"}
json.dump(out, open(os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
