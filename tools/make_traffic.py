"""Write profiles/traffic.json from an `ncu --set full` raw CSV export:
DRAM bytes (read + write) per launch of the main per-vertex kernel(s) of a
config, summed over the kernels that make up one main phase (e.g. the interior
and edge-tile variants of k_tile).

usage: python tools/make_traffic.py <ncu raw csv> <config> <kernel-regex>
"""
import csv
import json
import os
import re
import sys

raw, cfg, pat = sys.argv[1], sys.argv[2], re.compile(sys.argv[3])
rows = list(csv.reader(open(raw)))
h, units = rows[0], rows[1]
ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per_kernel = {}
for r in rows[2:]:
    name = r[ki].split("(")[0]
    if not pat.search(name):
        continue
    b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
    per_kernel.setdefault(name, b)           # first launch of each kernel
total = int(sum(per_kernel.values()))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[cfg] = total
data.setdefault("_source", {})[cfg] = {"ncu_raw": os.path.basename(raw), "kernels": per_kernel}
json.dump(data, open(path, "w"), indent=1)
print(cfg, total, per_kernel)
