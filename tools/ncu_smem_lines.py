"""Shared-memory wavefronts (and bank-conflict excess) per CUDA source line of
one kernel in an .ncu-rep (source page, cuda+sass).

usage: python tools/ncu_smem_lines.py REP FUNCTION-SUBSTRING [TOP]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
func, hdr = None, None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or func is None or want not in func:
        continue
    try:
        w = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
        x = float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
    except ValueError:
        continue
    if w == 0:
        continue
    key = r[0]
    agg[key][0] += w
    agg[key][1] += x
    agg[key][2] = r[1][:90]
tot = sum(v[0] for v in agg.values())
exc = sum(v[1] for v in agg.values())
print(f"shared wavefronts {tot:.4g}, excessive (bank conflicts) {exc:.4g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% wf  {v[1] / max(tot, 1) * 100:5.1f}% excess  line {k}: {v[2]}")
