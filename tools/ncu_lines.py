"""Per-source-line hot spots of one kernel in an .ncu-rep (cuda+sass source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
fname, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    out.append((s, ie, fname, r[0], r[1][:90]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("samples", tot, "warp-inst", ti)
for o in sorted(out, reverse=True)[:top]:
    print("%5.1f%% samp %5.1f%% inst  %s:%s  %s" % (100 * o[0] / tot, 100 * o[1] / ti, o[2], o[3], o[4].strip()))
