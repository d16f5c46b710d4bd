"""Per-source-line hot spots of one kernel in an .ncu-rep (cuda+sass source page).

usage: python tools/ncu_lines.py REP [TOP] [FUNCTION-SUBSTRING] [--by inst|samp]"""
import csv
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
by = "inst" if "--by" in sys.argv and sys.argv[sys.argv.index("--by") + 1] == "inst" else "samp"
args = [a for a in args if a not in ("inst", "samp")]
rep = args[0]
top = int(args[1]) if len(args) > 1 else 25
want = args[2] if len(args) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
fname, func, hdr, out, seen = None, None, None, [], set()
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    if want and (func is None or want not in func):
        continue
    key = (func, fname, r[0])
    if key in seen:  # the same function listed per profiled launch: keep the first
        continue
    seen.add(key)
    s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    out.append((s, ie, fname, r[0], r[1][:90]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("samples", tot, "warp-inst", ti)
key = (lambda o: -o[1]) if by == "inst" else (lambda o: -o[0])
for o in sorted(out, key=key)[:top]:
    print("%5.1f%% samp %5.1f%% inst  %s:%s  %s" % (100 * o[0] / tot, 100 * o[1] / ti, o[2], o[3], o[4].strip()))
