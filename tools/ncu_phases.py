"""Per-line and per-phase stall breakdown of one kernel in an .ncu-rep.

usage: python tools/ncu_phases.py REP FUNCTION-SUBSTRING [phase=a-b ...] [--top N]
Prints the top lines by samples with their three largest stall reasons, then
totals per named line range (phase)."""
import csv
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
phases = []
for a in sys.argv[3:]:
    if "=" in a:
        name, rng = a.split("=")
        lo, hi = rng.split("-")
        phases.append((name, int(lo), int(hi)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
func, fname, hdr, lines, seen = None, None, None, [], set()
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
    if hdr is None or len(r) < 8 or r[2] != "-" or func is None or want not in func:
        continue
    key = (func, fname, r[0])
    if key in seen:
        continue
    seen.add(key)
    st = {h[6:]: float(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    lines.append((float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0),
                  float(r[hdr.index("Instructions Executed")] or 0), fname, int(r[0]), r[1][:70], st))
tot = sum(l[0] for l in lines) or 1
ti = sum(l[1] for l in lines) or 1
print(f"samples {tot:.0f}  warp-inst {ti:.0f}")
for s, ie, fn, ln, src, st in sorted(lines, key=lambda l: -l[0])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print("%5.1f%% samp %5.1f%% inst %s:%d %-50s %s" % (100 * s / tot, 100 * ie / ti, fn, ln, src.strip()[:50],
          " ".join(f"{k}={100 * v / max(s, 1):.0f}%" for k, v in big)))
if phases:
    print("\nphase            samples   inst   top stalls")
    for name, lo, hi in phases:
        sel = [l for l in lines if l[2].startswith("k_grid3d") and lo <= l[3] <= hi]
        s = sum(l[0] for l in sel)
        i = sum(l[1] for l in sel)
        agg = {}
        for l in sel:
            for k, v in l[5].items():
                agg[k] = agg.get(k, 0) + v
        big = sorted(agg.items(), key=lambda kv: -kv[1])[:4]
        print("%-14s %6.1f%% %6.1f%%   %s" % (name, 100 * s / tot, 100 * i / ti,
              " ".join(f"{k}={100 * v / max(s, 1):.0f}%" for k, v in big)))
