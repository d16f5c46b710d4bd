#!/usr/bin/env python
"""the paper's GPU resolution sweep: the 3-D
Schwefel function resampled at 128^3 .. 1024^3, one bench.py run per size.
Each line is checked against the separable product rule (maxima = M^3,
2-saddles = 3 S M^2 with M / S the 1-D maxima / interior minima of the
sampled profile, SoS order) and bench.py's sampled oracle parity.
usage (GPU box): python tools/sweep_f1.py [out.json]"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import eg_inputs as G  # noqa: E402


def product_rule(n: int):
    h = -G.schwefel_profile(n).astype(np.float64)      # g = const - sum t(x_i): maximise -t
    M = S = 0
    for k in range(n):                                  # SoS: a later index is higher on ties
        up_left = k == 0 or h[k] >= h[k - 1]
        up_right = k == n - 1 or h[k] > h[k + 1]
        M += up_left and up_right
        if 0 < k < n - 1 and h[k] < h[k - 1] and h[k] <= h[k + 1]:
            S += 1
    return int(M) ** 3, 3 * int(S) * int(M) * int(M)


rows = []
for n in (128, 256, 512, 1024):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", f"F1-{n}", "--steps", "10",
                          "--warmup", "3", "--no-cpu", "--no-e2e"], capture_output=True, text=True, timeout=900)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    em, es = product_rule(n)
    row = dict(n=n, vertices=n ** 3, ms_per_step=d["ms_per_step"], mvert_s=d["value"],
               main_us=d["phases_us"]["main"], roofline_frac=d["roofline"]["frac"], maxima=d["graph"]["maxima"],
               saddles=d["graph"]["saddles"], arcs=d["graph"]["arcs"], expected_maxima=em, expected_saddles=es,
               closed_form_match=(d["graph"]["maxima"] == em and d["graph"]["saddles"] == es),
               parity_sample=d["parity_sample"], clocks=d["clocks"])
    rows.append(row)
    print(json.dumps(row), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
