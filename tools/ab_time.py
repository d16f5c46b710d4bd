"""A/B timing of runtime knobs (environment variables read by libeg_b200 at
each eg_compute) on one resident workload, one process:

    python tools/ab_time.py --config C3 --variants '{}' '{"EG_PERSIST": "0"}'

Prints one JSON line per variant: ms/step (CUDA events, 7 steps after 3
warm-ups), the main kernel's us (eg_stats.us_main) and the graph counts.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--repeat", type=int, default=2, help="passes over the variant list")
    ap.add_argument("--variants", nargs="+", default=["{}"])
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import paper_2303_02724_b200 as eg
    torch.cuda.set_device(0)
    f, dims, csr = bench.make_input(a.config, "cuda:0")
    kw = dict(dims=dims) if dims is not None else dict(csr=csr)
    ctx = eg.Context(0)
    ref = None
    for rep in range(a.repeat):
        for v in a.variants:
            env = json.loads(v)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            for _ in range(a.warmup):
                g = ctx.compute(f, flags=eg.EG_CHECK_NAN, materialize=False, **kw)
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            us = []
            e0.record(st)
            for _ in range(a.steps):
                ctx.compute(f, flags=eg.EG_CHECK_NAN, materialize=False, **kw)
                us.append(ctx.stats())
            e1.record(st)
            torch.cuda.synchronize()
            g = ctx.graph()
            lab = g.labels
            h = int(torch.sum(lab.to(torch.int64) * 2654435761 % 1000003).item())
            key = (len(g.maxima), len(g.saddles), len(g.arcs), h)
            if ref is None:
                ref = key
            row = {"variant": env, "rep": rep, "ms": round(e0.elapsed_time(e1) / a.steps, 4),
                   "us_main": round(float(np.mean([s["us_main"] for s in us])), 1),
                   "phases": {k: round(float(np.mean([s[k] for s in us])), 1)
                              for k in ("us_classify", "us_boundary", "us_arcs", "us_graph", "us_total")},
                   "counts": key[:3], "same_as_first": key == ref}
            print(json.dumps(row), flush=True)
            for k, x in old.items():
                if x is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = x


if __name__ == "__main__":
    main()
