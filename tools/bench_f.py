#!/usr/bin/env python
"""SURVEY 8(f) rows f2-f4 measured on the BASELINE workloads: the device time
of one eg_compute (CUDA events, steps after warm-ups, graph left in HBM as in
bench.py) for every flag combination the rows add, next to the plain maximum
graph of the same field, plus the host time of eg_simplify (f4) and the typed
inputs of f3.  Each variant's counts are printed; every variant is also
checked against the oracle in tests/test_gpu_parity.py (small fields).

usage (GPU box): python tools/bench_f.py [out.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    import paper_2303_02724_b200 as eg

    torch.cuda.set_device(0)
    ctx = eg.Context(0)
    st = torch.cuda.current_stream()
    rows = []

    def timed(f, kw, flags, steps=7, warmup=3, label=""):
        for _ in range(warmup):
            ctx.compute(f, flags=flags | eg.EG_NO_GRAPH_D2H, materialize=False, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            ctx.compute(f, flags=flags | eg.EG_NO_GRAPH_D2H, materialize=False, **kw)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        g = ctx.graph()
        row = {"variant": label, "ms_per_step": round(ms, 4), "mvert_s": round(f.numel() / ms / 1e3, 1),
               "maxima": int(len(g.maxima)), "saddles": int(len(g.saddles)), "arcs": int(len(g.arcs))}
        if g.raw_arcs is not None:
            row["raw_arcs"] = int(len(g.raw_arcs))
        if g.arc_paths is not None:
            row["path_vertices"] = int(len(g.arc_paths[1]))
        return row

    for cfg in ("C2", "C3", "C5"):
        f, dims, csr = bench.make_input(cfg, "cuda:0")
        kw = dict(dims=dims) if dims is not None else dict(csr=csr)
        base = eg.EG_CHECK_NAN | eg.EG_GRAPH32
        variants = [("maximum graph", base),
                    ("f3 minimum graph (EG_MINIMUM)", base | eg.EG_MINIMUM),
                    ("f2 arc bundling (EG_BUNDLE)", base | eg.EG_BUNDLE),
                    ("f2 raw arcs (EG_RAW_ARCS)", base | eg.EG_RAW_ARCS),
                    ("f2 arc paths (EG_ARC_PATHS)", base | eg.EG_ARC_PATHS)]
        for label, flags in variants:
            row = timed(f, kw, flags, steps=3 if (cfg == "C3" and flags & eg.EG_ARC_PATHS) else 7, label=label)
            row["config"] = cfg
            rows.append(row)
            print(json.dumps(row), flush=True)
        # f4: node values on the device, cancellation on the host (serial, as in the paper)
        ctx.compute(f, flags=base | eg.EG_NODE_VALUES, **kw)
        fv = f.float().cpu().numpy() if f.dtype != torch.float32 else f.cpu().numpy()
        span = float(np.max(fv) - np.min(fv))
        for frac in (0.01, 0.1):
            t0 = time.perf_counter()
            s = ctx.simplify(frac * span)
            dt = time.perf_counter() - t0
            row = {"config": cfg, "variant": f"f4 eg_simplify tau = {frac} x range (host)", "host_ms": round(dt * 1e3, 2),
                   "maxima": int(len(s.maxima)), "saddles": int(len(s.saddles)), "arcs": int(len(s.arcs))}
            rows.append(row)
            print(json.dumps(row), flush=True)
        # f3: other input types through eg_compute_typed
        for tdt, label in ((torch.float64, "f3 float64, every value a float32 (exact cast, no rank sort)"),
                           ("f64-wide", "f3 float64 with 52-bit mantissas (SoS-rank image: radix sort)"),
                           (torch.float16, "f3 float16 (exact image)")):
            if tdt == "f64-wide":
                g64 = torch.Generator(device=f.device).manual_seed(64)
                ft = f.double() * (1.0 + 1e-12 * torch.rand(f.shape, generator=g64, device=f.device, dtype=torch.float64))
            else:
                ft = f.to(tdt)
            row = timed(ft, kw, base, steps=5, label=label)
            row["config"] = cfg
            rows.append(row)
            print(json.dumps(row), flush=True)
            del ft
        del f
        torch.cuda.empty_cache()
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
