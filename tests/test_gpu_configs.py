"""Parity at BASELINE.json's configurations, in the launch configuration
bench.py times (one eg_compute on the resident field, flags EG_CHECK_NAN).

Every config is compared with the oracle over the WHOLE domain, element by
element: maxima, saddles + beta0+, deduplicated arcs, every label, and (via
eg_gradient) every vertex's gradient pointer and beta0+.  C3 (2^30 vertices),
C4 and C5 use oracle.grid_parallel / csr_parallel -- the oracle's own
per-vertex range function on disjoint ranges in forked processes, pinned to
the whole-domain oracle by test_oracle_pins.py::test_parallel_equals_whole.
With EG_PARITY_RECORD=<dir> the full-size tests also write a record (field
sha256, per-output sha256 of both sides, result) to <dir>/<config>_parity.json
(committed under profiles/r02/).
"""
import json
import os
import time

import numpy as np
import pytest

import eg_inputs as G
import oracle as O
from _parity import assert_full_equal, assert_graph_equal, first_diff, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2303_02724_b200 as eg
    return eg


@pytest.fixture(scope="module")
def ctx(eg):
    c = eg.Context()
    yield c
    c.close()


def _sampled_grid_checks(g, f, dims, labels, n_lab=400, n_sad=150, seed=0):
    """Sampled parity for a big grid: labels by the oracle's Alg. 2 walk,
    saddles (beta0+, arcs) by the oracle's single-vertex classification."""
    rng = np.random.default_rng(seed)
    N = len(f)
    for v in rng.integers(0, N, n_lab):
        m, _ = O.grid_walk(f, dims, int(v))
        assert labels[v] == m, f"label of {v}: gpu {labels[v]} oracle {m}"
    # every reported maximum is a maximum, and is its own label
    for m in rng.choice(g.maxima, min(len(g.maxima), 200), replace=False):
        p, b, _ = O.grid_vertex(f, dims, int(m))
        assert b == 0 and p == m and labels[m] == m
    # sampled saddles: beta0+ and the deduplicated arcs
    arcs_by_s = {}
    for s, m, c in g.arcs.tolist():
        arcs_by_s.setdefault(s, []).append((m, c))
    js = rng.choice(len(g.saddles), min(len(g.saddles), n_sad), replace=False) if len(g.saddles) else []
    for j in js:
        s = int(g.saddles[j])
        p, b, reps = O.grid_vertex(f, dims, s)
        assert b == g.saddle_beta[j] and b >= 2
        ms = sorted(O.grid_walk(f, dims, int(r))[0] for r in reps)
        exp = sorted((m, ms.count(m)) for m in set(ms))
        assert sorted(arcs_by_s[s]) == exp, f"arcs of saddle {s}"
    # sampled non-saddle, non-maximum vertices really are regular (beta0+ == 1)
    sad = set(g.saddles.tolist())
    mx = set(g.maxima.tolist())
    for v in rng.integers(0, N, n_lab):
        if int(v) in sad or int(v) in mx:
            continue
        p, b, _ = O.grid_vertex(f, dims, int(v))
        assert b == 1, f"vertex {v} has beta0+ {b} but is not reported"
    # properties at any size
    assert int(g.arcs[:, 2].sum()) == int(g.saddle_beta.sum())
    assert np.all(np.diff(g.saddles) > 0) and np.all(np.diff(g.maxima) > 0)
    assert np.all(labels[g.maxima] == g.maxima)


def test_c1_config(eg, ctx):
    import torch
    f, dims = G.c1_gaussians(0, 4.0)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_CHECK_NAN)
    assert_graph_equal(g, O.grid(f, dims), what="C1")


def test_c2_config_full(eg, ctx):
    import torch
    f, dims = G.c2_gaussians_noise()
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_CHECK_NAN | eg.EG_RAW_ARCS)
    assert_graph_equal(g, o, raw=True, what="C2 256^3")


def test_c3_recipe_128_full(eg, ctx):
    import torch
    t, dims = G.turbulence(128, seed=1024, device="cuda")
    f = t.cpu().numpy()
    o = O.grid(f, dims)
    g = ctx.compute(t, dims=dims, flags=eg.EG_CHECK_NAN | eg.EG_RAW_ARCS)
    assert_graph_equal(g, o, raw=True, what="C3 recipe at 128^3")
    g2 = ctx.compute(t, dims=dims, flags=eg.EG_FORCE_GENERIC)
    assert_graph_equal(g2, o, what="C3 recipe at 128^3 (generic kernels)")


def _record(cfg, f, g, o, t_gpu, t_oracle, extra=None):
    d = os.environ.get("EG_PARITY_RECORD")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    lab = g.labels.cpu().numpy().astype(np.int64)
    rec = {"config": cfg, "n_vertices": int(len(f)), "field_sha256": sha(f),
           "result": "exact (every output element-equal)",
           "gpu": {"maxima": sha(g.maxima), "saddles": sha(g.saddles), "saddle_beta": sha(g.saddle_beta.astype(np.int32)),
                   "arcs": sha(g.arcs), "labels": sha(lab)},
           "oracle": {"maxima": sha(o.maxima), "saddles": sha(o.saddles), "saddle_beta": sha(o.saddle_beta),
                      "arcs": sha(o.arcs), "labels": sha(o.label)},
           "counts": {"maxima": int(len(o.maxima)), "saddles": int(len(o.saddles)), "arcs": int(len(o.arc_s)),
                      "raw_arcs": int(len(o.raw_s)), "multi_saddles": int((o.saddle_beta >= 3).sum())},
           "seconds": {"gpu_compute": round(t_gpu, 4), "oracle_parallel": round(t_oracle, 1),
                       "oracle_procs": os.cpu_count()}}
    rec.update(extra or {})
    with open(os.path.join(d, f"{cfg}_parity.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


def _full_grid(eg, ctx, cfg, t, dims):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = ctx.compute(t, dims=dims, flags=eg.EG_CHECK_NAN)
    t_gpu = time.perf_counter() - t0
    ptr, beta = ctx.gradient(t, dims=dims)
    ptr, beta = ptr.cpu().numpy(), beta.cpu().numpy()
    f = t.cpu().numpy()
    t0 = time.perf_counter()
    o = O.grid_parallel(f, dims)
    t_or = time.perf_counter() - t0
    assert_full_equal(g, o, ptr, beta, what=cfg)
    _record(cfg, f, g, o, t_gpu, t_or)
    return g, o


def test_c3_config_full(eg, ctx):
    """C3 1024^3: the whole domain against the oracle (2^30 vertices)."""
    import torch
    t, dims = G.turbulence(1024, seed=1024, device="cuda")
    g, o = _full_grid(eg, ctx, "C3", t, dims)
    # SURVEY App. A expectations at this recipe (self-similar counts): order of
    # 10^5 maxima, saddles about 3x maxima
    assert 5e4 < len(g.maxima) < 5e5 and 1.5 * len(g.maxima) < len(g.saddles) < 6 * len(g.maxima)
    del t
    torch.cuda.empty_cache()


def test_c4_config_full(eg, ctx):
    import torch
    f, dims = G.schwefel()
    g, o = _full_grid(eg, ctx, "C4", torch.from_numpy(f).cuda(), dims)
    # separable product rule (tests/test_oracle_pins.py::test_schwefel_profile_counts)
    assert len(g.maxima) == 7 ** 5 == 16807
    assert len(g.saddles) == 5 * 6 * 7 ** 4 == 72030
    assert (g.saddle_beta == 2).all()


def test_c4_recipe_small_full(eg, ctx):
    import torch
    for dims in ([12] * 5, [9, 10, 11, 12, 13]):
        f, _ = G.schwefel(dims)
        o = O.grid(f, dims)
        g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_RAW_ARCS)
        assert_graph_equal(g, o, raw=True, what=f"Schwefel {dims}")
    f, dims, *_ = G.sumcos([16] * 5, seed=5)
    assert_graph_equal(ctx.compute(torch.from_numpy(f).cuda(), dims=dims), O.grid(f, dims), what="sumcos 16^5")


def test_c5_config_full(eg, ctx):
    import torch
    X, f = G.gmm_points(1_000_000, seed=10)
    rp, ci = G.knn_csr(X, 16, device="cuda")
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    ft = torch.from_numpy(f).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = ctx.compute(ft, csr=csr, flags=eg.EG_CHECK_NAN)
    t_gpu = time.perf_counter() - t0
    ptr, beta = ctx.gradient(ft, csr=csr)
    t0 = time.perf_counter()
    o = O.csr_parallel(f, rp, ci)
    t_or = time.perf_counter() - t0
    assert_full_equal(g, o, ptr.cpu().numpy(), beta.cpu().numpy(), what="C5")
    _record("C5", f, g, o, t_gpu, t_or, {"csr_sha256": {"row_ptr": sha(rp), "col_idx": sha(ci)}})
    assert int(g.arcs[:, 2].sum()) == int(g.saddle_beta.sum())


def test_f1_resolution_sweep(eg, ctx):
    """the Schwefel 3-D resolution sweep.  128^3 in full against
    the oracle; 256^3 and 512^3 against the separable product rule (the same
    512 maxima / 1344 2-saddles at every resolution >= 128) plus sampled parity."""
    import torch
    src = open(__file__.replace("test_gpu_configs.py", "../tools/sweep_f1.py")).read()
    ns = {}
    exec(src[src.index("def product_rule"):src.index("rows = []")], {"np": np, "G": G}, ns)
    f, dims = G.schwefel((128,) * 3)
    o = O.grid(f, dims)
    assert_graph_equal(ctx.compute(torch.from_numpy(f).cuda(), dims=dims), o, what="F1 128^3")
    assert (len(o.maxima), len(o.saddles)) == ns["product_rule"](128)
    for n in (256, 512):
        t, dims = G.schwefel((n,) * 3, device="cuda")
        g = ctx.compute(t, dims=dims)
        assert (len(g.maxima), len(g.saddles)) == ns["product_rule"](n)
        assert np.all(g.saddle_beta == 2)
        _sampled_grid_checks(g, t.cpu().numpy(), dims, g.labels.cpu().numpy().astype(np.int64), n_lab=200, n_sad=80)
