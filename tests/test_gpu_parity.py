"""GPU parity against the CPU oracle, element by element, through the C ABI.

Bit-exact on every output (labels, maxima, saddles + beta0+, deduplicated and
raw arcs, gradients): the method has no floating-point arithmetic, only
comparisons (reading L16), so the tolerance is zero.  Small / ragged sizes
that still span several tiles, every grid dimension 1..6, tie-heavy and
signed-zero fields, the degenerate cases, and both the tiled 3-D path and the
generic n-D kernels.
"""
import json
import os

import numpy as np
import pytest

import eg_inputs as G
import oracle as O
from _parity import assert_graph_equal, first_diff

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tiny_examples.json")
PATHS = [0, "generic"]


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


def _flags(eg, path, extra=0):
    return extra | (eg.EG_FORCE_GENERIC if path == "generic" else 0)


def _run(eg, ctx, f, dims, path=0, extra=0):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda()
    return ctx.compute(t, dims=dims, flags=_flags(eg, path, extra | eg.EG_RAW_ARCS | eg.EG_CHECK_NAN))


@pytest.mark.parametrize("path", PATHS)
def test_golden(eg, ctx, path):
    for case in json.load(open(GOLDEN))["cases"]:
        g = _run(eg, ctx, np.array(case["f"], np.float32), case["dims"], path)
        assert g.maxima.tolist() == case["maxima"], case["name"]
        assert [[int(s), int(b)] for s, b in zip(g.saddles, g.saddle_beta)] == case["saddles"], case["name"]
        assert g.arcs.tolist() == case["arcs"], case["name"]
        assert g.labels.cpu().numpy().tolist() == case["labels"], case["name"]


@pytest.mark.parametrize("path", PATHS)
def test_c1_full(eg, ctx, path):
    f, dims = G.c1_gaussians(0, 4.0)
    o = O.grid(f, dims)
    g = _run(eg, ctx, f, dims, path)
    assert_graph_equal(g, o, raw=True, what=f"C1 ({path})")
    assert len(g.maxima) == 8


@pytest.mark.parametrize("path", PATHS)
def test_sincos(eg, ctx, path):
    f, dims, *_ = G.sincos(4, 4, 7)
    assert_graph_equal(_run(eg, ctx, f, dims, path), O.grid(f, dims), raw=True, what="sincos")


CASES = [
    ([1], "normal"), ([2], "int"), ([37], "int"), ([1000], "normal"),
    ([1, 1], "const"), ([7, 1], "int"), ([1, 9], "int"), ([33, 17], "int"), ([64, 64], "normal"),
    ([130, 67], "signed_zero"), ([2, 2, 2], "int"), ([1, 1, 5], "int"), ([3, 1, 4], "int"),
    ([33, 35, 19], "int"), ([65, 33, 17], "normal"), ([70, 9, 40], "signed_zero"), ([31, 64, 33], "const"),
    ([7, 6, 5, 4], "int"), ([9, 8, 7, 6], "normal"), ([6, 5, 4, 3, 3], "int"), ([8, 7, 6, 5, 4], "normal"),
    ([4, 3, 3, 2, 3, 3], "int"), ([5, 4, 4, 3, 3, 2], "normal"),
    # extents of 1 and 2 on inner axes (the generic kernel's coordinate division and truncated link)
    ([5, 1, 4, 3], "int"), ([3, 4, 1, 2, 5], "int"), ([2, 1, 3, 1, 2, 3], "int"), ([1, 7, 1, 6, 1], "normal"),
    ([37, 3, 2, 2, 3], "signed_zero"),
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("dims,kind", CASES)
def test_random_fields(eg, ctx, path, dims, kind):
    f, _ = G.random_field(dims, 17 + len(dims), kind)
    assert_graph_equal(_run(eg, ctx, f, dims, path), O.grid(f, dims), raw=True, what=f"{dims} {kind} {path}")


@pytest.mark.parametrize("dims,kind", [([33, 17], "int"), ([65, 33, 17], "normal"), ([9, 8, 7, 6], "int"),
                                       ([8, 7, 6, 5, 4], "normal"), ([4, 3, 3, 2, 3, 3], "int")])
def test_gradient_and_beta(eg, ctx, dims, kind):
    # S1 (gradient) and S3 (beta0+) per vertex
    import torch
    f, _ = G.random_field(dims, 3, kind)
    o = O.grid(f, dims)
    ptr, beta = ctx.gradient(torch.from_numpy(f).cuda(), dims=dims)
    assert first_diff(ptr.cpu().numpy().astype(np.int64), o.ptr) is None
    assert first_diff(beta.cpu().numpy().astype(np.int32), np.minimum(o.beta, 255)) is None


def test_determinism(eg, ctx):
    f, dims = G.random_field([70, 40, 30], 5, "int")
    runs = [_run(eg, ctx, f, dims) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.arcs, runs[0].arcs)
        assert np.array_equal(r.labels.cpu().numpy(), runs[0].labels.cpu().numpy())


def test_tiled_equals_generic(eg, ctx):
    f, dims = G.c2_gaussians_noise(n=96, seed=3, k=12)
    a = _run(eg, ctx, f, dims, 0)
    la = a.labels.cpu().numpy().copy()
    b = _run(eg, ctx, f, dims, "generic")
    assert np.array_equal(a.arcs, b.arcs) and np.array_equal(a.saddles, b.saddles)
    assert np.array_equal(la, b.labels.cpu().numpy())


def test_nan_rejected(eg, ctx):
    f, dims = G.random_field([20, 10, 5], 1, "normal")
    f[123] = np.nan
    for path in PATHS:
        with pytest.raises(eg.EgError) as e:
            _run(eg, ctx, f, dims, path)
        assert "EG_ERR_NAN" in str(e.value)
    # the context stays usable after a NaN (not sticky)
    f2, _ = G.random_field([20, 10, 5], 1, "normal")
    assert_graph_equal(_run(eg, ctx, f2, dims), O.grid(f2, dims))


def test_invalid_args(eg, ctx):
    import torch
    t = torch.zeros(8, device="cuda")
    with pytest.raises(eg.EgError) as e:
        ctx.compute(t, dims=[2, 0, 4])
    assert "INVALID_ARG" in str(e.value)
    with pytest.raises(eg.EgError) as e:         # 1 <= ndim <= 8
        ctx.compute(t, dims=[2] * 9)
    assert "INVALID_ARG" in str(e.value)
    with pytest.raises(eg.EgError) as e:      # N >= 2^31: rejected before touching memory
        ctx.compute(t, dims=[2048, 2048, 1024])
    assert "UNSUPPORTED" in str(e.value)


def test_csr_equals_grid(eg, ctx):
    # L14: the CSR kernels on the Freudenthal graph == the grid kernels
    import torch
    from oracle import brute
    dims = [9, 7, 5]
    f, _ = G.random_field(dims, 8, "int")
    row_ptr, col_idx = brute.freudenthal_csr(dims)
    csr = (torch.from_numpy(row_ptr).cuda(), torch.from_numpy(col_idx).cuda())
    t = torch.from_numpy(f).cuda()
    a = ctx.compute(t, csr=csr, flags=eg.EG_RAW_ARCS)
    la = a.labels.cpu().numpy().copy()
    b = ctx.compute(t, dims=dims, flags=eg.EG_RAW_ARCS)
    assert np.array_equal(a.arcs, b.arcs) and np.array_equal(a.raw_arcs, b.raw_arcs)
    assert np.array_equal(la, b.labels.cpu().numpy())


@pytest.mark.parametrize("n,p,seed,kind", [(12, 0.3, 0, "normal"), (40, 0.2, 1, "int"), (300, 0.05, 2, "int"),
                                           (500, 0.02, 3, "normal")])
def test_csr_random(eg, ctx, n, p, seed, kind):
    import torch
    row_ptr, col_idx = G.random_csr(n, p, seed)
    f, _ = G.random_field([n], seed, kind, levels=3)
    o = O.csr(f, row_ptr, col_idx)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(row_ptr).cuda(),
                                                     torch.from_numpy(col_idx).cuda()),
                    flags=eg.EG_RAW_ARCS | eg.EG_CHECK_NAN)
    assert_graph_equal(g, o, raw=True, what="csr random")


@pytest.mark.parametrize("n,p,seed,kind", [(150, 0.35, 5, "normal"), (160, 0.4, 6, "int"), (220, 0.7, 7, "normal"),
                                           (260, 0.8, 8, "int")])
def test_csr_dense(eg, ctx, n, p, seed, kind):
    """Rows longer than a warp (the flattened link-edge pass spans several
    chunks per row) and upper sets larger than 64 (the serial fallback of the
    warp kernel): there is no degree cap."""
    import torch
    row_ptr, col_idx = G.random_csr(n, p, seed)
    f, _ = G.random_field([n], seed, kind, levels=4)
    o = O.csr(f, row_ptr, col_idx)
    csr = (torch.from_numpy(row_ptr).cuda(), torch.from_numpy(col_idx).cuda())
    ft = torch.from_numpy(f).cuda()
    g = ctx.compute(ft, csr=csr, flags=eg.EG_RAW_ARCS | eg.EG_CHECK_NAN | eg.EG_CHECK_CSR)
    assert_graph_equal(g, o, raw=True, what=f"csr dense {n} {p}")
    ptr, beta = ctx.gradient(ft, csr=csr)
    assert first_diff(ptr.cpu().numpy().astype(np.int64), o.ptr) is None
    assert first_diff(beta.cpu().numpy().astype(np.int32), np.minimum(o.beta, 255)) is None
    if p >= 0.7:
        deg = np.diff(row_ptr)
        assert deg.max() > 128          # beyond the old per-thread cap


def test_csr_hub(eg, ctx):
    """One vertex adjacent to every other (a hub) on a path graph: the hub's
    upper set is everything, its link is the path (one component); the lowest
    path vertices see the hub."""
    import torch
    n = 300
    adj = [set() for _ in range(n)]
    for v in range(1, n - 1):
        adj[v].add(v + 1)
        adj[v + 1].add(v)
    for v in range(1, n):
        adj[0].add(v)
        adj[v].add(0)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(a) for a in adj])
    ci = np.array([u for a in adj for u in sorted(a)], np.int32)
    rng = np.random.default_rng(3)
    f = rng.standard_normal(n).astype(np.float32)
    f[0] = -10.0
    o = O.csr(f, rp, ci)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()),
                    flags=eg.EG_RAW_ARCS | eg.EG_CHECK_CSR)
    assert_graph_equal(g, o, raw=True, what="csr hub")


def test_check_csr(eg, ctx):
    """EG_CHECK_CSR: a malformed graph is EG_ERR_INVALID_ARG before any kernel
    indexes through it, and the context stays usable."""
    import torch
    rp, ci = G.random_csr(60, 0.2, 2)
    f, _ = G.random_field([60], 2, "normal")
    ft = torch.from_numpy(f).cuda()

    def run(rp_, ci_):
        return ctx.compute(ft[:len(rp_) - 1], csr=(torch.from_numpy(rp_).cuda(), torch.from_numpy(ci_).cuda()),
                           flags=eg.EG_CHECK_CSR)

    assert_graph_equal(run(rp, ci), O.csr(f, rp, ci), what="valid csr")
    bad = []
    c = ci.copy()                               # unsorted row
    r = int(np.argmax(np.diff(rp) >= 2))
    c[rp[r]], c[rp[r] + 1] = c[rp[r] + 1], c[rp[r]]
    bad.append((rp, c))
    c = ci.copy()                               # out of range
    c[3] = 60
    bad.append((rp, c))
    c = ci.copy()                               # self loop (keeps the row sorted only by luck; either code)
    v = int(np.searchsorted(rp, 5, side="right") - 1)
    c[5] = v
    bad.append((rp, c))
    rp2 = rp.copy()                             # row_ptr not ending at nnz
    rp2[-1] -= 1
    bad.append((rp2, ci))
    # asymmetric: drop one directed edge (u in N(v) but v not in N(u))
    v = int(np.argmax(np.diff(rp) >= 1))
    keep = np.ones(len(ci), bool)
    keep[rp[v]] = False
    rp3 = rp.copy()
    rp3[v + 1:] -= 1
    bad.append((rp3, ci[keep].copy()))
    for rp_, ci_ in bad:
        with pytest.raises(eg.EgError) as e:
            run(rp_, ci_)
        assert e.value.status == 1, str(e.value)     # EG_ERR_INVALID_ARG
    assert_graph_equal(run(rp, ci), O.csr(f, rp, ci), what="valid csr after refused calls")


def test_csr_knn_small(eg, ctx):
    import torch
    X, f = G.gmm_points(20000, seed=10)
    row_ptr, col_idx = G.knn_csr(X, 16, device="cuda")
    o = O.csr(f, row_ptr, col_idx)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(row_ptr).cuda(),
                                                     torch.from_numpy(col_idx).cuda()), flags=eg.EG_RAW_ARCS)
    assert_graph_equal(g, o, raw=True, what="knn 20K")


def test_compute_host_e2e(eg, ctx):
    import torch
    f, dims = G.c2_gaussians_noise(n=64, seed=1, k=8)
    o = O.grid(f, dims)
    host = torch.from_numpy(f).pin_memory()
    lab = torch.empty(len(f), dtype=torch.int32).pin_memory()
    g = ctx.compute_host(host, dims=dims, labels_out=lab)
    assert_graph_equal(g, o)
    assert np.array_equal(lab.numpy().astype(np.int64), o.label)
    g2 = ctx.compute_host(torch.from_numpy(f), dims=dims)      # pageable source
    assert_graph_equal(g2, o)


@pytest.mark.parametrize("dims,kind", [([3, 4, 3, 3, 3, 3, 4], "int"), ([3, 4, 3, 3, 3, 3, 4], "normal"),
                                       ([3, 2, 3, 2, 3, 2, 3, 4], "int"), ([4, 3, 3, 3, 3, 3, 3, 4], "normal")])
def test_grid_7d_8d(eg, ctx, dims, kind):
    """n = 7, 8 (1 <= ndim <= 8): the generic kernels on
    multi-limb lattice words (254 / 510 link vertices), raw arcs, gradient,
    and 2 virtual slabs."""
    import torch
    f, _ = G.random_field(dims, 40 + len(dims), kind, levels=3)
    o = O.grid(f, dims)
    t = torch.from_numpy(f).cuda()
    assert_graph_equal(ctx.compute(t, dims=dims, flags=eg.EG_RAW_ARCS | eg.EG_CHECK_NAN), o, raw=True,
                       what=f"{len(dims)}-D {kind}")
    assert_graph_equal(ctx.compute(t, dims=dims, flags=eg.EG_VIRTUAL_PARTS(2)), o, what=f"{len(dims)}-D 2 slabs")
    ptr, beta = ctx.gradient(t, dims=dims)
    assert first_diff(ptr.cpu().numpy().astype(np.int64), o.ptr) is None
    assert first_diff(beta.cpu().numpy().astype(np.int32), np.minimum(o.beta, 255)) is None


def test_graph32(eg, ctx):
    """EG_GRAPH32: the graph crosses to the host with 32-bit ids (eg_get_graph32);
    eg_get_graph widens it on demand, and a 64-bit graph narrows for
    eg_get_graph32 -- every path gives the oracle's graph."""
    import ctypes as C
    import torch
    from paper_2303_02724_b200 import _abi
    f, dims = G.c2_gaussians_noise(n=64, seed=3, k=8)
    o = O.grid(f, dims)
    t = torch.from_numpy(f).cuda()
    for extra in (0, eg.EG_FORCE_GENERIC, eg.EG_VIRTUAL_PARTS(3), eg.EG_BUNDLE, eg.EG_NODE_VALUES):
        g = ctx.compute(t, dims=dims, flags=eg.EG_GRAPH32 | extra)
        exp = O.bundle(o, f) if extra == eg.EG_BUNDLE else o
        assert_graph_equal(g, exp, what=f"graph32 {extra}")
        g64 = _abi.EgGraph()                      # the other width from the same compute
        assert _abi.lib().eg_get_graph(ctx._h, C.byref(g64)) == 0
        assert g64.n_arc == len(exp.arc_s) and [g64.arc_max[i] for i in range(min(5, g64.n_arc))] == \
            exp.arc_m[:5].tolist()
    g = ctx.compute(t, dims=dims)                 # 64-bit graph, read as 32-bit
    g32 = _abi.EgGraph32()
    assert _abi.lib().eg_get_graph32(ctx._h, C.byref(g32)) == 0
    assert [g32.saddles[i] for i in range(g32.n_saddle)] == o.saddles.tolist()
    X, fc = G.gmm_points(5000, seed=2)
    rp, ci = G.knn_csr(X, 12)
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    assert_graph_equal(ctx.compute(torch.from_numpy(fc).cuda(), csr=csr, flags=eg.EG_GRAPH32), O.csr(fc, rp, ci),
                       what="graph32 csr")
    host = torch.from_numpy(f).pin_memory()
    lab = torch.empty(len(f), dtype=torch.int32).pin_memory()
    assert_graph_equal(ctx.compute_host(host, dims=dims, labels_out=lab, flags=eg.EG_GRAPH32), o, what="graph32 e2e")


@pytest.mark.parametrize("chunks", ["2", "5", "16", "32", "1"])
def test_compute_host_pipeline(eg, ctx, chunks, monkeypatch):
    """eg_compute_host's pipeline (field in z-chunks, each chunk's labels
    copied while later chunks arrive, late-finished labels patched on the
    host): a smooth field whose chains cross several chunks, any chunk count;
    labels bit-exact, also with a pageable label buffer (no pipeline) and
    after a device-resident compute."""
    import torch
    monkeypatch.setenv("EG_E2E_CHUNKS", chunks)
    t, dims = G.turbulence(64, seed=5, device="cpu", kc_div=4)
    f = np.ascontiguousarray(np.tile(t.numpy().reshape(64, 64, 64), (4, 1, 1)).reshape(-1))   # 64 x 64 x 256
    dims = [64, 64, 256]
    o = O.grid(f, dims)
    host = torch.from_numpy(f).pin_memory()
    for _ in range(2):
        lab = torch.full((len(f),), -7, dtype=torch.int32).pin_memory()
        g = ctx.compute_host(host, dims=dims, labels_out=lab, flags=eg.EG_CHECK_NAN)
        assert_graph_equal(g, o, what=f"pipeline {chunks}")
        assert first_diff(lab.numpy().astype(np.int64), o.label) is None
    lab2 = torch.zeros(len(f), dtype=torch.int32)                 # pageable: plain path
    ctx.compute_host(host, dims=dims, labels_out=lab2)
    assert np.array_equal(lab2.numpy().astype(np.int64), o.label)
    g3 = ctx.compute(host.cuda(), dims=dims)
    assert_graph_equal(g3, o, what="device compute after the pipeline")


@pytest.mark.parametrize("dims,kind", [([70, 9, 40], "signed_zero"), ([33, 35, 19], "int"), ([96, 64, 48], "int")])
def test_tie_heavy_repeated(eg, ctx, dims, kind):
    # in-place races in the shared-memory chase / exit resolution must never
    # change a result: 20 repetitions, every one bit-exact
    import torch
    f, _ = G.random_field(dims, 17 + len(dims), kind)
    o = O.grid(f, dims)
    t = torch.from_numpy(f).cuda()
    for _ in range(20):
        g = ctx.compute(t, dims=dims)
        assert first_diff(g.labels.cpu().numpy().astype(np.int64), o.label) is None
        assert np.array_equal(g.arcs, o.arcs)


# ---------------------------------------------------------------- partitions
# the slab partition must give identical outputs for any number
# of slabs.  EG_VIRTUAL_PARTS(k) runs k slabs on one GPU with the exact
# multi-GPU protocol (halo planes, boundary-plane exchange rounds, per-slab
# graphs concatenated in slab order), the exchange done by device copies.

@pytest.mark.parametrize("k", [2, 3, 4, 7])
@pytest.mark.parametrize("path", PATHS)
def test_virtual_slabs_3d(eg, ctx, k, path):
    import torch
    t, dims = G.turbulence(64, seed=11, device="cuda", kc_div=8)
    f = t.cpu().numpy()
    o = O.grid(f, dims)
    g = ctx.compute(t, dims=dims, flags=_flags(eg, path, eg.EG_VIRTUAL_PARTS(k) | eg.EG_RAW_ARCS))
    assert_graph_equal(g, o, raw=True, what=f"turbulence 64^3, {k} slabs, {path}")
    st = ctx.stats()
    assert st["boundary_rounds"] >= 1


@pytest.mark.parametrize("k", [2, 5, 16])
@pytest.mark.parametrize("path", PATHS)
def test_virtual_slabs_ridge(eg, ctx, k, path):
    """A ramp along the slowest axis with a wavy ridge (SPEC S:313 analogue):
    nearly every ascending path crosses every slab boundary above it, so the
    boundary exchange needs about k - 1 rounds (several host-checked batches
    at k = 16) and every finalize chain ends in a remote label."""
    import torch
    nx, ny, nz = 40, 24, 64
    x, y, z = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    rng = np.random.default_rng(k)
    f = (z + 0.6 * np.sin(x / 3.0) * np.cos(y / 4.0) + 0.05 * rng.standard_normal(z.shape)).astype(np.float32)
    f = np.ascontiguousarray(f.transpose(2, 1, 0)).reshape(-1)      # axis 0 (x) fastest
    dims = [nx, ny, nz]
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=_flags(eg, path, eg.EG_VIRTUAL_PARTS(k)))
    assert_graph_equal(g, o, what=f"ridge, {k} slabs, {path}")
    assert ctx.stats()["boundary_rounds"] >= k - 1


@pytest.mark.parametrize("dims,kind,k", [([40, 36, 50], "int", 3), ([70, 9, 40], "signed_zero", 4),
                                         ([33, 35, 19], "normal", 2), ([64, 64, 64], "int", 8)])
def test_virtual_slabs_tie_heavy(eg, ctx, dims, kind, k):
    import torch
    f, _ = G.random_field(dims, 5, kind)
    o = O.grid(f, dims)
    for path in PATHS:
        g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=_flags(eg, path, eg.EG_VIRTUAL_PARTS(k)))
        assert_graph_equal(g, o, what=f"{dims} {kind} {k} slabs {path}")


@pytest.mark.parametrize("dims,k", [([9, 8, 7, 10], 3), ([8, 7, 6, 5, 12], 4), ([60, 50], 5), ([200], 6)])
def test_virtual_slabs_nd(eg, ctx, dims, k):
    import torch
    f, _ = G.random_field(dims, 9, "int")
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_VIRTUAL_PARTS(k) | eg.EG_RAW_ARCS)
    assert_graph_equal(g, o, raw=True, what=f"{dims} {k} slabs")


def test_virtual_slabs_schwefel_5d(eg, ctx):
    import torch
    f, dims = G.schwefel([12, 12, 12, 12, 16])
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_VIRTUAL_PARTS(4))
    assert_graph_equal(g, o, what="Schwefel 5D, 4 slabs")


@pytest.mark.parametrize("k", [2, 5])
def test_virtual_ranges_csr(eg, ctx, k):
    import torch
    X, f = G.gmm_points(5000, seed=10)
    rp, ci = G.knn_csr(X, 16, device="cuda")
    o = O.csr(f, rp, ci)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()),
                    flags=eg.EG_VIRTUAL_PARTS(k) | eg.EG_RAW_ARCS)
    assert_graph_equal(g, o, raw=True, what=f"knn 5K, {k} ranges")


def test_virtual_slabs_invalid(eg, ctx):
    import torch
    f, dims = G.random_field([8, 8, 5], 1, "int")
    with pytest.raises(eg.EgError) as e:          # 5 planes cannot make 3 slabs of >= 2 planes
        ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_VIRTUAL_PARTS(3))
    assert "INVALID_ARG" in str(e.value)


@pytest.mark.parametrize("env", [{"EG_LIST_DIV": "100000"},                       # maxima/saddle lists regrow + rerun
                                 {"EG_ELIST": "1"},                               # one slab with the exit list + resolve
                                 {"EG_ELIST": "0"},                               # one slab, no list: finalize chases
                                 {"EG_ELIST": "1", "EG_ELIST_DIV": "100000"}])    # exit list overflow -> per-vertex chase
def test_tiled_capacity_paths(eg, env, monkeypatch):
    """The tiled path's variants (list growth, exit list or finalize chase, exit-list overflow) stay bit-exact."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ctx = eg.Context()
    for dims, kind in [([96, 64, 48], "int"), ([70, 41, 37], "normal")]:
        f, _ = G.random_field(dims, 23 + len(dims), kind)
        o = O.grid(f, dims)
        g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims)
        assert_graph_equal(g, o, what=f"{env} {dims} {kind}")


@pytest.mark.parametrize("dims,kind", [([97], "int"), ([64, 64], "normal"), ([70, 41, 37], "int"),
                                       ([96, 64, 48], "signed_zero"), ([9, 8, 7, 6], "normal")])
@pytest.mark.parametrize("path", PATHS)
def test_minimum_graph(eg, ctx, dims, kind, path):
    """EG_MINIMUM (reading L11): minima, 1-saddles, descending arcs and labels,
    bit-exact against the oracle's reversed-order transcription (O10)."""
    import torch
    f, _ = G.random_field(dims, 31 + len(dims), kind)
    o = O.grid(f, dims, minimum=True)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=_flags(eg, path, eg.EG_MINIMUM | eg.EG_CHECK_NAN))
    assert_graph_equal(g, o, what=f"minimum {dims} {kind} {path}")
    # and the maximum graph of the same field on the same context is unaffected
    assert_graph_equal(ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=_flags(eg, path)), O.grid(f, dims))


@pytest.mark.parametrize("n,p,seed,kind", [(12, 0.3, 0, "normal"), (300, 0.05, 2, "int"), (500, 0.02, 3, "normal")])
def test_minimum_graph_csr(eg, ctx, n, p, seed, kind):
    """EG_MINIMUM on a CSR graph: the maximum graph of the reversed rank image
    (reading L22), against the oracle's reversed-order transcription (O10)."""
    import torch
    rp, ci = G.random_csr(n, p, seed)
    f, _ = G.random_field([n], seed, kind, levels=3)
    if kind == "normal":                                    # -0 ties with +0 (reading L2)
        f[::7], f[3::7] = -0.0, 0.0
    o = O.csr(f, rp, ci, minimum=True)
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=csr, flags=eg.EG_MINIMUM | eg.EG_CHECK_NAN)
    assert_graph_equal(g, o, what=f"csr minimum {n} {kind}")


def test_minimum_graph_csr_knn(eg, ctx):
    """kNN graph (C5 recipe, 20K points): minimum graph, bundled minimum graph,
    and the simplified minimum graph (node values from the caller's field)."""
    import torch
    X, f = G.gmm_points(20000, seed=12)
    rp, ci = G.knn_csr(X, 12)
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    t = torch.from_numpy(f).cuda()
    o = O.csr(f, rp, ci, minimum=True)
    assert_graph_equal(ctx.compute(t, csr=csr, flags=eg.EG_MINIMUM), o, what="knn minimum")
    assert_graph_equal(ctx.compute(t, csr=csr, flags=eg.EG_MINIMUM | eg.EG_BUNDLE),
                       O.bundle(o, f, minimum=True), what="knn minimum bundled")
    ctx.compute(t, csr=csr, flags=eg.EG_MINIMUM | eg.EG_NODE_VALUES)
    for tau in (0.0, 0.5):
        s = ctx.simplify(tau)
        e = O.simplify(o, f, tau, minimum=True)
        assert np.array_equal(s.maxima, e.maxima) and np.array_equal(s.arcs, e.arcs), tau
    assert_graph_equal(ctx.compute(t, csr=csr), O.csr(f, rp, ci), what="knn maximum after minimum")


def test_minimum_graph_unsupported(eg, ctx):
    import torch
    f, dims = G.random_field([20, 20, 20], 3, "normal")
    with pytest.raises(Exception):
        ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_MINIMUM | eg.EG_VIRTUAL_PARTS(2))
    rp, ci = G.random_csr(200, 0.05, 4)
    fc, _ = G.random_field([200], 4, "normal")
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    with pytest.raises(eg.EgError) as e:          # one GPU owns every vertex (the rank image needs them all)
        ctx.compute(torch.from_numpy(fc).cuda(), csr=csr, v_range=(0, 100), flags=eg.EG_MINIMUM)
    assert e.value.status == 1
    assert_graph_equal(ctx.compute(torch.from_numpy(fc).cuda(), csr=csr, flags=eg.EG_MINIMUM),
                       O.csr(fc, rp, ci, minimum=True), what="csr minimum after a refused call")


def _oracle_paths(o):
    """Alg. 2 integral lines from the oracle: s, rep, then ptr steps to m."""
    paths = []
    for s, rep, m in zip(o.raw_s.tolist(), o.raw_rep.tolist(), o.raw_m.tolist()):
        p = [s, rep]
        v = rep
        while o.ptr[v] != v:
            v = int(o.ptr[v])
            p.append(v)
        assert p[-1] == m
        paths.append(p)
    return paths


@pytest.mark.parametrize("dims,kind", [([61], "int"), ([48, 40], "normal"), ([40, 33, 29], "int"), ([9, 8, 7, 6], "normal")])
def test_arc_paths_grid(eg, ctx, dims, kind):
    """EG_ARC_PATHS: every integral line bit-exact against the oracle's gradient chain."""
    import torch
    f, _ = G.random_field(dims, 41 + len(dims), kind)
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_ARC_PATHS)
    assert_graph_equal(g, o, raw=True, what=f"paths {dims}")
    off, v = g.arc_paths
    exp = _oracle_paths(o)
    assert len(off) == len(exp) + 1
    got = [v[off[j]:off[j + 1]].tolist() for j in range(len(exp))]
    assert got == exp


def test_arc_paths_csr(eg, ctx):
    import torch
    X, f = G.gmm_points(3000, seed=4)
    rp, ci = G.knn_csr(X, 8)
    o = O.csr(f, rp, ci)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()),
                    flags=eg.EG_ARC_PATHS)
    off, v = g.arc_paths
    exp = _oracle_paths(o)
    assert [v[off[j]:off[j + 1]].tolist() for j in range(len(exp))] == exp


@pytest.mark.parametrize("dims,kind", [([64, 48], "int"), ([40, 33, 29], "normal"), ([9, 8, 7, 6], "int"),
                                       ("csr", "normal")])
def test_minimum_raw_arcs_and_paths(eg, ctx, dims, kind):
    """EG_MINIMUM with EG_RAW_ARCS / EG_ARC_PATHS (the reversed rank image,
    reading L22): raw descending arcs and every descending integral line."""
    import torch
    if dims == "csr":
        X, f = G.gmm_points(3000, seed=5)
        rp, ci = G.knn_csr(X, 8)
        o = O.csr(f, rp, ci, minimum=True)
        kw = dict(csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()))
    else:
        f, _ = G.random_field(dims, 43 + len(dims), kind)
        o = O.grid(f, dims, minimum=True)
        kw = dict(dims=dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), flags=eg.EG_MINIMUM | eg.EG_RAW_ARCS, **kw)
    assert_graph_equal(g, o, raw=True, what=f"minimum raw {dims}")
    g = ctx.compute(torch.from_numpy(f).cuda(), flags=eg.EG_MINIMUM | eg.EG_ARC_PATHS, **kw)
    off, v = g.arc_paths
    exp = _oracle_paths(o)
    assert [v[off[j]:off[j + 1]].tolist() for j in range(len(exp))] == exp


@pytest.mark.parametrize("dims,kind,minimum", [([64, 48], "normal", False), ([40, 33, 29], "normal", False),
                                               ([96, 64, 48], "int", False), ([9, 8, 7, 6], "normal", False),
                                               ([40, 33, 29], "normal", True)])
@pytest.mark.parametrize("path", PATHS)
def test_bundled_graph(eg, ctx, dims, kind, minimum, path):
    """EG_BUNDLE (reading L19) against the oracle's literal bundling."""
    import torch
    f, _ = G.random_field(dims, 51 + len(dims), kind)
    o = O.bundle(O.grid(f, dims, minimum=minimum), f, minimum=minimum)
    fl = eg.EG_BUNDLE | (eg.EG_MINIMUM if minimum else 0)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=_flags(eg, path, fl))
    assert_graph_equal(g, o, what=f"bundle {dims} {kind} min={minimum} {path}")


def test_bundled_graph_csr(eg, ctx):
    import torch
    X, f = G.gmm_points(5000, seed=6)
    rp, ci = G.knn_csr(X, 10)
    o = O.bundle(O.csr(f, rp, ci), f)
    g = ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()),
                    flags=eg.EG_BUNDLE)
    assert_graph_equal(g, o, what="bundle csr")


@pytest.mark.parametrize("dims,kind,minimum", [([300], "normal", False), ([64, 48], "normal", False),
                                               ([40, 33, 29], "normal", False), ([40, 33, 29], "int", True),
                                               ([9, 8, 7, 6], "normal", False)])
def test_simplify(eg, ctx, dims, kind, minimum):
    """eg_simplify (reading L20) against the oracle's literal lazy cancellation."""
    import math
    import torch
    f, _ = G.random_field(dims, 61 + len(dims), kind)
    o = O.grid(f, dims, minimum=minimum)
    fl = eg.EG_NODE_VALUES | (eg.EG_MINIMUM if minimum else 0)
    ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=fl)
    for tau in (0.0, 0.3, 1.0, math.inf):
        s = ctx.simplify(tau)
        e = O.simplify(o, f, tau, minimum=minimum)
        for name, a, b in [("maxima", s.maxima, e.maxima), ("saddles", s.saddles, e.saddles),
                           ("saddle_beta", s.saddle_beta, e.saddle_beta), ("arcs", s.arcs, e.arcs)]:
            assert first_diff(a, b) is None, f"{name} tau={tau}: {first_diff(a, b)}"


@pytest.mark.parametrize("k", [2, 3, 5])
def test_node_values_with_virtual_parts(eg, ctx, k):
    """EG_NODE_VALUES (bit 8) and EG_VIRTUAL_PARTS(k) (bits 16-31) are
    independent flag fields (odd k used to switch node values on)."""
    import torch
    f, dims = G.random_field([23, 19, 17], 70 + k, "normal")
    o = O.grid(f, dims)
    g = ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_NODE_VALUES | eg.EG_VIRTUAL_PARTS(k))
    assert_graph_equal(g, o, what=f"node values + {k} virtual parts")
    s = ctx.simplify(0.25)
    e = O.simplify(o, f, 0.25)
    assert np.array_equal(s.maxima, e.maxima) and np.array_equal(s.arcs, e.arcs)
    # a rank type without node values but with virtual parts of an even / odd count
    g = ctx.compute(torch.from_numpy(f.astype(np.float64)).cuda(), dims=dims)
    assert_graph_equal(g, o, what="float64 rank image")


def test_simplify_csr_and_state(eg, ctx):
    import torch
    X, f = G.gmm_points(4000, seed=8)
    rp, ci = G.knn_csr(X, 10)
    o = O.csr(f, rp, ci)
    ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()),
                flags=eg.EG_NODE_VALUES)
    s = ctx.simplify(0.5)
    e = O.simplify(o, f, 0.5)
    assert np.array_equal(s.maxima, e.maxima) and np.array_equal(s.arcs, e.arcs)
    ctx.compute(torch.from_numpy(f).cuda(), csr=(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()))
    with pytest.raises(Exception):
        ctx.simplify(0.5)                   # the last compute kept no node values


@pytest.mark.parametrize("tdtype", ["float16", "bfloat16", "uint8", "int8", "int16", "uint16"])
@pytest.mark.parametrize("dims", [[64, 48], [40, 33, 29]])
def test_other_dtypes(eg, ctx, tdtype, dims):
    """eg_compute_typed (reading L21): exact float32 images -> identical graphs."""
    import torch
    if not hasattr(torch, tdtype):
        pytest.skip(f"torch has no {tdtype}")
    dt = getattr(torch, tdtype)
    rng = np.random.default_rng(len(dims) * 7 + len(tdtype))
    N = int(np.prod(dims))
    if dt.is_floating_point:
        t = torch.from_numpy(rng.standard_normal(N).astype(np.float32)).to(dt)
    else:
        info = torch.iinfo(dt)
        lo, hi = max(info.min, -300), min(info.max, 300)     # ties on purpose
        t = torch.from_numpy(rng.integers(lo, hi + 1, N)).to(dt)
    f = t.to(torch.float32).numpy()                           # the exact float32 image
    o = O.grid(f, dims)
    g = ctx.compute(t.cuda(), dims=dims, flags=eg.EG_CHECK_NAN)
    assert_graph_equal(g, o, what=f"{tdtype} {dims}")


def _rank_image(x):
    """SoS rank of every vertex (value, then index) as float32 -- exact for the
    test sizes; the extremum graph depends on the field only through this
    order (SURVEY 8(c) order invariance, pinned in
    test_oracle_pins.py)."""
    r = np.empty(len(x), dtype=np.int64)
    r[np.argsort(x, kind="stable")] = np.arange(len(x))
    return r.astype(np.float32)


def _wide_field(tdtype, N, rng):
    """Values f32 cannot tell apart, plus exact ties."""
    if tdtype == "float64":
        x = 1.0 + 1e-12 * rng.standard_normal(N)
    elif tdtype == "int32":
        x = rng.integers(-100, 100, N) * 16777259 + rng.integers(0, 3, N)
    elif tdtype == "uint32":
        x = (np.uint64(0xFFFFFF00) + rng.integers(0, 200, N).astype(np.uint64)).astype(np.uint32)
    elif tdtype == "int64":
        x = (rng.integers(-50, 50, N) << 40) + rng.integers(0, 3, N)
    else:
        x = (np.uint64(1) << np.uint64(63)) + rng.integers(0, 40, N).astype(np.uint64) * np.uint64(1 << 20)
    x = np.asarray(x).astype(getattr(np, tdtype))
    x[rng.integers(0, N, N // 8)] = x[rng.integers(0, N, N // 8)]      # exact ties
    if tdtype == "float64":
        x[::11], x[5::11] = -0.0, 0.0                                  # -0 ties with +0 (reading L2)
    return x


@pytest.mark.parametrize("tdtype", ["float64", "int32", "uint32", "int64", "uint64"])
@pytest.mark.parametrize("dims,path", [([64, 48], 0), ([40, 33, 29], 0), ([40, 33, 29], "generic")])
def test_rank_dtypes(eg, ctx, tdtype, dims, path):
    """eg_compute_typed, types without an exact float32 image (reading L22):
    the graph is that of the type's own order -- the oracle run on the rank
    image -- where a float32 cast would merge values."""
    import torch
    if not hasattr(torch, tdtype):
        pytest.skip(f"torch has no {tdtype}")
    rng = np.random.default_rng(len(dims) * 11 + len(tdtype))
    N = int(np.prod(dims))
    x = _wide_field(tdtype, N, rng)
    assert len(np.unique(x.astype(np.float32))) < len(np.unique(x))   # the cast would lose order
    try:
        t = torch.from_numpy(x).cuda()
    except (TypeError, RuntimeError) as e:
        pytest.skip(f"torch cannot move {tdtype} to the device: {e}")
    fr = _rank_image(x)
    for minimum in (False, True):
        o = O.grid(fr, dims, minimum=minimum)
        g = ctx.compute(t, dims=dims, flags=_flags(eg, path, eg.EG_CHECK_NAN | (eg.EG_MINIMUM if minimum else 0)))
        assert_graph_equal(g, o, what=f"{tdtype} {dims} {path} minimum={minimum}")


def test_rank_dtype_errors(eg, ctx):
    """float64 NaN -> EG_ERR_NAN; EG_NODE_VALUES with a rank type -> unsupported."""
    import torch
    x = np.linspace(0.0, 1.0, 64 * 48)
    x[100] = np.nan
    with pytest.raises(eg.EgError) as e:
        ctx.compute(torch.from_numpy(x).cuda(), dims=[64, 48], flags=eg.EG_CHECK_NAN)
    assert e.value.status == 2
    with pytest.raises(eg.EgError) as e:
        ctx.compute(torch.from_numpy(np.arange(64 * 48, dtype=np.int64)).cuda(), dims=[64, 48],
                    flags=eg.EG_NODE_VALUES)
    assert e.value.status == 7
    g = ctx.compute(torch.from_numpy(np.arange(64 * 48, dtype=np.int64)).cuda(), dims=[64, 48])
    assert list(g.maxima) == [64 * 48 - 1] and len(g.saddles) == 0      # context still usable


def test_rank_dtype_beyond_2p24(eg, ctx):
    """The rank image past 2^24 vertices (ranks no float32 integer holds; the
    bit-pattern image stays exact): a float64 copy of a float32 field has the
    same SoS order, so its graph equals the float32 path's (itself pinned to
    the oracle by the sampled C3 checks) -- also for an int64 rank-equivalent."""
    import torch
    dims = [320, 256, 256]                         # 20,971,520 > 2^24 vertices
    f = torch.randn(int(np.prod(dims)), generator=torch.Generator().manual_seed(5)).to(torch.float32)
    f[::13] = 0.25                                # ties
    a = ctx.compute(f.cuda(), dims=dims)
    la = a.labels.cpu().numpy().copy()
    order = np.argsort(f.numpy(), kind="stable")
    rank = np.empty(len(order), np.int64)
    rank[order] = np.arange(len(order))
    for t in (f.to(torch.float64), torch.from_numpy(rank * 3 - 7)):
        b = ctx.compute(t.cuda(), dims=dims)
        assert_graph_equal(b, a, labels=False, what=f"rank image {t.dtype}")
        assert np.array_equal(b.labels.cpu().numpy(), la)


def test_deferred_graph(eg, ctx):
    """EG_NO_GRAPH_D2H: the graph stays in HBM after eg_compute and the first
    eg_get_graph / eg_get_graph32 / eg_get_raw_arcs copies it (one process) --
    the same graph as an eager compute, on the tiled, generic and CSR paths."""
    import torch
    f, dims = G.c2_gaussians_noise(n=48, seed=5, k=6)
    o = O.grid(f, dims)
    t = torch.from_numpy(f).cuda()
    for extra in (0, eg.EG_GRAPH32, eg.EG_FORCE_GENERIC, eg.EG_RAW_ARCS, eg.EG_VIRTUAL_PARTS(2)):
        g0 = ctx.compute(t, dims=dims, flags=eg.EG_NO_GRAPH_D2H | extra)
        assert len(g0.arcs) == 0                  # nothing copied by compute itself
        g = ctx.graph()
        assert_graph_equal(g, o, raw=bool(extra & eg.EG_RAW_ARCS), what=f"deferred {extra}")
        assert_graph_equal(ctx.graph(), o, what=f"deferred {extra} (second request)")
    X, fc = G.gmm_points(4000, seed=4)
    rp, ci = G.knn_csr(X, 10)
    csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    ctx.compute(torch.from_numpy(fc).cuda(), csr=csr, flags=eg.EG_NO_GRAPH_D2H | eg.EG_GRAPH32)
    assert_graph_equal(ctx.graph(), O.csr(fc, rp, ci), what="deferred csr")
    # arc geometry stays on the device too; eg_get_arc_paths copies it
    eager = ctx.compute(t, dims=dims, flags=eg.EG_ARC_PATHS)
    ctx.compute(t, dims=dims, flags=eg.EG_ARC_PATHS | eg.EG_NO_GRAPH_D2H)
    lazy = ctx.graph()
    assert np.array_equal(lazy.arc_paths[0], eager.arc_paths[0]) and np.array_equal(lazy.arc_paths[1], eager.arc_paths[1])
    assert np.array_equal(lazy.raw_arcs, eager.raw_arcs)


@pytest.mark.parametrize("split", ["0", "2", "3"])
@pytest.mark.parametrize("dims", [[64, 48, 80], [40, 37, 70], [33, 17, 33]])
def test_face_split_label_pass(eg, ctx, split, dims, monkeypatch):
    """The one-slab label pass split by tile faces (EG_FIN_SPLIT: one pass /
    z-face planes then the rest / z faces, y faces, rest): several tile layers
    in z and y, ragged last tiles, a turbulence field whose paths cross many
    tiles -- identical to the oracle either way."""
    import torch
    monkeypatch.setenv("EG_FIN_SPLIT", split)
    t3, d3 = G.turbulence(max(dims), seed=11, device="cpu", kc_div=8)
    f = t3.numpy().reshape(max(dims), max(dims), max(dims))[:dims[2], :dims[1], :dims[0]].ravel().copy()
    o = O.grid(f, dims)
    assert_graph_equal(ctx.compute(torch.from_numpy(f).cuda(), dims=dims), o, what=f"split {split} {dims}")


@pytest.mark.parametrize("tdtype", ["float64", "int32", "uint32", "int64", "uint64"])
@pytest.mark.parametrize("dims,path", [([64, 48], 0), ([40, 33, 29], 0), ([9, 8, 7, 6], "generic")])
def test_exact_image_dtypes(eg, ctx, tdtype, dims, path):
    """eg_compute_typed on wide types whose every value is exactly a float32
    (float32 data stored as float64, integers below 2^24, with ties): the
    library takes the plain cast instead of the rank sort; the graph is still
    the type's own -- equal to the oracle on the rank image, and on the values."""
    import torch
    if not hasattr(torch, tdtype):
        pytest.skip(f"torch has no {tdtype}")
    rng = np.random.default_rng(len(dims) * 7 + len(tdtype))
    N = int(np.prod(dims))
    if tdtype == "float64":
        x = rng.standard_normal(N).astype(np.float32).astype(np.float64)
        x[::5] = x[1::5][: len(x[::5])]              # ties
    else:
        x = rng.integers(0, 1 << 20, N).astype(tdtype)
        x[::3] = 7                                    # ties
    try:
        t = torch.from_numpy(x).cuda()
    except (TypeError, RuntimeError) as e:
        pytest.skip(f"torch cannot move {tdtype} to the device: {e}")
    fr = _rank_image(x)
    for minimum in (False, True):
        o = O.grid(fr, dims, minimum=minimum)
        o2 = O.grid(x.astype(np.float32), dims, minimum=minimum)
        assert np.array_equal(o.arcs, o2.arcs) and np.array_equal(o.label, o2.label)
        g = ctx.compute(t, dims=dims, flags=_flags(eg, path, eg.EG_CHECK_NAN | (eg.EG_MINIMUM if minimum else 0)))
        assert_graph_equal(g, o, what=f"{tdtype} {dims} {path} minimum={minimum}")
