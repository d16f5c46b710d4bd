"""Pins for the CPU oracle (oracle/eg_oracle.c) against things other than itself.

Each test names what it is pinned to: a value printed in the paper or SPEC, a
closed form, an invariant, a textbook special case, or the literal brute force
in oracle/brute.py (which takes the BFS / Alg. 2 route instead of union-find /
memoised walks).  None of these tests needs a GPU.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import eg_inputs as G
import oracle as O
from oracle import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tiny_examples.json")


def _coords(v, dims):
    c = []
    for d in dims:
        c.append(v % d)
        v //= d
    return c


def _on_boundary(v, dims):
    return any(c in (0, d - 1) for c, d in zip(_coords(v, dims), dims))


# ----------------------------------------------------------- Alg. 1 / links


def test_grid_adjacency_spec_examples():
    # SPEC S:45-48 (Alg. 1; p == q excluded, reading L6)
    assert O.grid_adjacent((0, 0, 0), (1, 1, 0))
    assert not O.grid_adjacent((1, 0), (0, 1))
    assert not O.grid_adjacent((2, 2, 2), (2, 2, 2))
    assert O.grid_adjacent((5, 5), (4, 4))
    assert not O.grid_adjacent((0, 0), (2, 0))         # |d| = 2 is not an edge
    with pytest.raises(ValueError):
        O.grid_adjacent((0, 0), (0, 0, 0))


def test_grid_adjacency_matches_brute_exhaustively():
    # every pair of points in {0,1,2}^3: C oracle == literal Python Alg. 1
    pts = list(itertools.product(range(3), repeat=3))
    for p in pts:
        for q in pts:
            assert O.grid_adjacent(p, q) == brute.grid_adjacency(p, q)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_interior_link_size_and_sphere(n):
    # "the number of edges incident on a vertex ... namely 2 x (2^n - 1)".
    # Link-edge counts 0, 6, 36, 150, 540, 1806 (S:64-65 for n = 2, 3).
    # The interior link's clique complex is an (n-1)-sphere: chi = 1 + (-1)^(n-1).
    dims = [3] * n
    v = (3 ** n - 1) // 2
    nl, ne, chi = O.grid_link_stats(dims, v)
    assert nl == 2 * (2 ** n - 1)
    assert ne == {1: 0, 2: 6, 3: 36, 4: 150, 5: 540, 6: 1806}[n]
    assert chi == 1 + (-1) ** (n - 1)


def test_link_truncation_and_brute():
    # 2D corner vertex has 3 neighbours; every vertex of small grids:
    # oracle link == brute link (Alg. 1 against every vertex of the grid).
    assert len(O.grid_link([4, 4], 0)) == 3
    assert len(O.grid_link([4, 4], 5)) == 6           # interior 2D (P:99 caption)
    assert len(O.grid_link([4, 4, 4], 21)) == 14      # interior 3D
    for dims in ([5], [4, 3], [3, 4, 3], [2, 3, 2, 2]):
        dom = brute.grid_domain(dims)
        for v in range(int(np.prod(dims))):
            assert list(O.grid_link(dims, v)) == sorted(dom.neighbours(v))


def test_link_symmetry():
    # u in Lk(v) <=> v in Lk(u)
    dims = [4, 3, 3]
    n = int(np.prod(dims))
    links = [set(O.grid_link(dims, v)) for v in range(n)]
    for v in range(n):
        for u in links[v]:
            assert v in links[u]


# ----------------------------------------------------------------- golden


def _check_graph(g, case):
    assert list(g.maxima) == case["maxima"]
    assert [[int(s), int(b)] for s, b in zip(g.saddles, g.saddle_beta)] == case["saddles"]
    assert g.arcs.tolist() == case["arcs"]
    assert list(g.label) == case["labels"]


def test_golden_examples():
    cases = json.load(open(GOLDEN))["cases"]
    for case in cases:
        g = O.grid(np.array(case["f"], np.float32), case["dims"])
        _check_graph(g, case)
        b = brute.grid_graph(np.array(case["f"], np.float32), case["dims"])
        assert b["arcs"].tolist() == case["arcs"]


# --------------------------------------------------------- special cases


@pytest.mark.parametrize("dims", [[7], [5, 4], [4, 3, 5], [3, 3, 3, 2]])
def test_constant_field(dims):
    # SoS makes a constant field the index order: exactly one maximum (N-1),
    # no saddles (S:198 one maximum), every label N-1.
    n = int(np.prod(dims))
    g = O.grid(np.zeros(n, np.float32), dims)
    assert list(g.maxima) == [n - 1]
    assert len(g.saddles) == 0
    assert (g.label == n - 1).all()


@pytest.mark.parametrize("seed", range(6))
def test_1d_textbook(seed):
    # n = 1: the link is {v-1, v+1} with no link edges, so beta0+ = number of
    # higher neighbours: maxima = local maxima, saddles = interior local minima
    # with beta0+ = 2; arcs climb monotonically left and right (textbook
    # peak/valley analysis).  Ties included via small integer values.
    rng = np.random.default_rng(seed)
    n = 40
    f = rng.integers(0, 6, size=n).astype(np.float32)
    hi = lambda a, b: f[a] > f[b] or (f[a] == f[b] and a > b)   # noqa: E731
    g = O.grid(f, [n])
    nbrs = lambda v: [u for u in (v - 1, v + 1) if 0 <= u < n]   # noqa: E731
    maxima = [v for v in range(n) if all(hi(v, u) for u in nbrs(v))]
    valleys = [v for v in range(1, n - 1) if hi(v - 1, v) and hi(v + 1, v)]

    def climb(v, step):
        while 0 <= v + step < n and hi(v + step, v):
            v += step
        return v

    def label(v):
        while True:
            ups = [u for u in nbrs(v) if hi(u, v)]
            if not ups:
                return v
            v = max(ups, key=lambda u: (f[u], u))

    assert list(g.maxima) == maxima
    assert list(g.saddles) == valleys and (g.saddle_beta == 2).all()
    exp_arcs = []
    for s in valleys:
        ms = sorted([label(climb(s - 1, -1)), label(climb(s + 1, +1))])
        for m in sorted(set(ms)):
            exp_arcs.append([s, m, ms.count(m)])
    assert g.arcs.tolist() == exp_arcs
    assert list(g.label) == [label(v) for v in range(n)]


@pytest.mark.parametrize("seed", range(5))
def test_2d_saddles_are_hexagon_runs(seed):
    # Banchoff: for an interior 2D vertex the link is the hexagon
    # (1,0),(1,1),(0,1),(-1,0),(-1,-1),(0,-1) (Fig. 2c); beta0+ is the
    # number of maximal runs of upper vertices around it (cycle), 0 if none.
    f, dims = G.random_field([9, 8], seed, "int", levels=3)
    g = O.grid(f, dims)
    W = dims[0]
    ring = [(1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1)]
    for y in range(1, dims[1] - 1):
        for x in range(1, W - 1):
            v = x + W * y
            up = []
            for dx, dy in ring:
                u = (x + dx) + W * (y + dy)
                up.append(f[u] > f[v] or (f[u] == f[v] and u > v))
            if all(up):
                runs = 1
            else:
                runs = sum(1 for i in range(6) if up[i] and not up[i - 1])
            assert g.beta[v] == runs, (x, y)


# -------------------------------------------------------------- Euler pin


@pytest.mark.parametrize("dims,seed", [([9, 7], 0), ([12, 12], 1), ([5, 6, 4], 2), ([6, 6, 6], 3),
                                       ([4, 3, 4, 3], 4)])
def test_euler_invariant_tie_heavy(dims, seed):
    # sum_v (1 - chi(Lk+(v))) = chi(box) = 1 for any injective order (Banchoff;
    # SURVEY 8(c) Euler pin), on tie-heavy integer fields (SoS decides).
    f, _ = G.random_field(dims, seed, "int", levels=4)
    assert O.grid_euler(f, dims) == 1


@pytest.mark.parametrize("seed", range(4))
def test_euler_2d_reduces_to_beta(seed):
    # In 2D the upper link is a union of paths (chi = beta0+) unless it is the
    # whole interior hexagon (chi = 0, a minimum): so
    # sum_v (1 - beta0+(v)) + #{interior v whose link is all upper} = 1.
    # This pins the oracle's union-find beta0+ (not chi) to the Euler number.
    f, dims = G.random_field([11, 9], seed, "int", levels=4)
    g = O.grid(f, dims)
    W = dims[0]
    full = 0
    for v in range(len(f)):
        if _on_boundary(v, dims):
            continue
        link = O.grid_link(dims, v)
        if all(f[u] > f[v] or (f[u] == f[v] and u > v) for u in link):
            full += 1
    assert int((1 - g.beta.astype(np.int64)).sum()) + full == 1


# --------------------------------------------------------- closed forms


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("sigma", [3.0, 4.0, 5.0])
def test_c1_gaussians_have_exactly_8_maxima(seed, sigma):
    # K well-separated Gaussians => exactly K maxima (SURVEY 8(c) pin; C1 recipe)
    f, dims = G.c1_gaussians(seed, sigma)
    g = O.grid(f, dims)
    assert len(g.maxima) == 8
    assert O.grid_euler(f, dims) == 1


@pytest.mark.slow
def test_lattice_gaussians_3d_32_maxima():
    # C2' at 128^3: a 4x4x2 lattice of well-separated Gaussians has 32 maxima
    f, dims = G.lattice_gaussians(128, seed=0)
    g = O.grid(f, dims)
    assert len(g.maxima) == 32


@pytest.mark.parametrize("p,q,seed", [(2, 4, 1), (4, 4, 7), (4, 3, 2), (2, 8, 3)])
def test_sincos_counts_and_arcs(p, q, seed):
    # f = sin x cos y with the domain edges pi/4 (+eps h) from every critical
    # line: interior saddles 4p^2 (all beta0+ = 2), interior maxima 2p^2,
    # boundary maxima 2p+1, boundary saddles 2p; every interior
    # saddle at (k pi, pi/2 + m pi) whose two analytic maxima (the diagonal
    # neighbours with f = +1) are interior has arcs to exactly the two discrete
    # maxima within one cell of them.
    f, dims, x0, y0, h = G.sincos(p, q, seed)
    g = O.grid(f, dims)
    N = dims[0]
    imax = [m for m in g.maxima if not _on_boundary(m, dims)]
    isad = [s for s in g.saddles if not _on_boundary(s, dims)]
    assert len(isad) == 4 * p * p
    assert len(imax) == 2 * p * p
    assert len(g.maxima) - len(imax) == 2 * p + 1
    assert len(g.saddles) - len(isad) == 2 * p
    assert (g.saddle_beta == 2).all()
    xy = lambda v: (x0 + h * (v % N), y0 + h * (v // N))   # noqa: E731
    lo, hi_ = x0, x0 + h * (N - 1)

    def discrete_max_near(ax, ay):
        cand = [m for m in g.maxima if abs(xy(m)[0] - ax) <= h and abs(xy(m)[1] - ay) <= h]
        assert len(cand) == 1
        return int(cand[0])

    arcs = {}
    for s, m, c in g.arcs.tolist():
        arcs.setdefault(s, []).append((m, c))
    checked = 0
    for s in isad:
        sx, sy = xy(s)
        k = round(sx / math.pi)
        mm = round((sy - math.pi / 2) / math.pi)
        cx, cy = k * math.pi, math.pi / 2 + mm * math.pi
        assert abs(sx - cx) <= h and abs(sy - cy) <= h
        tops = [(cx + dx, cy + dy) for dx in (-math.pi / 2, math.pi / 2) for dy in (-math.pi / 2, math.pi / 2)
                if math.sin(cx + dx) * math.cos(cy + dy) > 0.5]
        assert len(tops) == 2
        if not all(lo + h < tx < hi_ - h and lo + h < ty < hi_ - h for tx, ty in tops):
            continue
        exp = sorted((discrete_max_near(tx, ty), 1) for tx, ty in tops)
        assert sorted(arcs[s]) == exp
        checked += 1
    assert checked >= (2 * p - 2) ** 2


def _scan_1d(h):
    """Textbook 1D extrema scan of a tie-free profile: (#local maxima incl.
    endpoints higher than their single neighbour, #interior local minima)."""
    h = np.asarray(h, np.float64)
    n = len(h)
    M = sum(1 for i in range(n) if all(h[i] > h[j] for j in (i - 1, i + 1) if 0 <= j < n))
    S = sum(1 for i in range(1, n - 1) if h[i] < h[i - 1] and h[i] < h[i + 1])
    return M, S


def _product_rule(profiles):
    MS = [_scan_1d(p) for p in profiles]
    n_max = int(np.prod([m for m, _ in MS]))
    n_sad = sum(MS[i][1] * int(np.prod([MS[j][0] for j in range(len(MS)) if j != i])) for i in range(len(MS)))
    return n_max, n_sad


@pytest.mark.parametrize("n", [7, 8])
def test_interior_link_size_high_dim(n):
    # P:112's 2 x (2^n - 1) incident edges for n = 7, 8 (254, 510 link vertices);
    # link-edge count = sum over link vertices of their link-link degree / 2,
    # where +d ~ +d' iff one mask contains the other (likewise -e), and
    # +d ~ -e iff the masks are disjoint (Alg. 1 on offsets):
    # a closed form counted here independently of the oracle.
    dims = [3] * n
    v = (3 ** n - 1) // 2
    nl, ne, _ = O.grid_link_stats(dims, v)
    assert nl == 2 * (2 ** n - 1)
    M = 1 << n
    same = sum(1 for a in range(1, M) for b in range(1, M) if a != b and (a & b) in (a, b))   # ordered pairs
    cross = sum(1 for a in range(1, M) for b in range(1, M) if (a & b) == 0)
    assert ne == same + cross      # (2 * same / 2) over the +/- halves, + cross edges


@pytest.mark.parametrize("dims,seed", [([40, 40], 0), ([40, 40], 1), ([24, 24, 24], 2), ([24, 24, 24], 3),
                                       ([12, 12, 12, 12], 4), ([7, 7, 7, 7, 7], 5),
                                       ([3, 4, 3, 3, 4, 3, 3], 6), ([3, 2, 3, 2, 3, 2, 3, 2], 7)])
def test_separable_product_rule(dims, seed):
    # tie-free separable f = sum_i h_i(x_i): #maxima = prod M_i and
    # #(n-1)-saddles = sum_i S_i prod_{j != i} M_j, all beta0+ = 2.
    rng = np.random.default_rng(seed)
    profiles = [rng.standard_normal(d) for d in dims]
    f, _ = G.separable(profiles)
    g = O.grid(f, dims)
    n_max, n_sad = _product_rule(profiles)
    assert len(g.maxima) == n_max
    assert len(g.saddles) == n_sad
    assert (g.saddle_beta == 2).all()


def test_schwefel_profile_counts():
    # C4 pin: the 32-sample Schwefel profile on [-500, 500] has M = 7 local
    # maxima and S = 6 interior minima, so C4 has 7^5 = 16,807 maxima and
    # 5 * 6 * 7^4 = 72,030 saddles by the product rule.
    x = -500.0 + np.arange(32) * 1000.0 / 31
    prof = -(x * np.sin(np.sqrt(np.abs(x))))
    assert _scan_1d(prof) == (7, 6)
    assert _product_rule([prof] * 5) == (16807, 72030)


@pytest.mark.parametrize("dims", [[12, 12, 12, 12, 12], [9, 10, 11, 12, 13]])
def test_schwefel_reduced_5d_product_rule(dims):
    # the C4 generator itself (float64 -> f32, slowest-axis-first sum) at
    # reduced resolution obeys the product rule on its own 1D profiles.
    f, _ = G.schwefel(dims)
    g = O.grid(f, dims)
    profiles = []
    for D in dims:
        x = -500.0 + np.arange(D) * 1000.0 / (D - 1)
        profiles.append(-(x * np.sin(np.sqrt(np.abs(x)))))
    assert (len(g.maxima), len(g.saddles)) == _product_rule(profiles)
    assert (g.saddle_beta == 2).all()


@pytest.mark.parametrize("dims", [[32, 32, 32], [24, 24, 24, 24], [16, 16, 16, 16, 16]])
def test_sumcos_interior_closed_form(dims):
    # f = sum cos x_i with edges at pi/2 from the critical lines: interior
    # maxima = p^n and interior (n-1)-saddles = n q p^(n-1) with p analytic
    # maxima and q analytic minima per axis strictly inside (SURVEY 8(c):
    # n p^n when q = p); totals follow the product rule.
    f, _, eps, h = G.sumcos(dims, seed=5)
    g = O.grid(f, dims)
    n = len(dims)
    ps, qs = [], []
    for ax, D in enumerate(dims):
        x0 = -math.pi / 2 + eps[ax] * h
        x1 = x0 + h * (D - 1)
        ps.append(sum(1 for k in range(-4, 40) if x0 < 2 * k * math.pi < x1))          # analytic maxima
        qs.append(sum(1 for k in range(-4, 40) if x0 < (2 * k + 1) * math.pi < x1))    # analytic minima
    assert len(set(ps)) == 1 and len(set(qs)) == 1
    p, q = ps[0], qs[0]
    imax = [m for m in g.maxima if not _on_boundary(m, dims)]
    isad = [s for s in g.saddles if not _on_boundary(s, dims)]
    assert len(imax) == p ** n
    assert len(isad) == n * q * p ** (n - 1)        # = n p^n when q = p (the 32^5 C4' case)
    profiles = [np.cos(-math.pi / 2 + eps[ax] * h + h * np.arange(D)) for ax, D in enumerate(dims)]
    assert (len(g.maxima), len(g.saddles)) == _product_rule(profiles)


# ---------------------------------------------------------- brute force


def _assert_same(g, b):
    assert np.array_equal(g.ptr, b["ptr"])
    assert np.array_equal(g.beta, b["beta"])
    assert np.array_equal(g.label, b["label"])
    assert np.array_equal(g.maxima, b["maxima"])
    assert np.array_equal(g.saddles, b["saddles"])
    assert np.array_equal(g.saddle_beta, b["saddle_beta"])
    assert g.arcs.tolist() == b["arcs"].tolist()


def test_brute_all_binary_3x3():
    # exhaustive: every field on 3x3 with values {0, 1} (ties everywhere)
    dom = brute.grid_domain([3, 3])
    for bits in range(512):
        f = np.array([(bits >> i) & 1 for i in range(9)], np.float32)
        _assert_same(O.grid(f, [3, 3]), brute.extremum_graph(dom, f))


def test_brute_sampled_4level_3x3():
    dom = brute.grid_domain([3, 3])
    rng = np.random.default_rng(0)
    for _ in range(1500):
        f = rng.integers(0, 4, size=9).astype(np.float32)
        _assert_same(O.grid(f, [3, 3]), brute.extremum_graph(dom, f))


@pytest.mark.parametrize("dims,kind,count", [([6, 5], "int", 30), ([4, 4, 3], "int", 20), ([8, 8, 8], "normal", 6),
                                             ([8, 8, 8], "int", 4), ([6, 6, 6, 6], "normal", 2),
                                             ([4, 3, 3, 3], "int", 4), ([3, 3, 2, 2, 2], "int", 4),
                                             ([5, 4], "signed_zero", 20)])
def test_brute_random(dims, kind, count):
    # random 8^3 and 6^4 fields against an independent BFS oracle
    dom = brute.grid_domain(dims)
    for s in range(count):
        f, _ = G.random_field(dims, 1000 + s, kind)
        _assert_same(O.grid(f, dims), brute.extremum_graph(dom, f))


def test_brute_paths_are_monotone_and_adjacent():
    # every traced path is monotone under SoS and consecutive
    # vertices are adjacent; sum of beta0+ over saddles = #paths.
    f, dims = G.random_field([7, 6, 5], 3, "int", levels=3)
    b = brute.grid_graph(f, dims)
    n_paths = 0
    for s, P in b["paths"].items():
        for p in P:
            n_paths += 1
            assert len(p) >= 2
            for a, c in zip(p, p[1:]):
                assert brute.grid_adjacency(brute.coords(a, dims), brute.coords(c, dims))
                assert brute.higher(f, c, a)
    assert n_paths == int(b["saddle_beta"].sum())


# ----------------------------------------------------------- invariants


@pytest.mark.parametrize("seed", range(3))
def test_label_invariants(seed):
    f, dims = G.c2_gaussians_noise(n=24, seed=seed, k=6, eta=1e-3)
    g = O.grid(f, dims)
    mx = set(g.maxima.tolist())
    assert all(g.label[m] == m for m in mx)
    assert np.array_equal(g.label, g.label[g.ptr])
    assert set(np.unique(g.label).tolist()) <= mx
    assert (g.ptr[g.maxima] == g.maxima).all()
    nonmax = np.setdiff1d(np.arange(len(f)), g.maxima)
    # the gradient goes strictly up
    up = (f[g.ptr[nonmax]] > f[nonmax]) | ((f[g.ptr[nonmax]] == f[nonmax]) & (g.ptr[nonmax] > nonmax))
    assert up.all()
    # P:477 "a little over twice": every saddle has >= 2 raw arcs
    assert len(g.raw_s) == int(g.saddle_beta.sum()) >= 2 * len(g.saddles)
    assert int(g.arc_mult.sum()) == int(g.saddle_beta.sum())
    # sampled walks (Alg. 2 from scratch) agree with the memoised labels
    for v in np.random.default_rng(seed).integers(0, len(f), 50):
        assert O.grid_walk(f, dims, int(v))[0] == g.label[v]
    for v in np.random.default_rng(seed).integers(0, len(f), 50):
        p, b, reps = O.grid_vertex(f, dims, int(v))
        assert p == g.ptr[v] and b == g.beta[v]


def test_order_invariance():
    # exact monotone maps leave every output unchanged: f -> 2f, f -> rank(f)
    f, dims = G.random_field([9, 8, 7], 11, "int", levels=5)
    g = O.grid(f, dims)
    g2 = O.grid((2 * f).astype(np.float32), dims)
    order = np.lexsort((np.arange(len(f)), f))          # SoS order
    rank = np.empty(len(f), np.float32)
    rank[order] = np.arange(len(f), dtype=np.float32)
    g3 = O.grid(rank, dims)
    for h in (g2, g3):
        assert np.array_equal(g.label, h.label)
        assert np.array_equal(g.saddles, h.saddles)
        assert g.arcs.tolist() == h.arcs.tolist()


def test_signed_zero_and_nan():
    # reading L2: -0 == +0 (IEEE), so the tie goes to the index; NaN rejected
    f, dims = G.random_field([6, 5], 4, "signed_zero")
    canon = (f + np.float32(0)).astype(np.float32)      # -0 + 0 = +0
    a, b = O.grid(f, dims), O.grid(canon, dims)
    assert np.array_equal(a.label, b.label) and a.arcs.tolist() == b.arcs.tolist()
    bad = f.copy()
    bad[3] = np.nan
    with pytest.raises(O.OracleError):
        O.grid(bad, dims)


# ------------------------------------------------------------------- CSR


def _clique_chi(n, adj):
    """chi of the clique complex of a graph, counted globally (independent of
    the oracle): sum_k (-1)^(k+1) #k-cliques."""
    chi = 0

    def rec(cands, depth):
        nonlocal chi
        for i, a in enumerate(cands):
            chi += 1 if depth % 2 == 1 else -1
            rec([b for b in cands[i + 1:] if b in adj[a]], depth + 1)

    rec(list(range(n)), 1)
    return chi


@pytest.mark.parametrize("n,p,seed,kind", [(12, 0.3, 0, "normal"), (15, 0.4, 1, "int"), (20, 0.25, 2, "int"),
                                           (18, 0.5, 3, "normal")])
def test_csr_brute_and_euler(n, p, seed, kind):
    # L14: the CSR link is the induced subgraph on N(v).  Brute force (BFS +
    # Alg. 2) and the clique Euler identity sum_v (1 - chi(Lk+(v))) = chi(K(G)).
    row_ptr, col_idx = G.random_csr(n, p, seed)
    f, _ = G.random_field([n], seed, kind, levels=3)
    g = O.csr(f, row_ptr, col_idx)
    b = brute.csr_graph(f, row_ptr, col_idx)
    _assert_same(g, b)
    adj = [set(col_idx[row_ptr[v]:row_ptr[v + 1]].tolist()) for v in range(n)]
    assert O.csr_euler(f, row_ptr, col_idx) == _clique_chi(n, adj)


@pytest.mark.parametrize("dims,kind", [([6, 5], "int"), ([5, 4, 4], "normal"), ([4, 4, 3], "int"),
                                       ([3, 3, 3, 3], "int")])
def test_csr_equals_grid_on_freudenthal_graph(dims, kind):
    # L14: Freudenthal is a flag complex, so the CSR path on the Freudenthal
    # adjacency graph must equal the grid path exactly.
    f, _ = G.random_field(dims, 5, kind)
    row_ptr, col_idx = brute.freudenthal_csr(dims)
    a = O.grid(f, dims)
    c = O.csr(f, row_ptr, col_idx)
    assert np.array_equal(a.ptr, c.ptr) and np.array_equal(a.label, c.label)
    assert np.array_equal(a.saddles, c.saddles) and a.arcs.tolist() == c.arcs.tolist()


@pytest.mark.parametrize("dims,kind", [([6, 5], "int"), ([5, 4, 4], "normal")])
def test_csr_minimum_equals_grid_minimum(dims, kind):
    # L11 + L14: the minimum graph on the Freudenthal adjacency graph is the grid's
    f, _ = G.random_field(dims, 6, kind)
    row_ptr, col_idx = brute.freudenthal_csr(dims)
    a = O.grid(f, dims, minimum=True)
    c = O.csr(f, row_ptr, col_idx, minimum=True)
    assert np.array_equal(a.label, c.label) and np.array_equal(a.maxima, c.maxima)
    assert np.array_equal(a.saddles, c.saddles) and a.arcs.tolist() == c.arcs.tolist()


@pytest.mark.parametrize("n,p,seed,kind", [(40, 0.2, 1, "int"), (200, 0.05, 2, "normal")])
def test_csr_minimum_by_relabelled_reflection(n, p, seed, kind):
    # L11 on any graph: relabel every vertex i -> n-1-i and negate f; the
    # maximum graph of that, mapped back, is the minimum graph (the reversed
    # order's index tie-break is the relabelled index order).
    row_ptr, col_idx = G.random_csr(n, p, seed)
    f, _ = G.random_field([n], seed, kind, levels=3)
    adj = [sorted(n - 1 - int(u) for u in col_idx[row_ptr[n - 1 - i]:row_ptr[n - i]]) for i in range(n)]
    rp2 = np.zeros(n + 1, np.int64)
    rp2[1:] = np.cumsum([len(a) for a in adj])
    ci2 = np.array([u for a in adj for u in a], np.int32)
    g = np.ascontiguousarray(-f[::-1])
    mx = O.csr(g, rp2, ci2)
    mn = O.csr(f, row_ptr, col_idx, minimum=True)
    assert np.array_equal(mn.label, (n - 1 - mx.label)[::-1])
    assert np.array_equal(mn.maxima, np.sort(n - 1 - mx.maxima))
    assert np.array_equal(mn.saddles, np.sort(n - 1 - mx.saddles))
    back = sorted((n - 1 - int(s), n - 1 - int(m), int(k)) for s, m, k in mx.arcs.tolist())
    assert mn.arcs.tolist() == [list(a) for a in back]


def test_knn_small_sanity():
    # C5 recipe at 2,000 points: symmetric sorted CSR, degree >= k, Euler
    # identity on the kNN graph, sampled walks agree with labels.
    X, f = G.gmm_points(2000, seed=10)
    row_ptr, col_idx = G.knn_csr(X, 16)
    deg = np.diff(row_ptr)
    assert deg.min() >= 16
    for v in range(0, 2000, 97):
        nb = col_idx[row_ptr[v]:row_ptr[v + 1]]
        assert (np.diff(nb) > 0).all() and v not in nb
        for u in nb:
            assert v in col_idx[row_ptr[u]:row_ptr[u + 1]]
    g = O.csr(f, row_ptr, col_idx)
    assert int(g.arc_mult.sum()) == int(g.saddle_beta.sum())
    for v in range(0, 2000, 131):
        assert O.csr_walk(f, row_ptr, col_idx, v)[0] == g.label[v]


# ------------------------------------------- O10: the minimum graph (L11)
# Pinned independently of the reflection the GPU path uses: hand-derived 1-D
# valleys, the constant field under the reversed order, the Euler identity for
# the lower links, the separable product rule applied to minima, and the
# literal brute force run on -f with the tie order reversed (the max graph of
# -f under descending-index SoS is the min graph of f).

def test_minimum_graph_1d_golden():
    # [0, 5, 1, 9, 2]: minima 0, 2, 4; 1-saddles (interior maxima) 1 and 3,
    # each with one descending arc to either side; labels follow steepest descent
    f = np.array([0, 5, 1, 9, 2], np.float32)
    g = O.grid(f, [5], minimum=True)
    assert g.maxima.tolist() == [0, 2, 4]
    assert g.saddles.tolist() == [1, 3] and g.saddle_beta.tolist() == [2, 2]
    assert g.arcs.tolist() == [[1, 0, 1], [1, 2, 1], [3, 2, 1], [3, 4, 1]]
    assert g.label.tolist() == [0, 0, 2, 2, 4]


@pytest.mark.parametrize("dims", [[7], [5, 4], [4, 3, 5], [3, 3, 3, 2]])
def test_minimum_graph_constant_field(dims):
    # reversed SoS on a constant field: the LOWEST index is the only minimum
    N = int(np.prod(dims))
    g = O.grid(np.zeros(N, np.float32), dims, minimum=True)
    assert g.maxima.tolist() == [0] and len(g.saddles) == 0
    assert (g.label == 0).all()


@pytest.mark.parametrize("dims,seed", [([9, 7], 0), ([5, 6, 4], 2), ([4, 3, 4, 3], 4)])
def test_minimum_graph_euler(dims, seed):
    # sum_v (1 - chi(Lk-(v))) = chi(box) = 1 for the reversed order too (Banchoff)
    f, _ = G.random_field(dims, seed, "int")
    with O.reversed_order():
        assert O.grid_euler(f, dims) == 1


@pytest.mark.parametrize("dims,seed", [([40, 40], 0), ([24, 24, 24], 2), ([7, 7, 7, 7, 7], 5)])
def test_minimum_graph_product_rule(dims, seed):
    # tie-free separable f: #minima = prod m_i, #1-saddles = sum_i s_i prod_{j != i} m_j
    # with m_i, s_i the 1-D minima / interior maxima = the maximum rule on -h_i
    rng = np.random.default_rng(seed)
    profiles = [rng.standard_normal(d) for d in dims]
    f, _ = G.separable(profiles)
    g = O.grid(f, dims, minimum=True)
    n_min, n_sad = _product_rule([-p for p in profiles])
    assert (len(g.maxima), len(g.saddles)) == (n_min, n_sad)
    assert (g.saddle_beta == 2).all()


@pytest.mark.parametrize("dims,kind,seed", [([6, 5], "int", 1), ([4, 4, 3], "int", 2), ([5, 4, 3], "normal", 3)])
def test_minimum_graph_brute(dims, kind, seed):
    # brute force on the reflected, negated field: g[i] = -f[N-1-i] (point
    # reflection maps the Freudenthal grid to itself and reverses the index
    # order), mapped back by i -> N-1-i
    f, _ = G.random_field(dims, seed, kind)
    N = len(f)
    o = O.grid(f, dims, minimum=True)
    b = brute.grid_graph((-f[::-1]).copy(), dims)
    rev = lambda a: sorted(N - 1 - int(x) for x in a)
    assert o.maxima.tolist() == rev(b["maxima"])
    assert o.saddles.tolist() == rev(b["saddles"])
    assert o.label.tolist() == [N - 1 - int(b["label"][N - 1 - v]) for v in range(N)]
    assert sorted(map(tuple, o.arcs.tolist())) == sorted((N - 1 - s, N - 1 - m, c) for s, m, c in b["arcs"])


# ------------------------------------------- arc bundling

def test_bundle_two_bumps_two_saddles():
    # 2-D, two bumps (ids 7 and 9 on row 1 of a 5x3 grid) joined through
    # separate saddles on rows 0 and 2: only the highest saddle of each pair of
    # maxima survives bundling
    f = np.array([0.0, 0.1, 0.2, 2.0, 0.3,
                  0.4, 0.5, 9.0, -5.0, 8.0,
                  0.6, 0.7, 0.8, 3.0, 0.9], np.float32)
    g = O.grid(f, [5, 3])
    b = O.bundle(g, f)
    pairs = lambda gr: {s: sorted(m for s2, m, _ in gr.arcs.tolist() if s2 == s) for s in gr.saddles.tolist()}
    two = {s: ms for s, ms in pairs(g).items() if len(ms) == 2}
    assert len(two) >= 2                                   # the field really has parallel saddles
    for s, ms in pairs(b).items():
        assert s in pairs(g)
    kept2 = [s for s, ms in pairs(b).items() if len(ms) == 2]
    assert len({tuple(pairs(b)[s]) for s in kept2}) == len(kept2)   # one saddle per pair
    for s in kept2:                                        # the kept one is the highest of its pair
        rivals = [t for t, ms in two.items() if ms == pairs(b)[s]]
        assert max(rivals, key=lambda t: (f[t], t)) == s


@pytest.mark.parametrize("dims,seed", [([40, 30], 0), ([20, 20, 16], 1), ([9, 9, 8, 7], 2)])
def test_bundle_invariants(dims, seed):
    f, _ = G.random_field(dims, seed, "normal")
    g = O.grid(f, dims)
    b = O.bundle(g, f)
    # connectivity between maxima is unchanged (the Morse decomposition stays represented)
    conn = lambda gr: {tuple(sorted(set(m for s2, m, _ in gr.arcs.tolist() if s2 == s))) for s in gr.saddles.tolist()}
    assert conn(b) == conn(g)
    # one saddle per 2-maxima pair, idempotent, arcs belong to kept saddles
    ms = {}
    for s, m, _ in b.arcs.tolist():
        ms.setdefault(s, set()).add(m)
    twos = [tuple(sorted(v)) for v in ms.values() if len(v) == 2]
    assert len(twos) == len(set(twos))
    bb = O.bundle(b, f)
    assert np.array_equal(bb.saddles, b.saddles) and np.array_equal(bb.arcs, b.arcs)
    assert set(b.arc_s.tolist()) <= set(b.saddles.tolist())


# ------------------------------- persistence-directed cancellation

def test_simplify_1d_hand():
    # maxima 1 (5), 3 (9), 5 (7); saddles 2 (1), 4 (2); costs 4 and 5
    f = np.array([0, 5, 1, 9, 2, 7, 3], np.float32)
    g = O.grid(f, [7])
    assert g.maxima.tolist() == [1, 3, 5] and g.saddles.tolist() == [2, 4]
    s = O.simplify(g, f, 4.5)
    assert s.maxima.tolist() == [3, 5] and s.saddles.tolist() == [4]
    assert s.arcs.tolist() == [[4, 3, 1], [4, 5, 1]]
    assert O.simplify(g, f, 3.0).maxima.tolist() == [1, 3, 5]
    t = O.simplify(g, f, math.inf)
    assert t.maxima.tolist() == [3] and len(t.saddles) == 0


def _persistence_1d(h):
    """Textbook 0-dim persistence of superlevel sets of a 1-D sequence (elder
    rule, SoS ties by index): the persistence of every local maximum."""
    n = len(h)
    order = sorted(range(n), key=lambda i: (h[i], i), reverse=True)
    parent, birth, pers = {}, {}, {}
    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for i in order:
        parent[i] = i
        birth[i] = i
        for j in (i - 1, i + 1):
            if j in parent:
                a, b = find(i), find(j)
                if a == b:
                    continue
                young, old = (a, b) if (h[birth[a]], birth[a]) < (h[birth[b]], birth[b]) else (b, a)
                if birth[young] != i:
                    pers[birth[young]] = float(h[birth[young]]) - float(h[i])
                parent[young] = old
    root = find(order[0])
    pers[birth[root]] = math.inf
    return pers


@pytest.mark.parametrize("seed", range(5))
def test_simplify_matches_1d_persistence(seed):
    # in 1-D the lazy cancellation keeps exactly the maxima whose elder-rule
    # persistence exceeds tau
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(300).astype(np.float32)
    g = O.grid(f, [300])
    pers = _persistence_1d(f.astype(np.float64))
    for tau in (0.1, 0.5, 1.0, 2.0):
        s = O.simplify(g, f, tau)
        assert s.maxima.tolist() == sorted(m for m, p in pers.items() if p > tau and m in set(g.maxima.tolist()))


@pytest.mark.parametrize("dims,seed", [([40, 30], 0), ([16, 16, 12], 1)])
def test_simplify_invariants(dims, seed):
    f, _ = G.random_field(dims, seed, "normal")
    g = O.grid(f, dims)
    counts = [len(O.simplify(g, f, t).maxima) for t in (0.0, 0.2, 0.5, 1.0, 2.0, math.inf)]
    assert counts == sorted(counts, reverse=True)          # monotone in tau
    assert counts[-1] == 1                                   # a connected graph ends with one maximum
    z = O.simplify(g, f, -1.0)                               # nothing below a negative threshold
    assert np.array_equal(z.maxima, g.maxima) and np.array_equal(z.arcs, g.arcs)


# ------------------------------------------- big-domain harness (grid_parallel)
# The range entry points + O7 over the assembled gradient must reproduce the
# whole-domain run_all exactly (tie-heavy fields, several process counts,
# ranges that split saddles' neighbourhoods), so the full-size parity tests of
# C3 / C4 / C5 compare against the same oracle.

def _assert_identical(a, b):
    for k in ("ptr", "label", "beta", "maxima", "saddles", "saddle_beta", "arc_s", "arc_m", "arc_mult",
              "raw_s", "raw_rep", "raw_m"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k


@pytest.mark.parametrize("dims,kind,procs", [([64, 64], "int", 3), ([20, 17, 13], "normal", 4),
                                             ([9, 8, 7], "int", 1), ([5, 4, 5, 4, 3], "int", 2)])
def test_parallel_equals_whole(dims, kind, procs):
    f, _ = G.random_field(dims, 11, kind, levels=3)
    _assert_identical(O.grid_parallel(f, dims, procs=procs), O.grid(f, dims))


def test_parallel_equals_whole_csr():
    X, f = G.gmm_points(3000, seed=3)
    rp, ci = G.knn_csr(X, 16)
    _assert_identical(O.csr_parallel(f, rp, ci, procs=3), O.csr(f, rp, ci))
    rp, ci = G.random_csr(300, 0.05, 4)
    f, _ = G.random_field([300], 4, "int", levels=3)
    _assert_identical(O.csr_parallel(f, rp, ci, procs=2), O.csr(f, rp, ci))
