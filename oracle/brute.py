"""Literal brute force for tiny inputs -- TEST INFRASTRUCTURE ONLY.

A second, independent transcription of the paper used to pin the C oracle
(``oracle/eg_oracle.c``).  It deliberately takes the *other* routes the paper
describes, so that a mistake in one is unlikely to be repeated in the other:

* the link is found by testing Alg. 1 against EVERY vertex of the
  grid (no candidate offsets at all);
* beta0 of the upper link is computed by BFS ("typically computed by
  performing a BFS graph traversal"), not union-find;
* arcs come from Alg. 2 TraceGradientPaths run literally for every
  saddle, path lists included, with UpperLinkRep = highest vertex of each
  upper-link component;
* labels come from an un-memoised walk of every vertex.

Only for grids of at most a few thousand vertices / tiny CSR graphs.
"""
from __future__ import annotations

import itertools
from collections import deque

import numpy as np


def grid_adjacency(p, q) -> bool:
    """Alg. 1; p == q is not an edge (reading L6)."""
    if len(p) != len(q):
        raise ValueError("dimension mismatch")
    U = set()
    for pi, qi in zip(p, q):
        U.add(pi - qi)
    if U == {0}:
        return False
    return U <= {0, 1} or U <= {0, -1}


def coords(v, dims):
    c = []
    for d in dims:
        c.append(v % d)
        v //= d
    return tuple(c)


def higher(f, u, v) -> bool:
    """u is higher than v under simulated perturbation (reading L1)."""
    return bool(f[u] > f[v] or (f[u] == f[v] and u > v))


class _Domain:
    def __init__(self, n, neighbours, edge):
        self.n = n
        self.neighbours = neighbours   # v -> list of link vertices
        self.edge = edge               # (a, b) -> bool


def grid_domain(dims):
    n = int(np.prod(dims))
    cs = [coords(v, dims) for v in range(n)]
    links = [[u for u in range(n) if grid_adjacency(cs[v], cs[u])] for v in range(n)]
    return _Domain(n, lambda v: links[v], lambda a, b: grid_adjacency(cs[a], cs[b]))


def csr_domain(row_ptr, col_idx):
    n = len(row_ptr) - 1
    nb = [list(col_idx[row_ptr[v]:row_ptr[v + 1]]) for v in range(n)]
    sets = [set(x) for x in nb]
    return _Domain(n, lambda v: nb[v], lambda a, b: b in sets[a])


def upper_components(dom, f, v):
    """BFS components of the upper link of v; list of vertex lists."""
    U = [u for u in dom.neighbours(v) if higher(f, u, v)]
    seen, comps = set(), []
    for s in U:
        if s in seen:
            continue
        comp, dq = [], deque([s])
        seen.add(s)
        while dq:
            a = dq.popleft()
            comp.append(a)
            for b in U:
                if b not in seen and dom.edge(a, b):
                    seen.add(b)
                    dq.append(b)
        comps.append(comp)
    return comps


def gradient(dom, f, v):
    """Highest vertex of the upper link; None for a maximum."""
    best = None
    for u in dom.neighbours(v):
        if higher(f, u, v) and (best is None or higher(f, u, best)):
            best = u
    return best


def trace_gradient_paths(dom, f, s, M):
    """Alg. 2 TraceGradientPaths(s, M), literally."""
    P = []
    for comp in upper_components(dom, f, s):
        u = comp[0]
        for w in comp:                      # UpperLinkRep: highest vertex
            if higher(f, w, u):
                u = w
        p = [s]
        while u not in M:
            p.append(u)
            u = gradient(dom, f, u)
        p.append(u)                         # the path ends at the maximum it reached
        P.append(p)
    return P


def extremum_graph(dom, f):
    f = np.asarray(f, dtype=np.float32).reshape(-1)
    n = dom.n
    beta = [len(upper_components(dom, f, v)) for v in range(n)]
    M = {v for v in range(n) if beta[v] == 0}
    saddles = [v for v in range(n) if beta[v] >= 2]
    ptr = [v if v in M else gradient(dom, f, v) for v in range(n)]
    label = []
    for v in range(n):
        u = v
        while u not in M:
            u = ptr[u]
        label.append(u)
    arcs, raw, paths = {}, [], {}
    for s in saddles:
        P = trace_gradient_paths(dom, f, s, M)
        paths[s] = P
        for p in P:
            m = p[-1]
            raw.append((s, p[1] if len(p) > 2 else p[-1], m))
            arcs[(s, m)] = arcs.get((s, m), 0) + 1
    return dict(
        ptr=np.array(ptr, np.int64), label=np.array(label, np.int64), beta=np.array(beta, np.int32),
        maxima=np.array(sorted(M), np.int64), saddles=np.array(saddles, np.int64),
        saddle_beta=np.array([beta[s] for s in saddles], np.int32),
        arcs=np.array(sorted((s, m, c) for (s, m), c in arcs.items()), np.int64).reshape(-1, 3),
        paths=paths)


def grid_graph(f, dims):
    return extremum_graph(grid_domain(list(dims)), f)


def csr_graph(f, row_ptr, col_idx):
    return extremum_graph(csr_domain(row_ptr, col_idx), f)


def freudenthal_csr(dims):
    """The Freudenthal edge set as a symmetric CSR (brute force, tiny grids)."""
    dom = grid_domain(list(dims))
    rows = [sorted(dom.neighbours(v)) for v in range(dom.n)]
    row_ptr = np.zeros(dom.n + 1, np.int64)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col_idx = np.array(list(itertools.chain.from_iterable(rows)), np.int32)
    return row_ptr, col_idx
