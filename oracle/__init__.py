"""CPU oracle for the extremum-graph hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2303_02724_b200``) never imports it and shares no code
with it; see the header of ``oracle/eg_oracle.c`` for what each step follows
in PAPER.md.

This module is a thin ctypes/numpy wrapper around ``liboracle`` (plain C,
single thread, built with ``gcc -O2`` by :func:`build`).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eg_oracle.c")
_LIB = os.path.join(_HERE, "libeg_oracle.so")

OK, ERR_INVALID, ERR_NAN, ERR_OOM = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2, no OpenMP: single-threaded by construction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Result(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("ptr", C.POINTER(C.c_int64)),
        ("label", C.POINTER(C.c_int64)),
        ("beta", C.POINTER(C.c_int32)),
        ("n_max", C.c_int64),
        ("maxima", C.POINTER(C.c_int64)),
        ("n_saddle", C.c_int64),
        ("saddles", C.POINTER(C.c_int64)),
        ("saddle_beta", C.POINTER(C.c_int32)),
        ("n_arc", C.c_int64),
        ("arc_s", C.POINTER(C.c_int64)),
        ("arc_m", C.POINTER(C.c_int64)),
        ("arc_mult", C.POINTER(C.c_int32)),
        ("n_raw", C.c_int64),
        ("raw_s", C.POINTER(C.c_int64)),
        ("raw_rep", C.POINTER(C.c_int64)),
        ("raw_m", C.POINTER(C.c_int64)),
    ]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64p, i32p, f32p = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_float)
        _lib.ego_grid.argtypes = [C.c_int, i64p, f32p, C.POINTER(_Result)]
        _lib.ego_csr.argtypes = [C.c_int64, i64p, i32p, f32p, C.POINTER(_Result)]
        _lib.ego_free.argtypes = [C.POINTER(_Result)]
        _lib.ego_grid_adjacent.argtypes = [C.c_int, i64p, i64p]
        _lib.ego_grid_link.argtypes = [C.c_int, i64p, C.c_int64, i64p]
        _lib.ego_grid_link.restype = C.c_int64
        _lib.ego_grid_vertex.argtypes = [C.c_int, i64p, f32p, C.c_int64, i64p, i32p, i64p, C.c_int32]
        _lib.ego_csr_vertex.argtypes = [C.c_int64, i64p, i32p, f32p, C.c_int64, i64p, i32p, i64p, C.c_int32]
        _lib.ego_grid_walk.argtypes = [C.c_int, i64p, f32p, C.c_int64, i64p]
        _lib.ego_grid_walk.restype = C.c_int64
        _lib.ego_csr_walk.argtypes = [C.c_int64, i64p, i32p, f32p, C.c_int64, i64p]
        _lib.ego_csr_walk.restype = C.c_int64
        _lib.ego_grid_euler.argtypes = [C.c_int, i64p, f32p, i64p]
        _lib.ego_csr_euler.argtypes = [C.c_int64, i64p, i32p, f32p, i64p]
        _lib.ego_grid_link_stats.argtypes = [C.c_int, i64p, C.c_int64, i64p, i64p, i64p]
        _lib.ego_set_order.argtypes = [C.c_int]
        _lib.ego_grid_range.argtypes = [C.c_int, i64p, f32p, C.c_int64, C.c_int64, i64p, i32p, i64p, i64p,
                                        C.c_int64, i64p]
        _lib.ego_csr_range.argtypes = [C.c_int64, i64p, i32p, f32p, C.c_int64, C.c_int64, i64p, i32p, i64p, i64p,
                                       C.c_int64, i64p]
        _lib.ego_labels.argtypes = [C.c_int64, i64p, i64p]
    return _lib


class reversed_order:
    """Context manager: every oracle call inside runs under the reversed total
    order (O10), i.e. computes the MINIMUM graph: minima, 1-saddles (beta0 of the
    lower link >= 2) and the descending arcs / labels (reading L11)."""

    def __enter__(self):
        _L().ego_set_order(1)
        return self

    def __exit__(self, *exc):
        _L().ego_set_order(0)
        return False


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class Graph:
    """Oracle output (O9): everything as int64 numpy arrays, ids are global."""
    ptr: np.ndarray
    label: np.ndarray
    beta: np.ndarray
    maxima: np.ndarray
    saddles: np.ndarray
    saddle_beta: np.ndarray
    arc_s: np.ndarray
    arc_m: np.ndarray
    arc_mult: np.ndarray
    raw_s: np.ndarray
    raw_rep: np.ndarray
    raw_m: np.ndarray

    @property
    def arcs(self):
        return np.stack([self.arc_s, self.arc_m, self.arc_mult.astype(np.int64)], axis=1)


class OracleError(RuntimeError):
    pass


def _take(res: _Result) -> Graph:
    def arr(p, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

    n = res.n
    g = Graph(
        ptr=arr(res.ptr, n, np.int64), label=arr(res.label, n, np.int64), beta=arr(res.beta, n, np.int32),
        maxima=arr(res.maxima, res.n_max, np.int64), saddles=arr(res.saddles, res.n_saddle, np.int64),
        saddle_beta=arr(res.saddle_beta, res.n_saddle, np.int32),
        arc_s=arr(res.arc_s, res.n_arc, np.int64), arc_m=arr(res.arc_m, res.n_arc, np.int64),
        arc_mult=arr(res.arc_mult, res.n_arc, np.int32),
        raw_s=arr(res.raw_s, res.n_raw, np.int64), raw_rep=arr(res.raw_rep, res.n_raw, np.int64),
        raw_m=arr(res.raw_m, res.n_raw, np.int64))
    _L().ego_free(C.byref(res))
    return g


def _dims_arr(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


def grid(f: np.ndarray, dims, minimum: bool = False) -> Graph:
    """Extremum graph of a float32 field on a Freudenthal grid; ``dims`` is
    fastest axis first and ``f`` is the flat row-major array (axis 0 fastest).
    minimum=True: the minimum graph (O10)."""
    if minimum:
        with reversed_order():
            return grid(f, dims)
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32).reshape(-1))
    d = _dims_arr(dims)
    res = _Result()
    rc = _L().ego_grid(len(d), _p(d, C.c_int64), _p(f, C.c_float), C.byref(res))
    if rc != OK:
        raise OracleError(f"ego_grid failed: {rc}")
    return _take(res)


def csr(f: np.ndarray, row_ptr: np.ndarray, col_idx: np.ndarray, minimum: bool = False) -> Graph:
    """Extremum graph of a float32 field on a CSR graph; minimum=True: the
    minimum graph (O10)."""
    if minimum:
        with reversed_order():
            return csr(f, row_ptr, col_idx)
    f = np.ascontiguousarray(f, dtype=np.float32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    res = _Result()
    rc = _L().ego_csr(len(f), _p(rp, C.c_int64), _p(ci, C.c_int32), _p(f, C.c_float), C.byref(res))
    if rc != OK:
        raise OracleError(f"ego_csr failed: {rc}")
    return _take(res)


def grid_adjacent(p, q) -> bool:
    p = _dims_arr(p)
    q = _dims_arr(q)
    if len(p) != len(q):
        raise ValueError("dimension mismatch")
    return bool(_L().ego_grid_adjacent(len(p), _p(p, C.c_int64), _p(q, C.c_int64)))


def grid_link(dims, v: int) -> np.ndarray:
    d = _dims_arr(dims)
    out = np.zeros(3 ** len(d), np.int64)
    n = _L().ego_grid_link(len(d), _p(d, C.c_int64), int(v), _p(out, C.c_int64))
    if n < 0:
        raise OracleError("bad vertex")
    return out[:n].copy()


def grid_link_stats(dims, v: int):
    """(|Lk(v)|, #link edges, chi of the link's clique complex)."""
    d = _dims_arr(dims)
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    rc = _L().ego_grid_link_stats(len(d), _p(d, C.c_int64), int(v), C.byref(a), C.byref(b), C.byref(c))
    if rc != OK:
        raise OracleError("bad vertex")
    return a.value, b.value, c.value


def grid_vertex(f, dims, v: int):
    """(ptr, beta0+, reps) of one vertex (O3..O5)."""
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32).reshape(-1))
    d = _dims_arr(dims)
    ptr, beta = C.c_int64(), C.c_int32()
    reps = np.zeros(3 ** len(d), np.int64)
    rc = _L().ego_grid_vertex(len(d), _p(d, C.c_int64), _p(f, C.c_float), int(v), C.byref(ptr), C.byref(beta),
                              _p(reps, C.c_int64), len(reps))
    if rc != OK:
        raise OracleError("bad vertex")
    return ptr.value, beta.value, reps[:beta.value].copy()


def csr_vertex(f, row_ptr, col_idx, v: int):
    f = np.ascontiguousarray(f, dtype=np.float32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    ptr, beta = C.c_int64(), C.c_int32()
    deg = int(rp[v + 1] - rp[v])
    reps = np.zeros(max(deg, 1), np.int64)
    rc = _L().ego_csr_vertex(len(f), _p(rp, C.c_int64), _p(ci, C.c_int32), _p(f, C.c_float), int(v),
                             C.byref(ptr), C.byref(beta), _p(reps, C.c_int64), len(reps))
    if rc != OK:
        raise OracleError("bad vertex")
    return ptr.value, beta.value, reps[:beta.value].copy()


def grid_walk(f, dims, v: int):
    """Alg. 2 walk from v: (maximum reached, number of steps)."""
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32).reshape(-1))
    d = _dims_arr(dims)
    steps = C.c_int64()
    m = _L().ego_grid_walk(len(d), _p(d, C.c_int64), _p(f, C.c_float), int(v), C.byref(steps))
    return m, steps.value


def csr_walk(f, row_ptr, col_idx, v: int):
    f = np.ascontiguousarray(f, dtype=np.float32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    steps = C.c_int64()
    m = _L().ego_csr_walk(len(f), _p(rp, C.c_int64), _p(ci, C.c_int32), _p(f, C.c_float), int(v), C.byref(steps))
    return m, steps.value


def grid_euler(f, dims) -> int:
    """sum_v (1 - chi(Lk+(v))) over the grid."""
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32).reshape(-1))
    d = _dims_arr(dims)
    s = C.c_int64()
    rc = _L().ego_grid_euler(len(d), _p(d, C.c_int64), _p(f, C.c_float), C.byref(s))
    if rc != OK:
        raise OracleError("euler failed")
    return s.value


def csr_euler(f, row_ptr, col_idx) -> int:
    f = np.ascontiguousarray(f, dtype=np.float32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    s = C.c_int64()
    rc = _L().ego_csr_euler(len(f), _p(rp, C.c_int64), _p(ci, C.c_int32), _p(f, C.c_float), C.byref(s))
    if rc != OK:
        raise OracleError("euler failed")
    return s.value


def bundle(g: Graph, f: np.ndarray, minimum: bool = False) -> Graph:
    """Arc bundling, literally: "a pair of maxima [may] contain more
    than one common (n-1)-saddle ... We select a single representative saddle
    ... the saddle with the highest scalar value" -- reading L19: among the
    saddles whose arcs reach exactly two distinct maxima {m1, m2}, keep for each
    pair the highest one (SoS order: value, then index); saddles with one or
    with three or more distinct maxima are kept; arcs follow their saddles.
    minimum=True: a minimum graph (O10), "highest" in the reversed order, i.e.
    the lowest value, ties to the lower index."""
    f = np.asarray(f, dtype=np.float32).reshape(-1)
    by_saddle = {}
    for s, m, c in g.arcs.tolist():
        by_saddle.setdefault(s, []).append(m)
    best = {}
    for s, ms in by_saddle.items():
        if len(ms) != 2:
            continue
        key = (min(ms), max(ms))
        rank = (lambda t: (-f[t], -t)) if minimum else (lambda t: (f[t], t))
        if key not in best or rank(s) > rank(best[key]):
            best[key] = s
    drop = {s for s, ms in by_saddle.items() if len(ms) == 2 and best[(min(ms), max(ms))] != s}
    keep_s = np.array([s not in drop for s in g.saddles.tolist()], bool)
    keep_a = np.array([s not in drop for s in g.arc_s.tolist()], bool)
    return Graph(ptr=g.ptr, label=g.label, beta=g.beta, maxima=g.maxima, saddles=g.saddles[keep_s],
                 saddle_beta=g.saddle_beta[keep_s], arc_s=g.arc_s[keep_a], arc_m=g.arc_m[keep_a],
                 arc_mult=g.arc_mult[keep_a], raw_s=g.raw_s, raw_rep=g.raw_rep, raw_m=g.raw_m)


def simplify(g: Graph, f: np.ndarray, tau: float, minimum: bool = False) -> Graph:
    """Persistence-directed cancellation, literally, with lazy cost
    updates (reading L20 in DESIGN.md):
    * cost(s) = min over its two distinct maxima of f(m) - f(s) for a simple
      saddle; f(second highest maximum) - f(s) for a multi-saddle (>= 3
      distinct maxima); a saddle with one distinct maximum is never cancelled;
      costs are differences of the float32 values in double precision;
    * a min-priority queue of (cost, saddle id) holds every saddle; pop s,
      recompute its cost: above tau -> discard (s stays); above the cost now at
      the top -> reinsert; else cancel: every distinct maximum of s but the
      highest (SoS order) is merged into the highest (their other arcs are
      redirected to it, multiplicities added), and s and the merged maxima leave
      the graph.
    minimum=True: a minimum graph (O10): "higher" and the signs are reversed."""
    import heapq
    f = np.asarray(f, dtype=np.float32).reshape(-1)
    sgn = -1.0 if minimum else 1.0
    val = lambda v: sgn * float(f[v])
    key = lambda v: (val(v), -v if minimum else v)          # SoS order (reversed for minima)
    arcs = {}
    for s, m, c in g.arcs.tolist():
        arcs.setdefault(s, {})[m] = arcs.get(s, {}).get(m, 0) + c
    by_max = {}
    for s, ms in arcs.items():
        for m in ms:
            by_max.setdefault(m, set()).add(s)
    maxima = set(g.maxima.tolist())
    alive = set(g.saddles.tolist())

    def cost(s):
        ms = sorted(arcs.get(s, {}), key=key)
        if len(ms) < 2:
            return math.inf
        return (val(ms[0]) if len(ms) == 2 else val(ms[-2])) - val(s)

    heap = [(cost(s), s) for s in sorted(alive)]
    heapq.heapify(heap)
    while heap:
        _, s = heapq.heappop(heap)
        c = cost(s)
        if c > tau:
            continue
        if heap and c > heap[0][0]:
            heapq.heappush(heap, (c, s))
            continue
        ms = sorted(arcs[s], key=key)
        top = ms[-1]
        for m in ms[:-1]:
            for s2 in by_max.pop(m, set()):
                if s2 == s:
                    continue
                mult = arcs[s2].pop(m)
                arcs[s2][top] = arcs[s2].get(top, 0) + mult
                by_max.setdefault(top, set()).add(s2)
            maxima.discard(m)
        for m in arcs.pop(s):
            if m in by_max:
                by_max[m].discard(s)
        alive.discard(s)
    keep = np.array([s in alive for s in g.saddles.tolist()], bool)
    out = sorted((s, m, c) for s in alive for m, c in arcs[s].items())
    a = np.array(out, np.int64).reshape(-1, 3)
    return Graph(ptr=g.ptr, label=g.label, beta=g.beta, maxima=np.array(sorted(maxima), np.int64),
                 saddles=g.saddles[keep], saddle_beta=g.saddle_beta[keep], arc_s=a[:, 0].copy(),
                 arc_m=a[:, 1].copy(), arc_mult=a[:, 2].astype(np.int32), raw_s=g.raw_s, raw_rep=g.raw_rep,
                 raw_m=g.raw_m)


# ------------------------------------------------------------ big domains
# The whole-domain oracle above is one thread; C3 (2^30 vertices) would take
# ~20 min that way.  Classification (O3..O6) is independent per vertex, so the
# harness below runs the oracle's own range function (ego_*_range: the same
# classify_vertex loop) on disjoint vertex ranges in forked worker processes,
# then O7 (ego_labels: the same memoised walk) and O8 (per saddle, label of
# every UpperLinkRep, reduced to unique (s, m) with multiplicity) on the
# assembled arrays.  No step is re-derived here; the result is the run_all
# result, which tests/test_oracle_pins.py::test_parallel_equals_whole checks.

_PAR = None   # (kind, args) inherited by the forked workers


def _range_worker(job):
    v0, v1 = job
    kind, args, ptr, beta = _PAR
    L = _L()
    cap = max(4096, (v1 - v0) // 2)
    while True:
        rs = np.zeros(cap, np.int64)
        rr = np.zeros(cap, np.int64)
        nrep = C.c_int64()
        pp = C.cast(C.c_void_p(ptr.ctypes.data + 8 * v0), C.POINTER(C.c_int64))
        bp = C.cast(C.c_void_p(beta.ctypes.data + 4 * v0), C.POINTER(C.c_int32))
        if kind == "grid":
            f, d = args
            rc = L.ego_grid_range(len(d), _p(d, C.c_int64), _p(f, C.c_float), v0, v1, pp, bp, _p(rs, C.c_int64),
                                  _p(rr, C.c_int64), cap, C.byref(nrep))
        else:
            f, rp, ci = args
            rc = L.ego_csr_range(len(f), _p(rp, C.c_int64), _p(ci, C.c_int32), _p(f, C.c_float), v0, v1, pp, bp,
                                 _p(rs, C.c_int64), _p(rr, C.c_int64), cap, C.byref(nrep))
        if rc != OK:
            return v0, rc, None, None
        if nrep.value <= cap:
            return v0, OK, rs[:nrep.value].copy(), rr[:nrep.value].copy()
        cap = nrep.value


def _parallel(kind, args, n, procs):
    import mmap
    import multiprocessing as mp
    global _PAR
    procs = procs or os.cpu_count() or 1
    pb = mmap.mmap(-1, max(8 * n, 8))            # MAP_SHARED | MAP_ANONYMOUS: the workers write into it
    bb = mmap.mmap(-1, max(4 * n, 4))
    ptr = np.frombuffer(pb, np.int64, count=n)
    beta = np.frombuffer(bb, np.int32, count=n)
    nchunk = max(1, min(n, procs * 16))
    edges = [n * i // nchunk for i in range(nchunk + 1)]
    jobs = [(edges[i], edges[i + 1]) for i in range(nchunk) if edges[i + 1] > edges[i]]
    _PAR = (kind, args, ptr, beta)
    try:
        if procs == 1:
            res = [_range_worker(j) for j in jobs]
        else:
            with mp.get_context("fork").Pool(procs) as pool:
                res = pool.map(_range_worker, jobs, chunksize=1)
    finally:
        _PAR = None
    res.sort(key=lambda r: r[0])
    for _, rc, _, _ in res:
        if rc != OK:
            raise OracleError(f"ego_{kind}_range failed: {rc}")
    ptr = ptr.copy()
    beta = beta.copy()
    del pb, bb
    label = np.empty(n, np.int64)
    rc = _L().ego_labels(n, _p(ptr, C.c_int64), _p(label, C.c_int64))
    if rc != OK:
        raise OracleError(f"ego_labels failed: {rc}")
    raw_s = np.concatenate([r[2] for r in res]) if res else np.zeros(0, np.int64)
    raw_rep = np.concatenate([r[3] for r in res]) if res else np.zeros(0, np.int64)
    raw_m = label[raw_rep]
    # O8: unique (s, m) per saddle with multiplicity, sorted by (s, m)
    if len(raw_s):
        o = np.lexsort((raw_m, raw_s))
        ss, mm = raw_s[o], raw_m[o]
        first = np.ones(len(ss), bool)
        first[1:] = (ss[1:] != ss[:-1]) | (mm[1:] != mm[:-1])
        idx = np.flatnonzero(first)
        mult = np.diff(np.append(idx, len(ss))).astype(np.int32)
        arc_s, arc_m = ss[idx], mm[idx]
    else:
        arc_s = arc_m = np.zeros(0, np.int64)
        mult = np.zeros(0, np.int32)
    maxima = np.flatnonzero(beta == 0).astype(np.int64)
    sad = np.flatnonzero(beta >= 2).astype(np.int64)
    return Graph(ptr=ptr, label=label, beta=beta, maxima=maxima, saddles=sad, saddle_beta=beta[sad].astype(np.int32),
                 arc_s=arc_s, arc_m=arc_m, arc_mult=mult, raw_s=raw_s, raw_rep=raw_rep, raw_m=raw_m)


def grid_parallel(f: np.ndarray, dims, procs: int = None) -> Graph:
    """grid() for big domains: the oracle's per-vertex steps over disjoint
    vertex ranges in `procs` forked processes (default: every host core)."""
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32).reshape(-1))
    d = _dims_arr(dims)
    return _parallel("grid", (f, d), len(f), procs)


def csr_parallel(f: np.ndarray, row_ptr: np.ndarray, col_idx: np.ndarray, procs: int = None) -> Graph:
    """csr() for big graphs, as grid_parallel."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    return _parallel("csr", (f, rp, ci), len(f), procs)
