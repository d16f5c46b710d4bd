"""B200-native extremum graphs (arXiv 2303.02724 hot path) -- Python binding.

    import paper_2303_02724_b200 as eg
    ctx = eg.Context()                      # one per GPU / process
    g = ctx.compute(field, dims=[nx, ny, nz])   # field: CUDA float32 tensor, axis 0 fastest
    g.maxima, g.saddles, g.saddle_beta, g.arcs, g.labels

All computation happens in libeg_b200.so (hand-written sm_100a kernels behind
the C ABI in include/eg.h).  This module only marshals arguments; it never
computes any step of the method itself and has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _abi
from ._abi import (EG_ARC_PATHS, EG_BUNDLE, EG_NODE_VALUES, EG_CHECK_CSR, EG_CHECK_NAN, EG_FORCE_GENERIC, EG_MINIMUM, EG_NO_GRAPH_D2H,
                   EG_RAW_ARCS, EG_STATS, EG_GRAPH32,  # noqa: F401
                   EG_VIRTUAL_PARTS)

__all__ = ["Context", "Graph", "EgError", "grid_domain", "csr_domain", "EG_CHECK_NAN", "EG_RAW_ARCS",
           "EG_CHECK_CSR", "EG_FORCE_GENERIC", "EG_NO_GRAPH_D2H", "EG_MINIMUM", "EG_ARC_PATHS", "EG_BUNDLE", "EG_NODE_VALUES",
           "EG_STATS", "EG_GRAPH32", "EG_VIRTUAL_PARTS"]


class EgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{_abi.STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")


@dataclass
class Graph:
    """The extremum graph: ascending maxima, saddles (+ beta0+), arcs
    (saddle, maximum, multiplicity) sorted by (saddle, maximum); labels are the
    owned vertices' maxima (CUDA int32 tensor, a copy owned by this object)."""
    maxima: np.ndarray
    saddles: np.ndarray
    saddle_beta: np.ndarray
    arcs: np.ndarray
    labels: Optional[torch.Tensor]
    raw_arcs: Optional[np.ndarray] = None
    # EG_ARC_PATHS: (offsets[n+1], vertices) -- path j = vertices[offsets[j]:offsets[j+1]]
    arc_paths: Optional[tuple] = None


def grid_domain(dims: Sequence[int], slab: Optional[Sequence[int]] = None) -> _abi.EgDomain:
    if not 1 <= len(dims) <= 8:      # the eg_grid struct holds 8 extents (include/eg.h)
        raise EgError(_abi.EG_ERR_INVALID_ARG, f"ndim {len(dims)} not in [1, 8]")
    d = _abi.EgDomain()
    d.kind = _abi.EG_DOMAIN_GRID
    d.grid.ndim = len(dims)
    for i, x in enumerate(dims):
        d.grid.dims[i] = int(x)
    if slab is None:
        slab = (0, int(dims[-1]))
    d.grid.slab_begin, d.grid.slab_end = int(slab[0]), int(slab[1])
    return d


def csr_domain(row_ptr: torch.Tensor, col_idx: torch.Tensor, v_range: Optional[Sequence[int]] = None) -> _abi.EgDomain:
    if row_ptr.dtype != torch.int64 or col_idx.dtype != torch.int32:
        raise TypeError("row_ptr must be int64 and col_idx int32")
    if not (row_ptr.is_cuda and col_idx.is_cuda):
        raise TypeError("row_ptr / col_idx must be CUDA tensors")
    n = row_ptr.numel() - 1
    d = _abi.EgDomain()
    d.kind = _abi.EG_DOMAIN_CSR
    d.csr.n_vertices = n
    d.csr.nnz = col_idx.numel()
    d.csr.row_ptr = row_ptr.data_ptr()
    d.csr.col_idx = col_idx.data_ptr()
    v0, v1 = v_range if v_range is not None else (0, n)
    d.csr.v_begin, d.csr.v_end = int(v0), int(v1)
    return d


class _DevView:
    """Zero-copy view of a device buffer owned by the library."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _arr(p, n, dt):
    if n == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)


class Context:
    """One library context per GPU (and per process / rank)."""

    def __init__(self, device: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None,
                 nccl_id: Optional[bytes] = None, rank: int = 0, world: int = 1):
        L = _abi.lib()
        if not torch.cuda.is_available():
            raise EgError(_abi.EG_ERR_CUDA, "no CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        if world > 1:
            buf = C.create_string_buffer(nccl_id, 128)
            st = L.eg_create_dist(C.byref(h), self.device, C.c_void_p(self.stream.cuda_stream), buf, rank, world)
        else:
            st = L.eg_create(C.byref(h), self.device, C.c_void_p(self.stream.cuda_stream))
        if st != _abi.EG_OK:
            raise EgError(st, "eg_create failed")
        self._h = h
        self.rank, self.world = rank, world

    # ------------------------------------------------------------ helpers
    def _check(self, st: int, what: str):
        if st != _abi.EG_OK:
            msg = _abi.lib().eg_last_error(self._h)
            raise EgError(st, f"{what}: {msg.decode() if msg else ''}")

    @staticmethod
    def _domain(dims, csr, slab, v_range):
        if (dims is None) == (csr is None):
            raise ValueError("give exactly one of dims= or csr=")
        if dims is not None:
            return grid_domain(dims, slab)
        return csr_domain(csr[0], csr[1], v_range)

    # -------------------------------------------------------------- calls
    def compute(self, field: torch.Tensor, dims: Optional[Sequence[int]] = None, csr=None, flags: int = 0,
                slab=None, v_range=None, materialize: bool = True) -> Optional[Graph]:
        """S1..S4 on a device-resident field (flat, axis 0 fastest): float32;
        float16 / bfloat16 / (u)int8 / (u)int16, which the library converts
        exactly to float32 on the device; or float64 / (u)int32 / (u)int64,
        which it replaces by the field's SoS-rank image (one GPU, no
        EG_NODE_VALUES) -- both through eg_compute_typed.
        The graph is always copied to host memory owned by the library; with
        materialize=False no numpy copies are made (use graph() later)."""
        dtypes = {torch.float32: _abi.EG_DTYPE_F32, torch.float16: _abi.EG_DTYPE_F16,
                  torch.bfloat16: _abi.EG_DTYPE_BF16, torch.uint8: _abi.EG_DTYPE_U8, torch.int8: _abi.EG_DTYPE_I8,
                  torch.int16: _abi.EG_DTYPE_I16, torch.float64: _abi.EG_DTYPE_F64, torch.int32: _abi.EG_DTYPE_I32,
                  torch.int64: _abi.EG_DTYPE_I64}
        for name, code in (("uint16", _abi.EG_DTYPE_U16), ("uint32", _abi.EG_DTYPE_U32),
                           ("uint64", _abi.EG_DTYPE_U64)):
            if hasattr(torch, name):
                dtypes[getattr(torch, name)] = code
        if not (field.is_cuda and field.dtype in dtypes and field.is_contiguous()):
            raise TypeError("field must be a contiguous CUDA tensor of float32/64, float16, bfloat16 or an "
                            "8/16/32/64-bit integer type")
        dom = self._domain(dims, csr, slab, v_range)
        if field.dtype == torch.float32:
            st = _abi.lib().eg_compute(self._h, C.byref(dom), C.c_void_p(field.data_ptr()), flags)
        else:
            st = _abi.lib().eg_compute_typed(self._h, C.byref(dom), C.c_void_p(field.data_ptr()),
                                             dtypes[field.dtype], flags)
        self._check(st, "eg_compute")
        self._last_flags = flags
        return self._graph(flags) if materialize else None

    def graph(self) -> Graph:
        """The graph of the last compute as numpy arrays (copies).  After a
        compute with EG_NO_GRAPH_D2H (graph left in HBM) the library copies
        it to the host here (one process)."""
        self._fetch = True
        try:
            return self._graph(getattr(self, "_last_flags", 0))
        finally:
            self._fetch = False

    def compute_host(self, field: torch.Tensor, dims=None, csr=None, flags: int = 0, labels_out=None,
                     slab=None, v_range=None, materialize: bool = True) -> Optional[Graph]:
        """End to end from a host (ideally pinned) float32 tensor; optional
        host int32 labels_out (pinned: the library's chunked pipeline copies
        each chunk's labels while later chunks of the field arrive) receives
        the owned labels.  The graph is in host memory owned by the library
        when this returns; materialize=False skips the numpy copies (graph())."""
        if field.is_cuda or field.dtype != torch.float32 or not field.is_contiguous():
            raise TypeError("field must be a contiguous host float32 tensor")
        dom = self._domain(dims, csr, slab, v_range)
        lp = C.c_void_p(labels_out.data_ptr()) if labels_out is not None else C.c_void_p()
        st = _abi.lib().eg_compute_host(self._h, C.byref(dom), C.c_void_p(field.data_ptr()), lp, flags)
        self._check(st, "eg_compute_host")
        self._last_flags = flags
        return self._graph(flags) if materialize else None

    def gradient(self, field: torch.Tensor, dims=None, csr=None, slab=None, v_range=None):
        """S1 + S3 per owned vertex: (ptr int32 global ids, beta0+ uint8)."""
        dom = self._domain(dims, csr, slab, v_range)
        if dims is not None:
            n = int(np.prod(dims[:-1], dtype=np.int64)) * (dom.grid.slab_end - dom.grid.slab_begin)
        else:
            n = dom.csr.v_end - dom.csr.v_begin
        ptr = torch.empty(max(n, 1), dtype=torch.int32, device=field.device)
        beta = torch.empty(max(n, 1), dtype=torch.uint8, device=field.device)
        st = _abi.lib().eg_gradient(self._h, C.byref(dom), C.c_void_p(field.data_ptr()), C.c_void_p(ptr.data_ptr()),
                                    C.c_void_p(beta.data_ptr()))
        self._check(st, "eg_gradient")
        return ptr[:n], beta[:n]

    def labels(self) -> torch.Tensor:
        """The owned labels of the last compute as a zero-copy view of the
        library's device buffer: valid only until the next compute / gradient
        / close on this context (Graph.labels is a copy)."""
        p, n = C.c_void_p(), C.c_int64()
        self._check(_abi.lib().eg_get_labels(self._h, C.byref(p), C.byref(n)), "eg_get_labels")
        if n.value == 0:
            return torch.zeros(0, dtype=torch.int32, device=f"cuda:{self.device}")
        return torch.as_tensor(_DevView(p.value, n.value, "<i4"), device=f"cuda:{self.device}")

    def _graph(self, flags: int) -> Graph:
        if flags & _abi.EG_NO_GRAPH_D2H and not getattr(self, "_fetch", False):
            return Graph(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32),
                         np.zeros((0, 3), np.int64), self.labels().clone())
        if flags & _abi.EG_GRAPH32:      # 32-bit ids on the host (widened here, outside the library)
            g = _abi.EgGraph32()
            self._check(_abi.lib().eg_get_graph32(self._h, C.byref(g)), "eg_get_graph32")
        else:
            g = _abi.EgGraph()
            self._check(_abi.lib().eg_get_graph(self._h, C.byref(g)), "eg_get_graph")
        arcs = np.stack([_arr(g.arc_saddle, g.n_arc, np.int64), _arr(g.arc_max, g.n_arc, np.int64),
                         _arr(g.arc_mult, g.n_arc, np.int64)], axis=1) if g.n_arc else np.zeros((0, 3), np.int64)
        raw = None
        if flags & _abi.EG_ARC_PATHS:
            flags |= _abi.EG_RAW_ARCS
        if flags & _abi.EG_RAW_ARCS:
            n = C.c_int64()
            s, r, m = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
            self._check(_abi.lib().eg_get_raw_arcs(self._h, C.byref(n), C.byref(s), C.byref(r), C.byref(m)),
                        "eg_get_raw_arcs")
            raw = np.stack([_arr(s, n.value, np.int64), _arr(r, n.value, np.int64), _arr(m, n.value, np.int64)],
                           axis=1) if n.value else np.zeros((0, 3), np.int64)
        paths = None
        if flags & _abi.EG_ARC_PATHS:
            n = C.c_int64()
            o, v = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
            self._check(_abi.lib().eg_get_arc_paths(self._h, C.byref(n), C.byref(o), C.byref(v)), "eg_get_arc_paths")
            off = _arr(o, n.value + 1, np.int64)
            paths = (off, _arr(v, int(off[-1]), np.int64))
        return Graph(maxima=_arr(g.maxima, g.n_max, np.int64), saddles=_arr(g.saddles, g.n_saddle, np.int64),
                     saddle_beta=_arr(g.saddle_beta, g.n_saddle, np.int32), arcs=arcs, labels=self.labels().clone(),
                     raw_arcs=raw, arc_paths=paths)

    def simplify(self, tau: float) -> Graph:
        """Persistence-directed cancellation of the last graph, which
        must have been computed with EG_NODE_VALUES; serial on the host."""
        g = _abi.EgGraph()
        self._check(_abi.lib().eg_simplify(self._h, C.c_double(tau), C.byref(g)), "eg_simplify")
        arcs = np.stack([_arr(g.arc_saddle, g.n_arc, np.int64), _arr(g.arc_max, g.n_arc, np.int64),
                         _arr(g.arc_mult, g.n_arc, np.int64)], axis=1) if g.n_arc else np.zeros((0, 3), np.int64)
        return Graph(maxima=_arr(g.maxima, g.n_max, np.int64), saddles=_arr(g.saddles, g.n_saddle, np.int64),
                     saddle_beta=_arr(g.saddle_beta, g.n_saddle, np.int32), arcs=arcs, labels=None)

    def stats(self) -> dict:
        s = _abi.EgStats()
        self._check(_abi.lib().eg_get_stats(self._h, C.byref(s)), "eg_get_stats")
        d = {k: getattr(s, k) for k, _ in _abi.EgStats._fields_}
        d["chase_hist"] = list(s.chase_hist)
        return d

    def close(self):
        if getattr(self, "_h", None):
            _abi.lib().eg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _abi.lib().eg_nccl_unique_id(buf)
    if st != _abi.EG_OK:
        raise EgError(st, "eg_nccl_unique_id failed")
    return buf.raw


# ------------------------------------------------------------ multi-GPU host logic

def plan_slabs(depth: int, world: int):
    """Slab partition of the slowest grid axis (P:278 blocks along z; SURVEY
    8(e)): `world` contiguous plane ranges [z0, z1) in rank order, balanced to
    +-1 plane, each of at least 2 planes (the boundary exchange needs distinct
    first and last planes)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if world > 1 and depth < 2 * world:
        raise ValueError(f"{world} slabs need at least {2 * world} planes, the grid has {depth}")
    return [(depth * r // world, depth * (r + 1) // world) for r in range(world)]


def plan_ranges(n: int, world: int):
    """Vertex-range partition of a CSR graph: `world` contiguous ranges."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def init_distributed(group=None, device: Optional[int] = None, stream=None) -> "Context":
    """One Context per rank sharing an NCCL communicator owned by the library.
    torch.distributed (any backend) only carries the 128-byte NCCL unique id
    from rank 0 to the others; every exchange of the hot path is NCCL inside
    libeg_b200.so.  Collective over `group`."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return Context(device=device, stream=stream)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return Context(device=device, stream=stream, nccl_id=box[0], rank=rank, world=world)
