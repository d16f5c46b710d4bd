"""ctypes binding of include/eg.h -- argument marshalling only.

Every step of the hot path runs in libeg_b200.so (sm_100a kernels).  There is
no CPU fallback: if the library is missing or no CUDA device is present,
loading or eg_create fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EG_LIB_PATH") or os.path.join(HERE, "libeg_b200.so")   # (override: timing experiments)

EG_OK, EG_ERR_INVALID_ARG, EG_ERR_NAN, EG_ERR_OOM, EG_ERR_CUDA, EG_ERR_NCCL, EG_ERR_STATE, EG_ERR_UNSUPPORTED = range(8)
STATUS_NAMES = ["EG_OK", "EG_ERR_INVALID_ARG", "EG_ERR_NAN", "EG_ERR_OOM", "EG_ERR_CUDA", "EG_ERR_NCCL",
                "EG_ERR_STATE", "EG_ERR_UNSUPPORTED"]
EG_DOMAIN_GRID, EG_DOMAIN_CSR = 0, 1
(EG_DTYPE_F32, EG_DTYPE_F16, EG_DTYPE_BF16, EG_DTYPE_U8, EG_DTYPE_I8, EG_DTYPE_U16, EG_DTYPE_I16, EG_DTYPE_F64,
 EG_DTYPE_I32, EG_DTYPE_U32, EG_DTYPE_I64, EG_DTYPE_U64) = range(12)
(EG_CHECK_NAN, EG_RAW_ARCS, EG_CHECK_CSR, EG_FORCE_GENERIC, EG_NO_GRAPH_D2H, EG_MINIMUM, EG_ARC_PATHS,
 EG_BUNDLE, EG_NODE_VALUES, EG_STATS, EG_GRAPH32) = 1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 2048


def EG_VIRTUAL_PARTS(k: int) -> int:
    """k virtual slabs / ranges on one GPU: bits 16-31 of the flags (no flag bit)."""
    if not 0 <= int(k) < 65536:
        raise ValueError("EG_VIRTUAL_PARTS: 0 <= k < 65536")
    return int(k) << 16


# every symbol include/eg.h declares (checked by tests/test_abi_exports.py)
EXPORTS = ["eg_create", "eg_nccl_unique_id", "eg_create_dist", "eg_compute", "eg_compute_host", "eg_gradient",
           "eg_compute_typed", "eg_get_graph", "eg_get_graph32", "eg_get_raw_arcs", "eg_get_arc_paths", "eg_simplify", "eg_get_labels", "eg_get_stats",
           "eg_destroy", "eg_last_error"]


class EgGrid(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("dims", C.c_int64 * 8), ("slab_begin", C.c_int64), ("slab_end", C.c_int64)]


class EgCsr(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("v_begin", C.c_int64), ("v_end", C.c_int64)]


class EgDomain(C.Structure):
    _fields_ = [("kind", C.c_int32), ("grid", EgGrid), ("csr", EgCsr)]


class EgGraph(C.Structure):
    _fields_ = [("n_max", C.c_int64), ("n_saddle", C.c_int64), ("n_arc", C.c_int64),
                ("maxima", C.POINTER(C.c_int64)), ("saddles", C.POINTER(C.c_int64)),
                ("saddle_beta", C.POINTER(C.c_int32)), ("arc_saddle", C.POINTER(C.c_int64)),
                ("arc_max", C.POINTER(C.c_int64)), ("arc_mult", C.POINTER(C.c_int32))]


class EgGraph32(C.Structure):
    _fields_ = [("n_max", C.c_int64), ("n_saddle", C.c_int64), ("n_arc", C.c_int64),
                ("maxima", C.POINTER(C.c_int32)), ("saddles", C.POINTER(C.c_int32)),
                ("saddle_beta", C.POINTER(C.c_int32)), ("arc_saddle", C.POINTER(C.c_int32)),
                ("arc_max", C.POINTER(C.c_int32)), ("arc_mult", C.POINTER(C.c_int32))]


class EgStats(C.Structure):
    _fields_ = [("us_classify", C.c_double), ("us_jump", C.c_double), ("us_boundary", C.c_double),
                ("us_label", C.c_double), ("us_arcs", C.c_double), ("us_graph", C.c_double),
                ("us_total", C.c_double), ("jump_rounds", C.c_int32), ("boundary_rounds", C.c_int32),
                ("kernel_launches", C.c_int32), ("path", C.c_int32), ("n_vertices", C.c_int64),
                ("n_raw_arcs", C.c_int64), ("n_exit_targets", C.c_int64), ("bytes_alg", C.c_int64),
                ("us_main", C.c_double), ("bytes_main", C.c_int64), ("tile_rounds", C.c_int32),
                ("chase_max", C.c_int32), ("n_exit", C.c_int64), ("chase_hist", C.c_int64 * 16)]


_lib = None


def lib():
    """Load libeg_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32 = C.c_void_p, C.c_uint32
    L.eg_create.argtypes = [C.POINTER(vp), C.c_int, vp]
    L.eg_nccl_unique_id.argtypes = [vp]
    L.eg_create_dist.argtypes = [C.POINTER(vp), C.c_int, vp, vp, C.c_int, C.c_int]
    L.eg_compute.argtypes = [vp, C.POINTER(EgDomain), vp, u32]
    L.eg_compute_host.argtypes = [vp, C.POINTER(EgDomain), vp, vp, u32]
    L.eg_compute_typed.argtypes = [vp, C.POINTER(EgDomain), vp, C.c_int, u32]
    L.eg_gradient.argtypes = [vp, C.POINTER(EgDomain), vp, vp, vp]
    L.eg_get_graph.argtypes = [vp, C.POINTER(EgGraph)]
    L.eg_get_graph32.argtypes = [vp, C.POINTER(EgGraph32)]
    P64 = C.POINTER(C.c_int64)
    L.eg_get_raw_arcs.argtypes = [vp, P64, C.POINTER(P64), C.POINTER(P64), C.POINTER(P64)]
    L.eg_get_labels.argtypes = [vp, C.POINTER(vp), P64]
    L.eg_get_arc_paths.argtypes = [vp, P64, C.POINTER(P64), C.POINTER(P64)]
    L.eg_simplify.argtypes = [vp, C.c_double, C.POINTER(EgGraph)]
    L.eg_get_stats.argtypes = [vp, C.POINTER(EgStats)]
    L.eg_destroy.argtypes = [vp]
    L.eg_last_error.argtypes = [vp]
    L.eg_last_error.restype = C.c_char_p
    for name in EXPORTS:
        if name != "eg_last_error":
            getattr(L, name).restype = C.c_int
    _lib = L
    return L
