"""Helpers for GPU-vs-oracle parity (bit-exact: every output is integer)."""
import numpy as np


def first_diff(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    idx = np.nonzero(a != b)
    if len(idx[0]) == 0:
        return None
    i = tuple(x[0] for x in idx)
    return f"{len(idx[0])} differences; first at {i}: gpu={a[i]} oracle={b[i]}"


def assert_graph_equal(g, o, labels=True, raw=False, what=""):
    """g: paper_2303_02724_b200.Graph, o: oracle.Graph (whole domain)."""
    msgs = []
    for name, a, b in [("maxima", g.maxima, o.maxima), ("saddles", g.saddles, o.saddles),
                       ("saddle_beta", g.saddle_beta, o.saddle_beta), ("arcs", g.arcs, o.arcs)]:
        d = first_diff(a, b)
        if d:
            msgs.append(f"{name}: {d}")
    if labels:
        d = first_diff(g.labels.cpu().numpy().astype(np.int64), o.label)
        if d:
            msgs.append(f"labels: {d}")
    if raw:
        ro = np.stack([o.raw_s, o.raw_rep, o.raw_m], axis=1)
        d = first_diff(g.raw_arcs, ro)
        if d:
            msgs.append(f"raw arcs: {d}")
    assert not msgs, f"{what} parity failure:\n  " + "\n  ".join(msgs)


def assert_full_equal(g, o, ptr=None, beta=None, what=""):
    """Whole-domain parity at full size: every graph output, every label and,
    when given (eg_gradient of the same field), every gradient pointer and
    beta0+ (uint8, saturated at 255 by the ABI) -- element by element."""
    msgs = []
    for name, a, b in [("maxima", g.maxima, o.maxima), ("saddles", g.saddles, o.saddles),
                       ("saddle_beta", g.saddle_beta, o.saddle_beta), ("arcs", g.arcs, o.arcs)]:
        d = first_diff(a, b)
        if d:
            msgs.append(f"{name}: {d}")
    lab = g.labels.cpu().numpy()
    d = first_diff(lab.astype(np.int64), o.label)
    if d:
        msgs.append(f"labels: {d}")
    if ptr is not None:
        d = first_diff(ptr.astype(np.int64), o.ptr)
        if d:
            msgs.append(f"gradient: {d}")
    if beta is not None:
        d = first_diff(beta.astype(np.int32), np.minimum(o.beta, 255))
        if d:
            msgs.append(f"beta0+: {d}")
    assert not msgs, f"{what} parity failure:\n  " + "\n  ".join(msgs)


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
