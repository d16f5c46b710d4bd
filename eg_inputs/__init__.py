"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only builds scalar fields and
neighbourhood graphs (the inputs of P:104 "scalar field ... samples at vertices
of an n-dimensional grid").  Both ``oracle/`` and the product path consume the
same bytes produced here.  Recipes follow SURVEY.md 8(d) and are restated in
DESIGN.md ("Input recipes").  Layout: flat float32, axis 0 fastest,
i.e. a numpy array of shape (D_{n-1}, ..., D_0) flattened in C order.
"""
from __future__ import annotations

import math

import numpy as np

# ----------------------------------------------------------------- helpers


def _outer_axes(vecs):
    """vecs[i] is the 1D factor along axis i (axis 0 fastest); returns the
    product field with numpy shape (D_{n-1}, ..., D_0)."""
    out = np.ones(1, np.float64)
    for v in reversed(vecs):          # slowest axis first in numpy shape
        out = np.multiply.outer(out, v)
    return out.reshape([len(v) for v in reversed(vecs)])


def flat32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32).reshape(-1))


# --------------------------------------------------------------- C1 / C1'


def c1_gaussians(seed: int = 0, sigma: float = 4.0, size=(64, 64)):
    """C1: 2D 64x64 sum of 8 Gaussians on a 4 (axis 0) x 2 (axis 1) lattice,
    cell (16, 32); centre = (a+1/2, b+1/2)*cell + U(-0.15, 0.15)^2 * cell;
    A ~ U(0.5, 1).  Draw order: 8 jitter pairs (a outer, b inner), then 8
    amplitudes.  Returns (f32 flat, dims)."""
    rng = np.random.default_rng(seed)
    na, nb = 4, 2
    cell = (size[0] / na, size[1] / nb)
    centres = []
    for a in range(na):
        for b in range(nb):
            j = rng.uniform(-0.15, 0.15, size=2)
            centres.append(((a + 0.5 + j[0]) * cell[0], (b + 0.5 + j[1]) * cell[1]))
    amps = rng.uniform(0.5, 1.0, size=na * nb)
    i0 = np.arange(size[0], dtype=np.float64)
    i1 = np.arange(size[1], dtype=np.float64)
    f = np.zeros((size[1], size[0]))
    for (c0, c1), A in zip(centres, amps):
        f += A * _outer_axes([np.exp(-(i0 - c0) ** 2 / (2 * sigma ** 2)), np.exp(-(i1 - c1) ** 2 / (2 * sigma ** 2))])
    return flat32(f), [size[0], size[1]]


def sincos(p: int = 4, q: int = 4, seed: int = 7):
    """C1': f = sin(x) cos(y), P = 4q samples per period, N = pP + 1 per axis,
    h = 2 pi / P, x_0 = pi/4 + eps_x h, y_0 = pi/4 + eps_y h, eps ~ U(-0.3, 0.3)
    from default_rng(seed): the domain edges sit pi/4 (+eps h) from every
    critical line.  Returns (f32 flat, dims, x0, y0, h)."""
    rng = np.random.default_rng(seed)
    eps = rng.uniform(-0.3, 0.3, size=2)
    P = 4 * q
    N = p * P + 1
    h = 2 * math.pi / P
    x0 = math.pi / 4 + eps[0] * h
    y0 = math.pi / 4 + eps[1] * h
    x = x0 + h * np.arange(N)
    y = y0 + h * np.arange(N)
    f = _outer_axes([np.sin(x), np.cos(y)])
    return flat32(f), [N, N], x0, y0, h


# ----------------------------------------------------------------- C2 / C2'


def c2_gaussians_noise(n: int = 256, seed: int = 256, k: int = 32, eta: float = 1e-3):
    """C2: 3D n^3, 32 Gaussians: sigma ~ U(6, 16) (32 values), then centres
    c = U(0,1)^(32x3) (255 - 2 sigma) + sigma (columns = axes 0, 1, 2), then
    A ~ U(0.5, 1); f = sum A prod_a exp(-(i_a - c_a)^2 / 2 sigma^2) in float64,
    plus eta U(-1, 1) drawn as one array in linear-index order; cast to f32."""
    rng = np.random.default_rng(seed)
    sig = rng.uniform(6.0, 16.0, size=k)
    cen = rng.uniform(0.0, 1.0, size=(k, 3)) * ((n - 1) - 2 * sig)[:, None] + sig[:, None]
    amp = rng.uniform(0.5, 1.0, size=k)
    i = np.arange(n, dtype=np.float64)
    f = np.zeros((n, n, n))
    for s, c, A in zip(sig, cen, amp):
        g = [np.exp(-(i - c[a]) ** 2 / (2 * s * s)) for a in range(3)]
        f += A * _outer_axes(g)
    f = f.reshape(-1) + eta * rng.uniform(-1.0, 1.0, size=n ** 3)
    return flat32(f), [n, n, n]


def lattice_gaussians(n: int = 128, seed: int = 0, lattice=(4, 4, 2)):
    """C2': noise-free lattice of 4 x 4 x 2 Gaussians in an n^3 box; per cell
    (a outer ... c inner): jitter U(-0.15, 0.15)^3 * cell, sigma ~ U(n/32, n/21),
    A ~ U(0.5, 1).  Exactly 32 maxima (pin)."""
    rng = np.random.default_rng(seed)
    cell = [n / lattice[0], n / lattice[1], n / lattice[2]]
    i = np.arange(n, dtype=np.float64)
    f = np.zeros((n, n, n))
    for a in range(lattice[0]):
        for b in range(lattice[1]):
            for c in range(lattice[2]):
                j = rng.uniform(-0.15, 0.15, size=3)
                s = rng.uniform(n / 32, n / 21)
                A = rng.uniform(0.5, 1.0)
                cen = [(a + 0.5 + j[0]) * cell[0], (b + 0.5 + j[1]) * cell[1], (c + 0.5 + j[2]) * cell[2]]
                f += A * _outer_axes([np.exp(-(i - cen[ax]) ** 2 / (2 * s * s)) for ax in range(3)])
    return flat32(f), [n, n, n]


# ---------------------------------------------------------------------- C3


def turbulence(n: int = 1024, seed: int = 1024, device: str = "cpu", kc_div: int = 16):
    """C3: n^3 Gaussian random field with power |k|^(-11/3) (E(k) ~ k^(-5/3))
    and a cutoff exp(-|k|^2 / 2 k_c^2), k_c = n / 16 (|k| in integer
    wavenumbers, A(0) = 0): white noise -> rfftn -> multiply -> irfftn ->
    (f - mean) / std -> float32.  White noise comes from torch's generator on
    ``device`` seeded with ``seed`` (CPU and CUDA streams differ; a given
    (device, seed) is reproducible on this torch build).  Computed in float32 /
    complex64 on the device.  Returns (torch tensor f32 flat on device, dims)."""
    import torch

    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    w = torch.randn((n, n, n), generator=gen, device=dev, dtype=torch.float32)
    F = torch.fft.rfftn(w)
    del w
    k = torch.fft.fftfreq(n, d=1.0 / n, device=dev, dtype=torch.float32)
    kr = torch.fft.rfftfreq(n, d=1.0 / n, device=dev, dtype=torch.float32)
    kc = n / kc_div
    for z in range(n):   # slab-wise to bound temporaries at n = 1024
        k2 = k[z] ** 2 + k[:, None] ** 2 + kr[None, :] ** 2
        amp = torch.where(k2 > 0, k2.clamp_min(1e-30) ** (-11.0 / 12.0) * torch.exp(-k2 / (2 * kc * kc)),
                          torch.zeros_like(k2))
        F[z] *= amp
    f = torch.fft.irfftn(F, s=(n, n, n))
    del F
    f = (f - f.mean()) / f.std()
    return f.reshape(-1).contiguous(), [n, n, n]


# ---------------------------------------------------------------------- C4


def schwefel_profile(D: int, lo: float = -500.0, hi: float = 500.0) -> np.ndarray:
    """The 1-D Schwefel term t(x) = x sin(sqrt|x|) at x = lo + k (hi - lo) / (D - 1), float64."""
    x = lo + np.arange(D, dtype=np.float64) * (hi - lo) / (D - 1)
    return x * np.sin(np.sqrt(np.abs(x)))


def schwefel(dims=(32,) * 5, lo: float = -500.0, hi: float = 500.0, device=None):
    """C4: g(x) = 418.9829 n - sum_i x_i sin(sqrt|x_i|) on [lo, hi]^n,
    x = lo + k (hi - lo) / (D - 1); evaluated in float64 starting from
    418.9829 n and subtracting the slowest axis' term first, then cast to f32.
    device: build the field there (the 1-D terms come from numpy, the float64
    subtractions and the rounding to f32 are IEEE-exact on either side, so the
    bytes are the same); returns a torch tensor then."""
    n = len(dims)
    terms = [schwefel_profile(D, lo, hi) for D in dims]
    shape = list(reversed(dims))
    if device is not None:
        import torch
        acc = torch.full(shape, 418.9829 * n, dtype=torch.float64, device=device)
        for ax in reversed(range(n)):
            view = [1] * n
            view[n - 1 - ax] = dims[ax]
            acc -= torch.from_numpy(terms[ax]).to(device).reshape(view)
        return acc.to(torch.float32).reshape(-1).contiguous(), list(dims)
    acc = np.full(shape, 418.9829 * n, dtype=np.float64)
    for ax in reversed(range(n)):         # axis n-1 (slowest) first
        view = [1] * n
        view[n - 1 - ax] = dims[ax]
        acc -= terms[ax].reshape(view)
    return flat32(acc), list(dims)


def sumcos(dims=(32,) * 5, seed: int = 5, period_samples: int = 16):
    """C4': f = sum_i cos(x_i), h = 2 pi / 16, x_0 = -pi/2 + eps_i h with
    eps_i ~ U(-0.3, 0.3) from default_rng(seed), one per axis."""
    rng = np.random.default_rng(seed)
    n = len(dims)
    eps = rng.uniform(-0.3, 0.3, size=n)
    h = 2 * math.pi / period_samples
    shape = list(reversed(dims))
    acc = np.zeros(shape)
    for ax in range(n):
        x = -math.pi / 2 + eps[ax] * h + h * np.arange(dims[ax])
        view = [1] * n
        view[n - 1 - ax] = dims[ax]
        acc = acc + np.cos(x).reshape(view)
    return flat32(acc), list(dims), eps, h


def separable(profiles):
    """f(x) = sum_i h_i(x_i) for 1D profiles (axis 0 first), float64 -> f32."""
    dims = [len(p) for p in profiles]
    n = len(dims)
    acc = np.zeros(list(reversed(dims)))
    for ax in range(n):
        view = [1] * n
        view[n - 1 - ax] = dims[ax]
        acc = acc + np.asarray(profiles[ax], np.float64).reshape(view)
    return flat32(acc), dims


# ---------------------------------------------------------------------- C5


def gmm_points(n: int = 1_000_000, seed: int = 10, dim: int = 10, comps: int = 16):
    """C5 points: means U(-6, 6)^(16 x 10), ids integers(0, 16, n),
    X = mu[id] + standard_normal((n, 10)); f = log sum_c exp(-|x - mu_c|^2 / 2)
    (float64, then f32)."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-6.0, 6.0, size=(comps, dim))
    ids = rng.integers(0, comps, size=n)
    X = mu[ids] + rng.standard_normal((n, dim))
    f = np.empty(n, np.float64)
    for s in range(0, n, 65536):
        d2 = ((X[s:s + 65536, None, :] - mu[None, :, :]) ** 2).sum(-1)
        m = (-0.5 * d2).max(1)
        f[s:s + 65536] = m + np.log(np.exp(-0.5 * d2 - m[:, None]).sum(1))
    return X, f.astype(np.float32)


def knn_csr(X: np.ndarray, k: int = 16, device: str = "cpu"):
    """Exact k nearest neighbours (float64 squared distances, ties by index,
    self excluded), union-symmetrised; returns (row_ptr int64[N+1], sorted
    col_idx int32).  The graph is an input (not timed)."""
    import torch

    n = X.shape[0]
    dev = torch.device(device)
    Xt = torch.as_tensor(X, dtype=torch.float64, device=dev)
    sq = (Xt * Xt).sum(1)
    nbr = torch.empty((n, k), dtype=torch.int64, device=dev)
    chunk = 2048 if dev.type == "cuda" else 512
    ar = torch.arange(n, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d2 = sq[s:e, None] + sq[None, :] - 2.0 * (Xt[s:e] @ Xt.T)
        d2[torch.arange(e - s, device=dev), ar[s:e]] = float("inf")       # exclude self
        # ties by index: sort by (d2, index) via a stable sort of the k+8 best
        vals, idx = torch.topk(d2, k + 8, dim=1, largest=False, sorted=True)
        order = torch.argsort(idx, dim=1, stable=True)
        vals, idx = torch.gather(vals, 1, order), torch.gather(idx, 1, order)
        order = torch.argsort(vals, dim=1, stable=True)
        nbr[s:e] = torch.gather(idx, 1, order)[:, :k]
    src = torch.arange(n, device=dev).repeat_interleave(k)
    dst = nbr.reshape(-1)
    a = torch.cat([src, dst])
    b = torch.cat([dst, src])
    key = torch.unique(a * n + b)                 # sorted, de-duplicated
    rows, cols = key // n, key % n
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return row_ptr.cpu().numpy(), cols.to(torch.int32).cpu().numpy()


# -------------------------------------------------------------- random fields


def random_field(dims, seed: int, kind: str = "normal", levels: int = 4):
    """Random test fields: 'normal' (tie-free), 'int' (values in {0..levels-1},
    ties everywhere), 'signed_zero' (mix of +0/-0 and small ints), 'const'."""
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    if kind == "normal":
        f = rng.standard_normal(n)
    elif kind == "int":
        f = rng.integers(0, levels, size=n).astype(np.float64)
    elif kind == "signed_zero":
        f = rng.integers(-1, 2, size=n).astype(np.float64) * 0.0
        f[rng.random(n) < 0.5] = -0.0
        f[rng.random(n) < 0.3] = 1.0
        return np.asarray(f, np.float32), list(dims)
    elif kind == "const":
        f = np.zeros(n)
    else:
        raise ValueError(kind)
    return flat32(f), list(dims)


def random_csr(n: int, p: float, seed: int):
    """Erdos-Renyi style symmetric graph without self loops, sorted CSR."""
    rng = np.random.default_rng(seed)
    A = rng.random((n, n)) < p
    A = np.triu(A, 1)
    A = A | A.T
    rows = [np.nonzero(A[i])[0] for i in range(n)]
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col_idx = np.concatenate(rows).astype(np.int32) if row_ptr[-1] else np.zeros(0, np.int32)
    return row_ptr, col_idx
