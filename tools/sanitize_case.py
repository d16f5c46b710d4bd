"""One small invocation of the hot path, for compute-sanitizer runs
(tests/test_sanitizer.py): python tools/sanitize_case.py <case>

cases: c1 (2-D 64^2, generic + tiled), t64 (3-D 64^3 turbulence, tiled, and
2 virtual slabs), d5 (5-D 9^5, generic n-D kernels), knn (2,000-point kNN CSR
graph, plus eg_gradient).  Exits non-zero if the graph differs from the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import eg_inputs as G  # noqa: E402
import oracle as O  # noqa: E402
import paper_2303_02724_b200 as eg  # noqa: E402


def same(g, o):
    return (np.array_equal(g.maxima, o.maxima) and np.array_equal(g.saddles, o.saddles)
            and np.array_equal(g.arcs, o.arcs) and np.array_equal(g.labels.cpu().numpy().astype(np.int64), o.label))


def main(case):
    ok = True
    with eg.Context(0) as ctx:
        if case == "c1":
            f, dims = G.c1_gaussians(0, 4.0)
            o = O.grid(f, dims)
            t = torch.from_numpy(f).cuda()
            ok &= same(ctx.compute(t, dims=dims, flags=eg.EG_CHECK_NAN | eg.EG_RAW_ARCS), o)
            ok &= same(ctx.compute(t, dims=dims, flags=eg.EG_FORCE_GENERIC), o)
        elif case == "t64":
            t, dims = G.turbulence(64, seed=3, device="cpu", kc_div=8)
            f = t.numpy()
            o = O.grid(f, dims)
            t = torch.from_numpy(f).cuda()
            ok &= same(ctx.compute(t, dims=dims, flags=eg.EG_CHECK_NAN), o)
            ok &= same(ctx.compute(t, dims=dims, flags=eg.EG_VIRTUAL_PARTS(2)), o)
        elif case == "d5":
            f, dims = G.schwefel([9] * 5)
            o = O.grid(f, dims)
            ok &= same(ctx.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_CHECK_NAN), o)
        elif case == "knn":
            X, f = G.gmm_points(2000, seed=10)
            rp, ci = G.knn_csr(X, 16)
            o = O.csr(f, rp, ci)
            csr = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
            t = torch.from_numpy(f).cuda()
            ok &= same(ctx.compute(t, csr=csr, flags=eg.EG_CHECK_NAN | eg.EG_CHECK_CSR | eg.EG_RAW_ARCS), o)
            p, b = ctx.gradient(t, csr=csr)
            ok &= np.array_equal(p.cpu().numpy().astype(np.int64), o.ptr)
        else:
            raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"sanitize case {case}: {'ok' if ok else 'MISMATCH'}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
