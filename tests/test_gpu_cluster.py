"""The super-tile kernel (2x2x2 tiles in a thread-block cluster, paths followed
through the siblings' shared memory) against the oracle and against the
plain per-tile kernel (the default; EG_CLUSTER=1 selects the cluster kernel), on grids with several clusters,
odd leftovers and tie-heavy values."""
import os

import numpy as np
import pytest

import eg_inputs as G
import oracle as O
from _parity import assert_graph_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2303_02724_b200 as eg
    return eg


def _ctx(eg, cluster: bool):
    # the switch is read when a context's tiled state is first used
    old = os.environ.get("EG_CLUSTER")
    os.environ["EG_CLUSTER"] = "1" if cluster else "0"
    try:
        c = eg.Context()
        import torch
        c.compute(torch.zeros(64 * 64 * 64, device="cuda"), dims=[64, 64, 64])
        return c
    finally:
        if old is None:
            os.environ.pop("EG_CLUSTER")
        else:
            os.environ["EG_CLUSTER"] = old


@pytest.mark.parametrize("dims,kind", [([192, 96, 96], "turb"), ([224, 112, 80], "int"), ([160, 96, 128], "normal"),
                                       ([192, 96, 96], "signed_zero")])
def test_cluster_supertiles(eg, dims, kind):
    import torch
    if kind == "turb":
        t, _ = G.turbulence(dims[0], seed=3, device="cuda", kc_div=12)
        f = t.cpu().numpy().reshape(dims[0], dims[0], dims[0])[: dims[2], : dims[1], : dims[0]].reshape(-1)
        f = np.ascontiguousarray(f)
    else:
        f, _ = G.random_field(dims, 4, kind)
    o = O.grid(f, dims)
    ft = torch.from_numpy(f).cuda()
    with _ctx(eg, True) as a:
        g = a.compute(ft, dims=dims, flags=eg.EG_RAW_ARCS)
        assert_graph_equal(g, o, raw=True, what=f"cluster {dims} {kind}")
        ea = a.stats()["n_exit_targets"]
    with _ctx(eg, False) as b:
        g2 = b.compute(ft, dims=dims)
        assert_graph_equal(g2, o, what=f"no cluster {dims} {kind}")
        eb = b.stats()["n_exit_targets"]
    # the super-tiles leave fewer exit targets to the global resolution
    assert ea <= eb


def test_cluster_with_virtual_slabs(eg):
    import torch
    dims = [192, 96, 192]
    f, _ = G.random_field(dims, 8, "normal")
    o = O.grid(f, dims)
    with _ctx(eg, True) as a:
        for k in (1, 2, 3):
            g = a.compute(torch.from_numpy(f).cuda(), dims=dims, flags=eg.EG_VIRTUAL_PARTS(k))
            assert_graph_equal(g, o, what=f"cluster + {k} slabs")
