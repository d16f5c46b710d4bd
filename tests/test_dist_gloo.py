"""Multi-process host logic on CPU (world size 2 and 4, gloo, 127.0.0.1).

The hot-path exchanges are NCCL inside libeg_b200.so and need GPUs; what runs
here is everything around them: the slab / range planner, the NCCL-id
bootstrap over torch.distributed (rank 0's eg_nccl_unique_id reaches every
rank byte for byte), the tiling check every rank can do locally, and the
max-over-ranks timing reduction bench.py uses.  Context creation itself must
fail loudly without a GPU (no CPU fallback).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_02724_b200 as eg
        out = {}
        # planner: every rank computes the same plan and takes its own slab
        plan = eg.plan_slabs(1024, world)
        z0, z1 = plan[rank]
        mine = torch.tensor([z0, z1], dtype=torch.int64)
        gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, mine)
        out["tiles"] = all(int(gathered[r][0]) == (int(gathered[r - 1][1]) if r else 0) for r in range(world)) and \
            int(gathered[-1][1]) == 1024 and all(int(g[1] - g[0]) >= 2 for g in gathered)
        # NCCL id bootstrap: rank 0's id reaches every rank unchanged
        box = [eg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, box[0])
        out["id_ok"] = len(box[0]) == 128 and all(i == ids[0] for i in ids)
        # bench.py's reduction: the step time is the max over ranks
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["max_ok"] = float(t.item()) == float(world)
        # no CPU fallback: a Context cannot be created without a GPU
        try:
            eg.init_distributed()
            out["no_fallback"] = torch.cuda.is_available()
        except eg.EgError:
            out["no_fallback"] = True
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert len(res) == world
    for r, out in res.items():
        assert out == {"tiles": True, "id_ok": True, "max_ok": True, "no_fallback": True}, (r, out)


def test_plan_slabs_properties():
    import paper_2303_02724_b200 as eg
    for D in (2, 5, 32, 1024, 1025):
        for W in (1, 2, 3, 8):
            if W > 1 and D < 2 * W:
                with pytest.raises(ValueError):
                    eg.plan_slabs(D, W)
                continue
            p = eg.plan_slabs(D, W)
            assert p[0][0] == 0 and p[-1][1] == D
            assert all(a[1] == b[0] for a, b in zip(p, p[1:]))
            sizes = [b - a for a, b in p]
            assert max(sizes) - min(sizes) <= 1
    r = eg.plan_ranges(1_000_000, 8)
    assert r[0][0] == 0 and r[-1][1] == 1_000_000 and all(a[1] == b[0] for a, b in zip(r, r[1:]))
