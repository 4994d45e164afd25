"""Host logic of the multi-GPU path on CPU with world_size 2 over gloo:
image sharding, the plan broadcast and the one output gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_08314_b200.stack import broadcast_plan, gather_outputs, shard_range


def test_shard_range_partitions():
    for n in (1, 7, 256, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = broadcast_plan(["cpo", "im2col", "cps"] if rank == 0 else None)
        lo, hi = shard_range(n, world, rank)
        sizes = [shard_range(n, world, r)[1] - shard_range(n, world, r)[0] for r in range(world)]
        # each rank "computes" its images: image i carries the value i everywhere
        y = torch.arange(lo, hi, dtype=torch.float32).reshape(-1, 1, 1, 1).expand(-1, 3, 2, 2).contiguous()
        out = gather_outputs(y, sizes)
        q.put((rank, plan, out.shape, out[:, 0, 0, 0].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [8, 7])
def test_gloo_world2_plan_and_gather(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, plan, shape, vals in res:
        assert plan == ["cpo", "im2col", "cps"]
        assert tuple(shape) == (n, 3, 2, 2)
        assert np.array_equal(vals, np.arange(n))


def _plan_worker(rank, world, port, path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_08314_b200.stack import load_plan, save_plan
        names = [f"L{i:02d}" for i in range(16)]
        if rank == 0:   # the offline selection runs once, on rank 0, and persists the plan
            save_plan(path, names, ["im2col"] * 8 + ["cpo"] * 4 + ["cps"] * 4, "best_of_three",
                      times_ms=[[1.0, 2.0, 3.0]] * 16)
        dist.barrier()  # control plane only; the plan itself travels through the file
        q.put((rank, load_plan(path, names)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plan_file(tmp_path):
    """the per-layer plan is computed once (rank 0) and READ FROM A PLAN FILE
    by every rank -- no collective carries it."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = str(tmp_path / "plan.json")
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = ["im2col"] * 8 + ["cpo"] * 4 + ["cps"] * 4
    assert all(plan == want for _, plan in res)
    from paper_2104_08314_b200.stack import load_plan
    with pytest.raises(ValueError):
        load_plan(path, [f"X{i}" for i in range(16)])
