"""World-size-2 gloo tests of the multi-GPU host logic on CPU: instance
sharding, result gathering and loss reduction (no kernels run here)."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_06074_b200 import dist as sd


def test_shard_range_partitions():
    for n in (1, 2, 7, 1536, 4097):
        for world in (1, 2, 3, 8):
            spans = [sd.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3)
        local = sd.shard(full, rank, world) * 2.0          # stand-in for the per-shard solve
        got = sd.gather_instances(local, n)
        loss = sd.allreduce_loss(local.sum())
        mx = sd.max_over_ranks(float(rank + 1), "cpu")
        q.put((rank, torch.equal(got, full * 2.0), float(loss), mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 8])
def test_gather_and_reduce_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + n
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    full_sum = float(torch.arange(n * 3, dtype=torch.float64).sum() * 2.0)
    for rank, ok, loss, mx in res:
        assert ok and loss == full_sum and mx == 2.0
