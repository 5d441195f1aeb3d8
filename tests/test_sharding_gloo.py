"""CPU, world size 2 over gloo: the multi-GPU plumbing of bench.py.

Images are sharded by contiguous index range with no data-path collective;
the only collective is the MAX over ranks of the timed region. Here each rank
runs the oracle on its shard of a small seeded batch and the union of the
shards must equal the unsharded result, and the max-reduction must return the
slowest rank's time on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O

        n_total = 6
        lo, hi = bench.shard(n_total, world, rank)
        res = {}
        for i in range(lo, hi):
            a = O.seeded_u8_image(24, 16, 3, seed=20000 + i)
            res[i] = O.resize_u8(a, 12, 8)
        # the timing reduction bench.time_op uses: MAX over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.put((rank, lo, hi, res, float(t[0])))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_every_config_batch():
    for n_total in (1, 16, 32, 64, 512):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                lo, hi = bench.shard(n_total, world, r)
                got.extend(range(lo, hi))
            assert got == list(range(n_total))


@pytest.mark.timeout(300)
def test_two_rank_gloo_sharded_equals_unsharded():
    import oracle as O

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for rank, lo, hi, res, tmax in results:
        assert tmax == 2.0  # slowest rank's time on every rank
        assert sorted(res) == list(range(lo, hi))
        merged.update(res)
    assert sorted(merged) == list(range(6))
    for i in range(6):
        a = O.seeded_u8_image(24, 16, 3, seed=20000 + i)
        assert np.array_equal(merged[i], O.resize_u8(a, 12, 8))
