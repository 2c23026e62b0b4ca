"""CPU, world_size 2 over gloo: the column sharding of the batched path and
the max-over-ranks timing reduction used by bench.py under torchrun. The data
path has no collective, so a rank's output must equal the single-process
result for the same global columns (inputs are seeded per global column)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_00354_b200.shard import column_shard, max_over_ranks


def test_column_shard_partitions():
    for total in (1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [column_shard(total, world, r) for r in range(world)]
            cover = [c for first, cnt in spans for c in range(first, first + cnt)]
            assert cover == list(range(total))
    with pytest.raises(ValueError):
        column_shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1505_00354_b200 as fl
    total, n = 10, 64
    first, cnt = column_shard(total, world, rank)
    x = fl.random_uniform_pm1(n, 4000 + first, batch=cnt).reshape(cnt, n)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, x))
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        out.put((gathered, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_match_single_process():
    import paper_1505_00354_b200 as fl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    full = fl.random_uniform_pm1(64, 4000, batch=10).reshape(10, 64)
    for first, x in gathered:
        assert np.array_equal(x, full[first:first + len(x)])


def _dist_worker(rank, world, port, out):
    """Term-parallel orchestration (paper_1505_00354_b200/distributed.py) over
    gloo with a CPU stand-in for the per-term device stages."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1505_00354_b200 import distributed as D
    n, counts = 10, (7, 5)
    rng = np.random.default_rng(0)  # identical term matrices on every rank
    mats = [torch.from_numpy(rng.standard_normal((counts[s], n, n))) for s in range(2)]

    def stage_fn(inverse, stage, lo, hi, x, y):
        a = mats[stage][lo:hi].sum(0) if hi > lo else torch.zeros(n, n, dtype=torch.float64)
        y.copy_((a.T if inverse else a) @ x)

    x = torch.from_numpy(np.random.default_rng(1).standard_normal(n))
    full = D.transform(x, False, dist, counts=counts, stage_fn=stage_fn)
    part = D.transform(x, False, dist, counts=counts, stage_fn=stage_fn, scatter=True)
    inv = D.transform(x, True, dist, counts=counts, stage_fn=stage_fn)
    gathered = [None] * world
    dist.all_gather_object(gathered, part.numpy())
    if rank == 0:
        out.put((full.numpy(), np.concatenate(gathered), inv.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_term_parallel_transform_two_ranks():
    import torch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, scattered, inv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    n, counts = 10, (7, 5)
    mats = [rng.standard_normal((counts[s], n, n)) for s in range(2)]
    x = np.random.default_rng(1).standard_normal(n)
    A, B = mats[0].sum(0), mats[1].sum(0)
    assert np.allclose(full, B @ (A @ x), rtol=1e-12, atol=1e-12)
    assert np.allclose(scattered, full, rtol=1e-12, atol=1e-12)
    assert np.allclose(inv, A.T @ (B.T @ x), rtol=1e-12, atol=1e-12)
