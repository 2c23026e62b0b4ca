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


def test_term_slice_balanced():
    from paper_1505_00354_b200.distributed import term_slice
    for count in (0, 1, 5, 14, 74, 145):
        for world in (1, 2, 3, 4, 8):
            sl = [term_slice(count, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == count
            assert all(sl[r][1] == sl[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in sl]
            assert max(sizes) - min(sizes) <= 1 and max(sizes) == -(-count // world)
            sl2 = [term_slice(count, world, r, 2) for r in range(world)]
            assert sl2[0][0] == 0 and sl2[-1][1] == count
            assert all(sl2[r][1] == sl2[r + 1][0] for r in range(world - 1))
            assert all(lo % 2 == 0 for lo, hi in sl2 if hi > lo)


def test_weighted_slice_contiguous_and_balanced():
    """The asymptotic conversion's stage terms have unequal costs (60 (level,
    m) pairs of ~2 transforms, then ~7 recurrence bands of ~3 pairs each at
    2^26): contiguous slices covering all terms, each within one term's cost
    of the ideal share."""
    from paper_1505_00354_b200.distributed import weighted_slice
    rng = np.random.default_rng(0)
    cases = [[1.0] * 14, [1.86] * 60 + [5.7, 5.7, 5.8, 5.6, 5.7, 5.7, 3.8], list(rng.uniform(0.1, 3.0, 37)), [2.0]]
    for costs in cases:
        for world in (1, 2, 3, 4, 8):
            sl = [weighted_slice(costs, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == len(costs)
            assert all(sl[r][1] == sl[r + 1][0] for r in range(world - 1))
            share = sum(costs) / world
            for lo, hi in sl:
                assert sum(costs[lo:hi]) <= share + max(costs) + 1e-9
    with pytest.raises(ValueError):
        weighted_slice([1.0], 2, 2)


def _c4_worker(rank, world, port, out):
    """BASELINE C4's sharded data path (bench.py run_batched): contiguous
    column shards, inputs seeded per global column, one independent batched
    DLT per rank (no data collective), barrier + max over ranks. The device
    transform is stood in for by the CPU oracle's DLT on the same grid."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ORACLE as O, uniform_pm1
    n, total = 64, 11
    th, x, w = O.nodes_weights(n)
    first, cnt = column_shard(total, world, rank)
    cols = np.stack([uniform_pm1(n, 4000 + first + j) for j in range(cnt)]) if cnt else np.zeros((0, n))
    f = np.stack([O.dlt_grid(c, 1, 2.0 ** -52, th, x, w) for c in cols]) if cnt else np.zeros((0, n))
    dist.barrier()
    t = max_over_ranks(0.5 + rank, dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, f))
    if rank == 0:
        out.put((gathered, t))
    dist.barrier()
    dist.destroy_process_group()


def test_c4_sharded_data_path_two_ranks():
    from oracle import ORACLE as O, uniform_pm1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 1.5
    n, total = 64, 11
    th, x, w = O.nodes_weights(n)
    full = np.stack([O.dlt_grid(uniform_pm1(n, 4000 + j), 1, 2.0 ** -52, th, x, w) for j in range(total)])
    got = np.concatenate([f for _, f in sorted(gathered, key=lambda g: g[0])])
    assert np.array_equal(got, full)


def _c5_worker(rank, world, port, out):
    """BASELINE C5's term-parallel DLT / IDLT (distributed.transform, the
    bench's C5 call sequence) over gloo, with CPU stand-ins that compute the
    real stage arithmetic as sums of independent terms: the conversion as
    the direct product split by column blocks of M (transforms.hpp:47,
    conversion.hpp:100-140), the NDCT as its Taylor terms (ndct.hpp:98-143,
    oracle/ndct_np.py); the inverse with (m + 1/2) M^T and the weighted
    NDCT^T (transforms.hpp:58-62)."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ORACLE as O, ndct_np as NP
    from paper_1505_00354_b200 import distributed as D
    n, kind, blocks = 96, 1, 7
    th, x, w = O.nodes_weights(n)
    L = O.min_taylor_terms(kind, 2.0 ** -52)
    delta = O.reference_delta(n, kind, th)
    M = np.stack([O.leg2cheb(np.eye(n)[j]) for j in range(n)], axis=1)  # column j = M e_j
    edges = np.linspace(0, n, blocks + 1).astype(int)
    half = np.arange(n) + 0.5

    def stage_fn(inverse, stage, lo, hi, xin, y):
        v = xin.numpy()
        if stage == D.STAGE_LEG2CHEB:
            acc = np.zeros(n)
            for b in range(lo, hi):
                sl = slice(edges[b], edges[b + 1])
                acc += (half[:, None] * M.T[:, sl]) @ v[sl] if inverse else M[:, sl] @ v[sl]
        else:
            acc = (NP.ndct_apply_transpose(w * v, kind, hi, delta, lo) if inverse
                   else NP.ndct_apply(v, kind, hi, delta, lo)) if hi > lo else np.zeros(n)
        y.copy_(torch.from_numpy(acc))

    c = torch.from_numpy(O.random_decaying(n, 0.5, 7))
    counts = (blocks, L)
    f = D.transform(c, False, dist, counts=counts, stage_fn=stage_fn)
    f_part = D.transform(c, False, dist, counts=counts, stage_fn=stage_fn, scatter=True)
    back = D.transform(f, True, dist, counts=counts, stage_fn=stage_fn)
    gathered = [None] * world
    dist.all_gather_object(gathered, f_part.numpy())
    if rank == 0:
        out.put((c.numpy(), f.numpy(), np.concatenate(gathered), back.numpy(), th, x, w))
    dist.barrier()
    dist.destroy_process_group()


def test_c5_term_parallel_stages_two_ranks():
    from oracle import ORACLE as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    c, f, f_sc, back, th, x, w = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = len(c)
    tol = 1e-13 * np.log2(n)
    ref_f = O.dlt_grid(c, 1, 2.0 ** -52, th, x, w)
    assert np.max(np.abs(f - ref_f)) <= tol * np.abs(c).sum()
    assert np.array_equal(f_sc, f)
    ref_b = O.idlt_grid(f, 1, 2.0 ** -52, th, x, w)
    assert np.max(np.abs(back - ref_b)) <= tol * np.abs(f).sum()


def _fs_worker(rank, world, port, out):
    """BASELINE C5 sharded as the distributed four-step (distributed.
    dlt_four_step / idlt_four_step: the all-gather of the coefficient blocks,
    the conversion's term slice, the reduce-scatter into the residue layout,
    the term-group all-to-alls, the value all-to-all into natural blocks) over
    gloo with the real collectives; the rank-local halves are the NumPy
    restatement of the fl_fs_* kernels (tests/fourstep_np.py), the conversion
    the direct product split by column blocks of M."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ORACLE as O
    from paper_1505_00354_b200 import distributed as D
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from fourstep_np import FourStepNP
    n, blocks = 1024, 7
    th, x, w = O.nodes_weights(n)
    delta = O.reference_delta(n, 0, th)  # cheb1 offsets: the nodes about the cheb1 angles
    M = np.stack([O.leg2cheb(np.eye(n)[j]) for j in range(n)], axis=1)
    edges = np.linspace(0, n, blocks + 1).astype(int)
    half = np.arange(n) + 0.5

    def stage_fn(inverse, stage, lo, hi, xin, y):
        assert stage == D.STAGE_LEG2CHEB
        v = xin.numpy()
        acc = np.zeros(n)
        for b in range(lo, hi):
            sl = slice(edges[b], edges[b + 1])
            acc += (half[:, None] * M.T[:, sl]) @ v[sl] if inverse else M[:, sl] @ v[sl]
        y.copy_(torch.from_numpy(acc))

    fs = FourStepNP(n, world, rank, delta, w)
    groups = [(0, 5), (5, 10), (10, 14)]
    rng = D.term_slice(blocks, world, rank)
    c = O.random_decaying(n, 0.5, 7)
    B = n // world
    f_blk = D.dlt_four_step(None, torch.from_numpy(c[rank * B:(rank + 1) * B].copy()), dist, fs=fs,
                            groups=groups, stage_fn=stage_fn, conv_range=rng)
    f_all = [None] * world
    dist.all_gather_object(f_all, f_blk.numpy())
    f = np.concatenate(f_all)
    b_blk = D.idlt_four_step(None, torch.from_numpy(f[rank * B:(rank + 1) * B].copy()), dist, fs=fs,
                             groups=groups, stage_fn=stage_fn, conv_range=rng)
    b_all = [None] * world
    dist.all_gather_object(b_all, b_blk.numpy())
    if rank == 0:
        out.put((c, f, np.concatenate(b_all), th, x, w))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_c5_four_step_sharded_dlt_idlt(world):
    from oracle import ORACLE as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    c, f, back, th, x, w = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = len(c)
    tol = 1e-13 * np.log2(n)
    ref_f = O.dlt_grid(c, 1, 2.0 ** -52, th, x, w)
    assert np.max(np.abs(f - ref_f)) <= tol * np.abs(c).sum()
    ref_b = O.idlt_grid(f, 1, 2.0 ** -52, th, x, w)
    assert np.max(np.abs(back - ref_b)) <= tol * np.abs(f).sum()
