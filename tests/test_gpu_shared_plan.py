"""One TransformConfig shared by several host threads, each on its own CUDA
stream, with the first use of the plan racing (the reference documents
TransformConfig as immutable and safe to share across threads,
transforms.hpp:20-30). The plan builds its data-independent tables on first
use -- the asymptotic conversion's chunk start states, the multi-pass NDCT's
weight / stage tables, the packed-order weights of the fused unpack -- under
its own locks and publishes them only once complete: every thread must get
the bits a single-threaded run of a fresh plan produces."""
import threading

import numpy as np
import pytest

import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu


def _run(cfg, c_dev, out, idx, barrier):
    import torch
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        barrier.wait()
        f = fl.dlt(c_dev, cfg)
        b = fl.idlt(f, cfg).values
        st.synchronize()
        out[idx] = (f.cpu().numpy().copy(), b.cpu().numpy().copy())


@pytest.mark.parametrize("n", [1 << 15, 1 << 17])
def test_first_use_from_four_threads_matches_single_thread(n):
    import torch
    c = fl.random_decaying(n, 1.0, 3)
    c_dev = torch.from_numpy(c).cuda()
    # single-threaded reference on its own fresh plan
    ref_cfg = fl.TransformConfig(n)
    f0 = fl.dlt(c_dev, ref_cfg)
    b0 = fl.idlt(f0, ref_cfg).values
    torch.cuda.synchronize()
    f0, b0 = f0.cpu().numpy().copy(), b0.cpu().numpy().copy()
    # a fresh plan, first used by four threads at once
    cfg = fl.TransformConfig(n)
    nthreads = 4
    out = [None] * nthreads
    barrier = threading.Barrier(nthreads)
    ts = [threading.Thread(target=_run, args=(cfg, c_dev, out, i, barrier)) for i in range(nthreads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(nthreads):
        assert out[i] is not None, f"thread {i} failed"
        assert np.array_equal(out[i][0], f0), f"thread {i}: dlt differs from the single-threaded run"
        assert np.array_equal(out[i][1], b0), f"thread {i}: idlt differs from the single-threaded run"
