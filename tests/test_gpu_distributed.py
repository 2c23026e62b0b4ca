"""GPU: the term-parallel multi-GPU DLT/IDLT pieces (fl_dlt_stage,
paper_1505_00354_b200/distributed.py) on one device: the rank slices of each
stage sum to the full stage (emulated ranks run one after another -- no
kernel waits on another), and a world_size-1 NCCL process group runs the
real collective path."""
import math
import os
import socket

import numpy as np
import pytest

import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import distributed as D

pytestmark = pytest.mark.gpu


def _cfg(n):
    return fl.TransformConfig(n)


@pytest.mark.parametrize("n", [1 << 15, 1 << 18])
def test_stage_slices_sum_to_full(n):
    import torch
    cfg = _cfg(n)
    c = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
    tol = 1e-13 * math.log2(n)
    for inverse in (0, 1):
        for stage in (D.STAGE_LEG2CHEB, D.STAGE_NDCT):
            count = D.stage_terms(cfg, stage)
            full = torch.empty_like(c)
            D.gpu_stage(cfg, inverse, stage, 0, count, c, full)
            for world in (2, 3, 8):
                acc = torch.zeros_like(c)
                for r in range(world):
                    lo, hi = D.term_slice(count, world, r)
                    part = torch.empty_like(c)
                    D.gpu_stage(cfg, inverse, stage, lo, hi, c, part)
                    acc += part
                err = float((acc - full).abs().max() / c.abs().sum())
                assert err <= tol, (inverse, stage, world, err)
    # the staged composition is the library's own dlt / idlt
    f = D.dlt(cfg, c)
    ref = fl.dlt(c, cfg)
    assert float((f - ref).abs().max() / c.abs().sum()) <= tol
    back = D.idlt(cfg, f)
    assert float((back - fl.idlt(f, cfg).values).abs().max() / f.abs().sum()) <= tol


def test_nccl_world_size_one():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << 15
        cfg = _cfg(n)
        c = torch.from_numpy(fl.random_decaying(n, 0.5, 1)).cuda()
        f = D.dlt(cfg, c, dist)
        part = D.dlt(cfg, c, dist, scatter=True)
        assert torch.equal(f, part)
        assert float((f - fl.dlt(c, cfg)).abs().max() / c.abs().sum()) <= 1e-13 * 15
    finally:
        dist.destroy_process_group()
