"""GPU: the distributed four-step NDCT (C5 sharded over P ranks; fl_fs_* in
include/fastleg_b200.h, paper_1505_00354_b200/distributed.py).

P emulated ranks run one after another on one device: each rank's part 1
(pack, L2-point FFTs, twiddle) writes its exchange buffer, the test performs
the all-to-all by slicing those buffers exactly as all_to_all_single would,
then each rank's part 2 (L1-point FFTs, weighted unpack) runs -- no kernel
waits on another. The result, reassembled from the ranks' natural blocks,
is compared with the single-GPU NDCT stage and with the CPU oracle
(||gpu - oracle||_inf / ||input||_1 <= 1e-13 log2 N). A world-size-1 NCCL
group runs the real collective path of dlt_four_step / idlt_four_step."""
import math
import os
import socket

import numpy as np
import pytest

from oracle import CHEBSTAR, ORACLE as O
from oracle import ndct_np as NP
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import distributed as D

pytestmark = pytest.mark.gpu


def tol_n(n):
    return 1e-13 * math.log2(n)


def _a2a(sends, counts_send, world, nt):
    """all_to_all_single over emulated ranks: rank d receives, from every
    source s in order, the chunk s addressed to d (doubles: 2 per complex)."""
    import torch
    recvs = []
    for d in range(world):
        pieces = []
        for s in range(world):
            off = sum(2 * nt * c for c in counts_send[s][:d])
            pieces.append(sends[s][off:off + 2 * nt * counts_send[s][d]])
        recvs.append(torch.cat(pieces))
    return recvs


def _uniform_a2a(xs, world):
    import torch
    per = xs[0].numel() // world
    return [torch.cat([xs[s][d * per:(d + 1) * per] for s in range(world)]) for d in range(world)]


def emulated_ndct(cfg, chat_full, world, groups=None):
    """Forward four-step NDCT over `world` emulated ranks -> the full f."""
    import torch
    fss = [D.FourStep(cfg, world, r) for r in range(world)]
    slabs = fss[0].to_residue(chat_full)   # the reduce-scatter input of any rank
    chat = [slabs[r * fss[r].slab:(r + 1) * fss[r].slab] for r in range(world)]
    groups = groups or fss[0].groups()
    fx = [torch.empty(fss[r].B, dtype=torch.float64, device="cuda") for r in range(world)]
    for gi, (t0, t1) in enumerate(groups):
        nt = t1 - t0
        cnt = [fs.coef_counts(False, True) for fs in fss]
        sends = []
        for r, fs in enumerate(fss):
            send = torch.empty(2 * nt * sum(cnt[r]), dtype=torch.float64, device="cuda")
            work = torch.empty(2 * fs.work_elems(nt), dtype=torch.float64, device="cuda")
            fs.part(False, 1, t0, t1, chat[r], send, work)
            sends.append(send)
        recvs = _a2a(sends, cnt, world, nt)
        for r, fs in enumerate(fss):
            assert recvs[r].numel() == 2 * nt * sum(fs.coef_counts(False, False))
            work = torch.empty(2 * fs.work_elems(nt), dtype=torch.float64, device="cuda")
            fs.part(False, 2, t0, t1, recvs[r], fx[r], work, first=gi == 0)
    for fs in fss:
        fs.check(False, torch.device("cuda"))
    frecv = _uniform_a2a(fx, world)
    return torch.cat([fss[r].values(True, frecv[r]) for r in range(world)])


def emulated_ndct_t(cfg, f_full, world, groups=None):
    """Transposed four-step NDCT (quadrature weights folded in) -> the full result."""
    import torch
    fss = [D.FourStep(cfg, world, r) for r in range(world)]
    B = fss[0].B
    gx = [fss[r].values(False, f_full[r * B:(r + 1) * B].contiguous()) for r in range(world)]
    grecv = _uniform_a2a(gx, world)
    groups = groups or fss[0].groups()
    outs = [torch.zeros(fs.slab, dtype=torch.float64, device="cuda") for fs in fss]
    for gi, (t0, t1) in enumerate(groups):
        nt = t1 - t0
        cnt = [fs.coef_counts(True, True) for fs in fss]
        sends = []
        for r, fs in enumerate(fss):
            send = torch.empty(2 * nt * sum(cnt[r]), dtype=torch.float64, device="cuda")
            work = torch.empty(2 * fs.work_elems(nt), dtype=torch.float64, device="cuda")
            fs.part(True, 1, t0, t1, grecv[r], send, work)
            sends.append(send)
        recvs = _a2a(sends, cnt, world, nt)
        for r, fs in enumerate(fss):
            assert recvs[r].numel() == 2 * nt * sum(fs.coef_counts(True, False))
            work = torch.empty(2 * fs.work_elems(nt), dtype=torch.float64, device="cuda")
            fs.part(True, 2, t0, t1, recvs[r], outs[r], work, first=gi == 0)
    return fss[0].from_residue(torch.cat(outs))


@pytest.mark.parametrize("n", [1 << 15, 1 << 18, 1 << 20])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_four_step_ndct_matches_single_gpu_stage(n, world):
    import torch
    cfg = fl.TransformConfig(n)
    terms = D.stage_terms(cfg, D.STAGE_NDCT)
    c = torch.from_numpy(fl.random_decaying(n, 0.0, 77 + n)).cuda()
    t = tol_n(n)
    ref = torch.empty_like(c)
    D.gpu_stage(cfg, 0, D.STAGE_NDCT, 0, terms, c, ref)
    f = emulated_ndct(cfg, c, world)
    assert float((f - ref).abs().max() / c.abs().sum()) <= t
    ref_t = torch.empty_like(c)
    D.gpu_stage(cfg, 1, D.STAGE_NDCT, 0, terms, c, ref_t)
    g = emulated_ndct_t(cfg, c, world)
    assert float((g - ref_t).abs().max() / c.abs().sum()) <= t


@pytest.mark.parametrize("groups", [[(0, 14)], [(0, 5), (5, 10), (10, 14)], [(k, k + 1) for k in range(14)]])
def test_four_step_term_groups(groups):
    import torch
    n = 1 << 16
    cfg = fl.TransformConfig(n)
    assert D.stage_terms(cfg, D.STAGE_NDCT) == 14
    c = torch.from_numpy(fl.random_decaying(n, 0.0, 5)).cuda()
    ref = torch.empty_like(c)
    D.gpu_stage(cfg, 0, D.STAGE_NDCT, 0, 14, c, ref)
    f = emulated_ndct(cfg, c, 4, groups)
    assert float((f - ref).abs().max() / c.abs().sum()) <= tol_n(n)
    ref_t = torch.empty_like(c)
    D.gpu_stage(cfg, 1, D.STAGE_NDCT, 0, 14, c, ref_t)
    g = emulated_ndct_t(cfg, c, 4, groups)
    assert float((g - ref_t).abs().max() / c.abs().sum()) <= tol_n(n)


def test_four_step_ndct_vs_oracle_2_18():
    """The four-step NDCT / NDCT^T at 2^18 over 8 emulated ranks against the
    NumPy restatement of ndct.hpp:98-143 (the reference's chebstar angles)."""
    import torch
    n = 1 << 18
    cfg = fl.TransformConfig(n)
    plan = cfg.plan()
    delta = np.asarray(plan.reference.delta_theta)
    w = cfg.grid().weights
    c = fl.random_decaying(n, 0.0, 11)
    f = emulated_ndct(cfg, torch.from_numpy(c).cuda(), 8).cpu().numpy()
    ref = NP.ndct_apply(c, CHEBSTAR, plan.num_terms, delta)
    assert np.max(np.abs(f - ref)) / np.abs(c).sum() <= tol_n(n)
    g = emulated_ndct_t(cfg, torch.from_numpy(c).cuda(), 8).cpu().numpy()
    ref_t = NP.ndct_apply_transpose(w * c, CHEBSTAR, plan.num_terms, delta)
    assert np.max(np.abs(g - ref_t)) / np.abs(w * c).sum() <= tol_n(n)


def test_four_step_dlt_idlt_emulated_vs_oracle():
    """The whole sharded DLT / IDLT at 2^16 over 4 emulated ranks: each rank's
    conversion slice, the reduce-scatter of their residue slabs, the
    four-step NDCT; against the oracle's full DLT / IDLT on the same grid."""
    import torch
    n, world = 1 << 16, 4
    cfg = fl.TransformConfig(n)
    g = cfg.grid()
    c = fl.random_decaying(n, 1.0, 21)
    ct = torch.from_numpy(c).cuda()
    parts = []
    for r in range(world):
        lo, hi = D._conversion_slice(cfg, world, r)
        part = torch.empty_like(ct)
        D.gpu_stage(cfg, 0, D.STAGE_LEG2CHEB, lo, hi, ct, part)
        parts.append(part)
    chat = sum(parts)
    f = emulated_ndct(cfg, chat, world).cpu().numpy()
    ref = O.dlt_grid(c, CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
    assert np.max(np.abs(f - ref)) / np.abs(c).sum() <= tol_n(n)
    # IDLT of the oracle's values
    v = fl.random_decaying(n, 0.0, 22)
    gt = emulated_ndct_t(cfg, torch.from_numpy(v).cuda(), world)
    back = torch.zeros_like(gt)
    for r in range(world):
        lo, hi = D._conversion_slice(cfg, world, r)
        part = torch.empty_like(gt)
        D.gpu_stage(cfg, 1, D.STAGE_LEG2CHEB, lo, hi, gt, part)
        back += part
    ref_b = O.idlt_grid(v, CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
    assert np.max(np.abs(back.cpu().numpy() - ref_b)) / np.abs(v).sum() <= tol_n(n)


def test_four_step_nonfinite_and_shapes():
    import torch
    cfg = fl.TransformConfig(1 << 15)
    with pytest.raises(fl.InvalidArgument):
        D.FourStep(cfg, 3, 0)          # world not a power of two
    with pytest.raises(fl.InvalidArgument):
        D.FourStep(cfg, 128, 0)        # 2P > L1 = 128
    c = torch.from_numpy(fl.random_decaying(1 << 15, 0.0, 1)).cuda()
    c[123] = float("nan")
    with pytest.raises(fl.InvalidArgument, match="ndct_apply: non-finite input"):
        emulated_ndct(cfg, c, 2)
    # the flag is cleared after it is reported
    c[123] = 0.0
    emulated_ndct(cfg, c, 2)


def test_four_step_nccl_world_size_one():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << 16
        cfg = fl.TransformConfig(n)
        g = cfg.grid()
        c = fl.random_decaying(n, 0.5, 1)
        f = D.dlt_four_step(cfg, torch.from_numpy(c).cuda(), dist)
        ref = O.dlt_grid(c, CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        assert np.max(np.abs(f.cpu().numpy() - ref)) / np.abs(c).sum() <= tol_n(n)
        back = D.idlt_four_step(cfg, f, dist)
        ref_b = O.idlt_grid(f.cpu().numpy(), CHEBSTAR, fl.default_tolerance, g.theta, g.x, g.weights)
        assert np.max(np.abs(back.cpu().numpy() - ref_b)) / np.abs(f.cpu().numpy()).sum() <= tol_n(n)
    finally:
        dist.destroy_process_group()


def test_rank_buffers_match_numpy_restatement():
    """Every exchange buffer of the GPU halves equals the NumPy restatement's
    (tests/fourstep_np.py, which the gloo test runs under the real
    collectives) at 2^14 over 4 ranks: same layouts, same arithmetic."""
    import sys
    import torch
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from fourstep_np import FourStepNP
    n, world = 1 << 14, 4
    cfg = fl.TransformConfig(n)
    th = cfg.grid().theta
    delta = O.reference_delta(n, 0, th)
    w = cfg.grid().weights
    c = fl.random_decaying(n, 0.0, 9)
    ct = torch.from_numpy(c)
    scale = np.abs(c).sum()
    for r in range(world):
        g, h = D.FourStep(cfg, world, r), FourStepNP(n, world, r, delta, w)
        assert (g.slab, g.B, g.L1, g.L2, g.KB) == (h.slab, h.B, h.L1, h.L2, h.KB)
        assert g.coef_counts(False, True) == h.coef_counts(False, True)
        assert g.coef_counts(True, False) == h.coef_counts(True, False)
        slabs_g, slabs_h = g.to_residue(ct.cuda()).cpu(), h.to_residue(ct)
        assert torch.equal(slabs_g, slabs_h)
        mine = slabs_h[r * h.slab:(r + 1) * h.slab].contiguous()
        for t0, t1 in ((0, 6), (6, 14)):
            nt = t1 - t0
            for tr in (False, True):
                inp = mine if not tr else torch.from_numpy(c[:h.B].copy())
                size = 2 * nt * sum(h.coef_counts(tr, True))
                sg = torch.empty(size, dtype=torch.float64, device="cuda")
                sh = torch.empty(size, dtype=torch.float64)
                work = torch.empty(2 * g.work_elems(nt), dtype=torch.float64, device="cuda")
                g.part(tr, 1, t0, t1, inp.cuda(), sg, work)
                h.part(tr, 1, t0, t1, inp, sh, None)
                assert float((sg.cpu() - sh).abs().max()) <= 1e-12 * scale, (r, t0, tr)
        fxg = g.values(False, torch.from_numpy(c[:h.B].copy()).cuda()).cpu()
        fxh = h.values(False, torch.from_numpy(c[:h.B].copy()))
        assert torch.equal(fxg, fxh)
