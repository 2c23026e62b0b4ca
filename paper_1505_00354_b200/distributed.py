"""Multi-GPU DLT / IDLT of ONE large vector (BASELINE config C5, N = 2^26).

Both stages of the transform are sums of independent terms
(include/fastleg_b200.h, fl_dlt_stage):

  chat = M c       = sum_{r < K} D(l_r) T D(l_r) c     (Toeplitz-Hankel rank terms)
  f    = NDCT(chat) = sum_{m < M} W_m C_m T_m(n/N) chat  (Chebyshev-expansion terms
                                                        about cheb1, M = 14)

so each of P ranks (one process per GPU) evaluates a contiguous slice of the
terms on its own GPU -- full-length FFTs, no distributed FFT -- and one NCCL
collective per stage sums the partials over NVLink:

  chat = all_reduce(partial_leg2cheb)      (every rank needs all of chat)
  f    = all_reduce / reduce_scatter(partial_ndct)

Traffic per transform: 2 x N x 8 B per rank (1 GiB at N = 2^26) against
~K + 2L full-length FFT passes of compute split P ways. The inverse is the
same with the transposed stages in the opposite order.

`stage_fn` is injectable so the orchestration can be tested on CPU with gloo
(tests/test_multirank_cpu.py); on GPUs it is the C ABI (`gpu_stage`).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable

from . import _lib
from .shard import column_shard

STAGE_LEG2CHEB, STAGE_NDCT = 0, 1


def stage_terms(cfg, stage: int) -> int:
    out = C.c_int(0)
    _lib.check(_lib.LIB.fl_plan_stage_terms(cfg.handle, stage, C.byref(out)))
    return out.value


def gpu_stage(cfg, inverse: int, stage: int, lo: int, hi: int, x, y) -> None:
    """y = the partial sum of `stage` over terms [lo, hi) applied to x (CUDA
    float64 tensors of length N, on torch's current stream)."""
    import torch
    s = C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    _lib.check(_lib.LIB.fl_dlt_stage(cfg.handle, int(inverse), stage, lo, hi,
                                     C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), s))


def term_slice(count: int, world: int, rank: int, unit: int = 1) -> tuple[int, int]:
    """[lo, hi) of a stage's `count` equal-cost terms for `rank`: the first
    count % world ranks take one term more (a stage's time is its largest
    slice, ceil(count / world) terms; e.g. 14 NDCT terms over 8 ranks: 6 x 2 +
    2 x 1, bound 14 / 16 = 87.5 % of ideal; 74 rank terms: 2 x 10 + 6 x 9,
    92.5 %)."""
    if world <= 0 or not 0 <= rank < world or unit < 1:
        raise ValueError("term_slice: bad world/rank/unit")
    units = -(-count // unit)  # slices in whole units (the conversion's terms come in FFT pairs)
    base, extra = divmod(units, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return min(lo * unit, count), min(hi * unit, count)


def transform(x, inverse: bool, dist=None, *, counts: tuple[int, int],
              stage_fn: Callable, scatter: bool = False):
    """Term-parallel DLT (inverse = False) or IDLT (inverse = True) of x, the
    full input on every rank. Returns the full result on every rank, or with
    scatter=True this rank's contiguous block of it (reduce_scatter)."""
    import torch
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    order = (STAGE_NDCT, STAGE_LEG2CHEB) if inverse else (STAGE_LEG2CHEB, STAGE_NDCT)
    cur = x
    for step, stage in enumerate(order):
        # the conversion's rank terms share complex FFTs two at a time
        lo, hi = term_slice(counts[stage], world, rank, 2 if stage == STAGE_LEG2CHEB else 1)
        part = torch.empty_like(cur)
        stage_fn(int(inverse), stage, lo, hi, cur, part)
        last = step == len(order) - 1
        if world > 1:
            if last and scatter:
                n = part.numel()
                first, cnt = column_shard(n, world, rank)
                per = (n + world - 1) // world
                padded = torch.zeros(per * world, dtype=part.dtype, device=part.device)
                padded[:n] = part
                out = torch.empty(per, dtype=part.dtype, device=part.device)
                dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM)
                return out[:cnt]
            dist.all_reduce(part, op=dist.ReduceOp.SUM)
        cur = part
    return cur


def dlt(cfg, x, dist=None, scatter: bool = False):
    counts = (stage_terms(cfg, STAGE_LEG2CHEB), stage_terms(cfg, STAGE_NDCT))
    return transform(x, False, dist, counts=counts, scatter=scatter,
                     stage_fn=lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))


def idlt(cfg, f, dist=None, scatter: bool = False):
    counts = (stage_terms(cfg, STAGE_LEG2CHEB), stage_terms(cfg, STAGE_NDCT))
    return transform(f, True, dist, counts=counts, scatter=scatter,
                     stage_fn=lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))
