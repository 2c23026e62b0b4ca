"""Multi-GPU DLT / IDLT of ONE large vector (BASELINE config C5, N = 2^26).

Both stages of the transform are sums of independent terms
(include/fastleg_b200.h, fl_dlt_stage):

  chat = M c       = DCT-II( sum_{l,m} level l's term m + sum_b recurrence band b )
                     (the asymptotic expansion, power-of-two N >= 2^20; the
                      DCT-II is linear, so every partial ends with it), or
                   = sum_{r < K} D(l_r) T D(l_r) c     (Toeplitz-Hankel rank terms)
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


def stage_costs(cfg, stage: int, count: int) -> list[float]:
    """Relative cost of each term of a stage (fl_plan_stage_cost)."""
    out = []
    v = C.c_double(0.0)
    for t in range(count):
        _lib.check(_lib.LIB.fl_plan_stage_cost(cfg.handle, stage, t, C.byref(v)))
        out.append(v.value)
    return out


def weighted_slice(costs, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of a contiguous split of terms with unequal `costs`: rank r's
    slice ends at the first term whose prefix cost reaches (r + 1)/world of
    the total, rounded to the nearer boundary (the asymptotic conversion's
    (level, m) pairs and its heavier recurrence bands)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("weighted_slice: bad world/rank")
    n = len(costs)
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + float(c))
    total = pre[-1]

    def cut(r: int) -> int:  # boundary index for the r-th of world slices
        if r <= 0:
            return 0
        if r >= world:
            return n
        target = total * r / world
        i = 0
        while i < n and pre[i + 1] < target:
            i += 1
        # i: first term whose end reaches the target; choose the nearer edge
        return i + 1 if i < n and (pre[i + 1] - target) <= (target - pre[i]) else i

    lo, hi = cut(rank), cut(rank + 1)
    return lo, max(lo, hi)


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
              stage_fn: Callable, scatter: bool = False, costs=None):
    """Term-parallel DLT (inverse = False) or IDLT (inverse = True) of x, the
    full input on every rank. Returns the full result on every rank, or with
    scatter=True this rank's contiguous block of it (reduce_scatter).
    costs: per stage, None (equal terms) or each term's relative cost."""
    import torch
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    order = (STAGE_NDCT, STAGE_LEG2CHEB) if inverse else (STAGE_LEG2CHEB, STAGE_NDCT)
    cur = x
    for step, stage in enumerate(order):
        if costs is not None and costs[stage] is not None:
            lo, hi = weighted_slice(costs[stage], world, rank)
        else:
            # the Toeplitz-Hankel rank terms share complex FFTs two at a time
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


def _plan_split(cfg):
    counts = (stage_terms(cfg, STAGE_LEG2CHEB), stage_terms(cfg, STAGE_NDCT))
    cl = stage_costs(cfg, STAGE_LEG2CHEB, counts[0])
    # equal costs: Toeplitz-Hankel rank terms (sliced in FFT pairs)
    costs = (None if len(set(cl)) <= 1 else cl, None)
    return counts, costs


def dlt(cfg, x, dist=None, scatter: bool = False):
    counts, costs = _plan_split(cfg)
    return transform(x, False, dist, counts=counts, scatter=scatter, costs=costs,
                     stage_fn=lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))


def idlt(cfg, f, dist=None, scatter: bool = False):
    counts, costs = _plan_split(cfg)
    return transform(f, True, dist, counts=counts, scatter=scatter, costs=costs,
                     stage_fn=lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))
