"""Multi-GPU DLT / IDLT of ONE large vector (BASELINE config C5, N = 2^26).

Both stages of the transform are sums of independent terms
(include/fastleg_b200.h, fl_dlt_stage):

  chat = M c       = DCT-II( sum_{l,m} level l's term m + sum_b recurrence band b )
                     (the asymptotic expansion, power-of-two N >= 2^16; the
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


# ---------------------------------------------------------------------------
# Distributed four-step NDCT (the sharded form of C5 north_star names): the
# input and output of the NDCT stage are spread over the ranks and each
# term's N/2-point FFT is a four-step whose two FFT stages are separated by
# ONE NCCL all-to-all per group of terms (include/fastleg_b200.h, fl_fs_*).
# The conversion stays term-parallel (its partials are full-length), but its
# all-reduce becomes a reduce-scatter straight into the four-step's residue
# layout, and the result leaves through a uniform all-to-all into natural
# blocks of N/P:
#
#   dlt :  c (block) -all_gather-> c -> partial M c (term slice) -reduce_scatter->
#          chat (residue layout) -> [pack, L2-FFTs, twiddle] -all_to_all->
#          [L1-FFTs, weighted unpack] -all_to_all-> f (block)
#   idlt:  f (block) -all_to_all-> [weighted pack, L1-FFTs, twiddle] -all_to_all->
#          [L2-FFTs, unpack] -> g (residue layout) -all_gather-> g -> partial
#          M^T g (term slice) -reduce_scatter-> c (block)
#
# The all-to-all of term group j runs on NCCL's stream while part 1 of group
# j + 1 runs on the compute stream.
# ---------------------------------------------------------------------------
class FourStep:
    """Rank-local half of the distributed four-step NDCT (fl_fs_*)."""

    def __init__(self, cfg, world: int, rank: int):
        import torch
        self.cfg = cfg
        h = C.c_void_p()
        _lib.check(_lib.LIB.fl_fs_create(cfg.handle, int(world), int(rank), C.byref(h)))
        self.handle = h
        info = (C.c_size_t * 10)()
        _lib.check(_lib.LIB.fl_fs_info(h, info))
        (self.n, self.L, self.L1, self.L2, self.KB, self.B, self.nres, self.res_max,
         self.world, self.rank) = (int(v) for v in info)
        self.slab = self.res_max * 2 * self.L2    # doubles per rank of the residue slabs
        self.res_len = self.nres * 2 * self.L2    # valid doubles of this rank's slab
        self.terms = stage_terms(cfg, STAGE_NDCT)
        self._torch = torch

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.LIB.fl_fs_destroy(self.handle)
            self.handle = None

    def _s(self, dev):
        return C.c_void_p(self._torch.cuda.current_stream(dev).cuda_stream)

    def coef_counts(self, transpose: bool, send: bool) -> list[int]:
        """Complex entries per term exchanged with each peer (part 1 -> part 2)."""
        out = []
        v = C.c_size_t(0)
        for peer in range(self.world):
            _lib.check(_lib.LIB.fl_fs_coef_count(self.handle, int(transpose), peer, int(send), C.byref(v)))
            out.append(int(v.value))
        return out

    def work_elems(self, terms: int) -> int:
        return int(_lib.LIB.fl_fs_work_elems(self.handle, int(terms)))

    def groups(self, budget_bytes: int = 12 << 30, min_groups: int = 1) -> list[tuple[int, int]]:
        """Term groups: work + two send + two receive buffers per group within
        the budget (two groups in flight)."""
        per_term = 16 * self.work_elems(1) * 5
        g = max(min_groups, -(-self.terms * per_term // max(1, budget_bytes)))
        g = min(g, self.terms)
        size = -(-self.terms // g)
        return [(t, min(t + size, self.terms)) for t in range(0, self.terms, size)]

    def to_residue(self, full):
        slabs = self._torch.empty(self.world * self.slab, dtype=full.dtype, device=full.device)
        _lib.check(_lib.LIB.fl_fs_to_residue(self.handle, C.c_void_p(full.data_ptr()),
                                             C.c_void_p(slabs.data_ptr()), self._s(full.device)))
        return slabs

    def from_residue(self, slabs):
        full = self._torch.empty(self.n, dtype=slabs.dtype, device=slabs.device)
        _lib.check(_lib.LIB.fl_fs_from_residue(self.handle, C.c_void_p(slabs.data_ptr()),
                                               C.c_void_p(full.data_ptr()), self._s(slabs.device)))
        return full

    def values(self, to_block: bool, x):
        out = self._torch.empty(self.B, dtype=x.dtype, device=x.device)
        _lib.check(_lib.LIB.fl_fs_values(self.handle, int(to_block), C.c_void_p(x.data_ptr()),
                                         C.c_void_p(out.data_ptr()), self._s(x.device)))
        return out

    def part(self, transpose: bool, part: int, t0: int, t1: int, inp, out, work, first: bool = True):
        _lib.check(_lib.LIB.fl_fs_ndct_part(self.handle, int(transpose), int(part), int(t0), int(t1),
                                            C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()),
                                            C.c_void_p(work.data_ptr()), int(first), self._s(inp.device)))

    def check(self, transpose: bool, dev) -> None:
        _lib.check(_lib.LIB.fl_fs_check(self.handle, int(transpose), self._s(dev)))


class TorchComm:
    """The collectives of the four-step path over a torch.distributed group
    (NCCL on GPUs); world 1 without a group is the identity."""

    def __init__(self, dist=None):
        self.dist = dist if dist is not None and dist.is_initialized() else None
        self.world = self.dist.get_world_size() if self.dist else 1
        self.rank = self.dist.get_rank() if self.dist else 0

    def all_gather(self, x):
        if self.world == 1:
            return x
        import torch
        out = torch.empty(x.numel() * self.world, dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(out, x)
        return out

    def reduce_scatter(self, x):
        if self.world == 1:
            return x
        import torch
        out = torch.empty(x.numel() // self.world, dtype=x.dtype, device=x.device)
        self.dist.reduce_scatter_tensor(out, x, op=self.dist.ReduceOp.SUM)
        return out

    def all_to_all(self, out, x, out_splits=None, in_splits=None):
        """Returns a handle with .wait() (async where the backend allows)."""
        if self.world == 1:
            if out.data_ptr() != x.data_ptr():
                out.copy_(x)
            return _Done()
        return self.dist.all_to_all_single(out, x, out_splits, in_splits, async_op=True)


class _Done:
    def wait(self):
        return None


def _pipeline(fs: FourStep, comm, transpose: bool, groups, inp, out):
    """Part 1 of every term group, its all-to-all, part 2: the all-to-all of
    group j runs on NCCL's stream while part 1 of group j + 1 runs on the
    compute stream (double-buffered); at world 1 the exchange is the
    identity and part 2 follows part 1 in place."""
    import torch
    dev = inp.device
    tmax = max(t1 - t0 for t0, t1 in groups)
    work = torch.empty(2 * fs.work_elems(tmax), dtype=torch.float64, device=dev)
    s_cnt, r_cnt = fs.coef_counts(transpose, True), fs.coef_counts(transpose, False)
    multi = comm.world > 1
    bufs = [(torch.empty(2 * tmax * sum(s_cnt), dtype=torch.float64, device=dev),
             torch.empty(2 * tmax * sum(r_cnt) if multi else 0, dtype=torch.float64, device=dev))
            for _ in range(2 if multi else 1)]
    first = groups[0][0]
    pending = None
    for gi, (t0, t1) in enumerate(groups):
        nt = t1 - t0
        send, recv = bufs[gi % len(bufs)]
        send = send[:2 * nt * sum(s_cnt)]
        fs.part(transpose, 1, t0, t1, inp, send, work)
        if not multi:
            fs.part(transpose, 2, t0, t1, send, out, work, first=t0 == first)
            continue
        recv = recv[:2 * nt * sum(r_cnt)]
        h = comm.all_to_all(recv, send, [2 * nt * c for c in r_cnt], [2 * nt * c for c in s_cnt])
        if pending is not None:
            ph, prec, p0, p1 = pending
            ph.wait()
            fs.part(transpose, 2, p0, p1, prec, out, work, first=p0 == first)
        pending = (h, recv, t0, t1)
    if pending is not None:
        ph, prec, p0, p1 = pending
        ph.wait()
        fs.part(transpose, 2, p0, p1, prec, out, work, first=p0 == first)
    fs.check(transpose, dev)


def _ndct_four_step(fs: FourStep, comm, chat_res, groups):
    """Forward NDCT: residue-layout chat -> this rank's natural block of f."""
    import torch
    fx = torch.empty(fs.B, dtype=torch.float64, device=chat_res.device)
    _pipeline(fs, comm, False, groups, chat_res, fx)
    frecv = torch.empty_like(fx) if comm.world > 1 else fx
    comm.all_to_all(frecv, fx).wait()
    return fs.values(True, frecv)


def _ndct_t_four_step(fs: FourStep, comm, f_block, groups):
    """Transposed NDCT (with the quadrature weights): this rank's natural
    block of f -> residue-layout result."""
    import torch
    gx = fs.values(False, f_block)
    grecv = torch.empty_like(gx) if comm.world > 1 else gx
    comm.all_to_all(grecv, gx).wait()
    out = torch.zeros(fs.slab, dtype=torch.float64, device=f_block.device)
    _pipeline(fs, comm, True, groups, grecv, out)
    return out


def _conversion_slice(cfg, world: int, rank: int):
    counts, costs = _plan_split(cfg)
    if costs[STAGE_LEG2CHEB] is not None:
        return weighted_slice(costs[STAGE_LEG2CHEB], world, rank)
    return term_slice(counts[STAGE_LEG2CHEB], world, rank, 2)


def dlt_four_step(cfg, c_block, dist=None, fs=None, groups=None, stage_fn=None, conv_range=None):
    """DLT of one vector whose coefficients are spread over the ranks in
    natural blocks of N/P (c_block: this rank's); returns this rank's block of
    f. The NDCT is the distributed four-step; the conversion term-parallel.
    fs / stage_fn / conv_range are injectable (CPU stand-ins over gloo in
    tests/test_multirank_cpu.py); by default the C ABI on this rank's GPU."""
    import torch
    comm = TorchComm(dist)
    fs = fs or FourStep(cfg, comm.world, comm.rank)
    groups = groups or fs.groups(min_groups=2 if comm.world > 1 else 1)
    stage_fn = stage_fn or (lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))
    lo, hi = conv_range or _conversion_slice(cfg, comm.world, comm.rank)
    c = comm.all_gather(c_block)
    part = torch.empty_like(c)
    stage_fn(0, STAGE_LEG2CHEB, lo, hi, c, part)
    chat = comm.reduce_scatter(fs.to_residue(part))
    return _ndct_four_step(fs, comm, chat, groups)


def idlt_four_step(cfg, f_block, dist=None, fs=None, groups=None, stage_fn=None, conv_range=None):
    """IDLT of one vector whose values are spread over the ranks in natural
    blocks of N/P; returns this rank's block of the coefficients."""
    import torch
    comm = TorchComm(dist)
    fs = fs or FourStep(cfg, comm.world, comm.rank)
    groups = groups or fs.groups(min_groups=2 if comm.world > 1 else 1)
    stage_fn = stage_fn or (lambda inv, st, lo, hi, a, b: gpu_stage(cfg, inv, st, lo, hi, a, b))
    lo, hi = conv_range or _conversion_slice(cfg, comm.world, comm.rank)
    g = fs.from_residue(comm.all_gather(_ndct_t_four_step(fs, comm, f_block, groups)))
    part = torch.empty_like(g)
    stage_fn(1, STAGE_LEG2CHEB, lo, hi, g, part)
    return comm.reduce_scatter(part)
