"""Benchmark: fp64 DLT coefficients/sec on B200 (BASELINE.json metric), with
the reference CPU path timed beside it.

Workload (BASELINE.json configs[3], "C4"): batched DLT, N = 4096, 65536
independent columns (2 GiB fp64 input), coefficients iid U[-1,1) from
std::mt19937_64(4000 + j), columns sharded evenly over the
ranks with no collective. One step = one DLT of this rank's shard through
the C ABI (fl_dlt) on device-resident input. `e2e` is the same call with
pinned HOST buffers (H2D + D2H inside the timed region). The other configs
(C1, C2, the C3 sweep 2^10..2^20, C5) are timed after the headline and
reported under "configs" in the same JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4|c1|c3|c5] [--cols C] [--no-configs] [--dry-run]

Multi-GPU: one rank per GPU. Under torchrun the ranks come from the
environment; `--gpus N` without WORLD_SIZE relaunches this script under
torch.distributed.run with N ranks. NCCL is used only for the barrier and
the max-over-ranks timing on the batched path (no data-path collective) and
for the term-parallel C5 stages. `--dry-run` runs the launch, the sharding
and the timing protocol over gloo on CPU without touching a GPU.

`--impl reference` times the reference's own CPU implementation (the
unmodified reference headers compiled in place, oracle/_ref, fr_batch: a
std::thread pool over columns sharing one TransformConfig) on all host
cores, one bounded sample of the same workload per step, with inputs made by
the oracle's generator (the product library is never loaded on that arm).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_TFLOPS = 37.0  # tools/fp64_peak.cu on this pool's B200 (profiles/r01_fp64_peak.log): DMMA 37.0, DFMA 33.7
DFMA_PEAK_TFLOPS = 33.7  # fp64 CUDA-core FMA peak (same log): the NDCT's FFT arithmetic runs there
INT8_PEAK_TOPS = 4450.0  # tools/tc_i8_peak.cu: tcgen05 kind::i8 M=128 N=256, dense (profiles/r01_tc_i8_peak.log)
INT8_N64_CAP_TOPS = 2849.0  # same, N=64 tiles (the split GEMM's shape): shared-memory operand bound
HBM_FALLBACK_GBS = 6650.0

CONFIGS = {
    # name: (N, total columns, generator, description)
    "c4": (4096, 65536, "uniform", "C4 batched DLT N=4096 x 65536 cols, U[-1,1)"),
    "c1": (1024, 1, "decay0.5", "C1 DLT N=1024, c_n = g_n/(n+1)^0.5"),
    "c3": (1 << 20, 1, "decay1", "C3 DLT N=2^20, c_n = g_n/(n+1)"),
    "c5": (1 << 26, 1, "c5", "C5 DLT N=2^26 (512 MiB), c_n = g_n e^{-n/N}, term-parallel over ranks"),
}
REF_SAMPLE_COLS = {"c4": 1024, "c1": 1, "c3": 1, "c5": 1}


def hbm_peak() -> float:
    if os.path.exists(MEASURED):
        return float(json.load(open(MEASURED))["hbm_gbs"])
    return HBM_FALLBACK_GBS


def config_dict(name: str, world: int, total: int) -> dict:
    """The `config` object: identical on both arms (same keys and values)."""
    n, _, _, desc = CONFIGS[name]
    d = {"workload": desc, "N": n, "columns": total,
         "grid": "chebstar (default TransformConfig)",
         "tolerance": "2^-52"}
    if name == "c4":
        d.update({"parallelism": f"column shards x{world}, no collective",
                  "l2": "inputs (2 GiB) larger than L2 (126 MB); no flush"})
    elif name == "c5":
        d.update({"parallelism": f"term-parallel x{world}", "l2": "512 MiB vectors > L2"})
    else:
        d.update({"parallelism": "single vector", "l2": "vector L2-resident between steps"})
    return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--cols", type=int, default=0, help="override total columns")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C2/C3/C5 sub-results")
    ap.add_argument("--c5-mode", choices=["term", "four_step"], default="term",
                    help="--config c5: term-parallel (full vector on every rank) or the sharded "
                         "distributed four-step NDCT (N/P per rank in and out)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch + sharding + timing protocol over gloo on CPU (no GPU)")
    return ap.parse_args()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run
    with N ranks (one per GPU) on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank: int, world: int) -> None:
    """The multi-rank protocol without a GPU: gloo group, this rank's column
    shard of the workload, the C5 term slices, barrier + max over ranks."""
    import torch.distributed as dist
    from paper_1505_00354_b200.shard import column_shard, max_over_ranks
    from paper_1505_00354_b200.distributed import term_slice
    if world > 1:
        dist.init_process_group("gloo")
    n, total, _, _ = CONFIGS[args.config]
    total = args.cols or total
    shard = column_shard(total, world, rank)
    terms = [term_slice(k, world, rank) for k in (73, 14)]
    t = time.perf_counter()
    if world > 1:
        dist.barrier()
    gathered = [None] * world
    rec = {"rank": rank, "pid": os.getpid(), "columns": list(shard), "c5_term_slices": terms}
    if world > 1:
        dist.all_gather_object(gathered, rec)
    else:
        gathered = [rec]
    ms = max_over_ranks((time.perf_counter() - t) * 1e3, dist if world > 1 else None)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": config_dict(args.config, world, total),
                          "ranks": gathered, "barrier_ms_max": ms}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class Clocks:
    """SM clock / throttle-reason sampling during the timed region (B200_PROFILING.md
    clocks line). NVML queries take microseconds, so the whole timed region is sampled
    every 5 ms; nvidia-smi (~100 ms per query) is the fallback when NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.stop_ev = index, [], threading.Event()
        self.source, self.nvml = "nvidia-smi", None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            try:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.masks = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.nvml, self.h, self.source = pynvml, h, "nvml"
        except Exception:
            self.nvml = None
        self.th = threading.Thread(target=self._run, daemon=True)

    def _sample(self):
        if self.nvml is not None:
            p = self.nvml
            sm = float(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            return [str(sm), str(self.max_mhz), ""] + ["Active" if r & m else "Not Active" for m in self.masks]
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        return [s.strip() for s in out.split(",")] if out else None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                row = self._sample()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            self.stop_ev.wait(0.005 if self.nvml is not None else 0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.th.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": reasons, "samples": len(self.rows),
                "source": self.source}


def make_inputs(cfg: str, n: int, col0: int, cols: int) -> np.ndarray:
    """The product library's host generator (our arm)."""
    import paper_1505_00354_b200 as fl
    gen = CONFIGS[cfg][2]
    if cols == 0:
        return np.empty((0, n))
    if gen == "uniform":
        return fl.random_uniform_pm1(n, 4000 + col0, batch=cols).reshape(cols, n)
    if gen == "c5":
        return (fl.random_decaying(n, 0.0, 5) * np.exp(-np.arange(n) / n)).reshape(1, n)
    decay = 0.5 if gen == "decay0.5" else 1.0
    seed = 1 if cfg == "c1" else 3
    return fl.random_decaying(n, decay, seed + col0, batch=cols).reshape(cols, n)


def oracle_inputs(cfg: str, n: int, col0: int, cols: int) -> np.ndarray:
    """The same bits from the CPU oracle's generators (reference arm and CPU
    baseline: the product library is not loaded there)."""
    import oracle
    gen = CONFIGS[cfg][2]
    x = np.empty((cols, n))
    for j in range(cols):
        if gen == "uniform":
            x[j] = oracle.uniform_pm1(n, 4000 + col0 + j)
        elif gen == "c5":
            x[j] = oracle.ORACLE.random_decaying(n, 0.0, 5) * np.exp(-np.arange(n) / n)
        else:
            decay = 0.5 if gen == "decay0.5" else 1.0
            seed = 1 if cfg == "c1" else 3
            x[j] = oracle.ORACLE.random_decaying(n, decay, seed + col0 + j)
    return x


class RefBatch:
    """The reference's CPU DLT over a column block: oracle/_ref's fr_batch,
    stock fastleg::dlt on one shared TransformConfig (transforms.hpp:15-18),
    `threads` host threads over the columns."""

    def __init__(self, n: int, tol: float = 2.0 ** -52, kind: int = 1):
        import ctypes as C
        from oracle import _ref
        if _ref is None:
            raise RuntimeError("oracle/_ref is not built (python -c 'import __graft_entry__ as g; g.build()')")
        self.C, self.lib, self.n = C, _ref, n
        vp, sz, i, d = C.c_void_p, C.c_size_t, C.c_int, C.c_double
        _ref.fr_config_create.argtypes = [sz, d, i, C.POINTER(vp)]
        _ref.fr_config_create.restype = i
        _ref.fr_batch.argtypes = [vp, i, sz, sz, vp, vp, i]
        _ref.fr_batch.restype = i
        _ref.fr_config_destroy.argtypes = [vp]
        self.h = vp()
        t0 = time.perf_counter()
        assert _ref.fr_config_create(n, tol, kind, C.byref(self.h)) == 0
        self.config_s = time.perf_counter() - t0

    def dlt(self, x: np.ndarray, y: np.ndarray, threads: int) -> float:
        """Seconds for the DLT of every row of x into y."""
        vp = self.C.c_void_p
        t0 = time.perf_counter()
        rc = self.lib.fr_batch(self.h, 0, x.shape[0], self.n, vp(x.ctypes.data), vp(y.ctypes.data), threads)
        dt = time.perf_counter() - t0
        assert rc == 0
        return dt

    def close(self):
        self.lib.fr_config_destroy(self.h)


def cpu_baseline(cfg: str, n: int, budget_s: float, threads: int) -> dict:
    """The reference's own CPU path on a bounded sample of the workload
    (about `budget_s` of CPU work), all `threads` host threads."""
    try:
        ref = RefBatch(n)
    except RuntimeError as e:
        return {"value": None, "unit": "coeffs/s", "cores": 0, "kind": "reference", "sample": str(e)}
    cols = REF_SAMPLE_COLS[cfg]
    if cfg == "c4":
        cols = max(threads, 1) * 16
    x = oracle_inputs(cfg, n, 0, cols)
    y = np.empty_like(x)
    ref.dlt(x, y, threads)  # warm-up (plan caches, page faults)
    done, elapsed = 0, 0.0
    while elapsed < budget_s:
        elapsed += ref.dlt(x, y, threads)
        done += cols
        if n > 8192:
            break
    ref.close()
    return {"value": done * n / elapsed, "unit": "coeffs/s", "cores": threads, "kind": "reference",
            "sample": f"{done} columns of N={n} in {elapsed:.1f} s ({cols} per call; TransformConfig build "
                      f"{ref.config_s:.2f} s excluded); reference headers compiled in place + FFTW-API shim "
                      "(FFTW absent)"}


def run_reference(args, rank: int, world: int) -> None:
    """`--impl reference`: rank 0 times the reference's CPU DLT, one bounded
    sample of the workload per step (REF_SAMPLE_COLS columns), on all host
    threads; the other ranks exit without work."""
    if rank != 0:
        return
    n, total, _, _ = CONFIGS[args.config]
    total = args.cols or total
    if n > 65536:
        print(json.dumps({"impl": "reference", "unavailable": f"the reference's O(N^2) conversion and node "
                          f"solver take minutes to days per transform at N={n} (SURVEY.md 6.2)"}))
        return
    threads = 1 if total == 1 else (os.cpu_count() or 1)
    cols = min(REF_SAMPLE_COLS[args.config], total)
    ref = RefBatch(n)
    x = oracle_inputs(args.config, n, 0, cols)
    y = np.empty_like(x)
    for _ in range(args.warmup):
        ref.dlt(x, y, threads)
    times = [ref.dlt(x, y, threads) for _ in range(args.steps)]
    ref.close()
    ms = 1e3 * float(np.mean(times))
    v = n * cols / (ms / 1e3)
    sample = (f"each step: the DLT of {cols} of the {total} columns (N={n}, columns 0..{cols - 1}); "
              f"{threads} host threads; reference headers compiled in place + FFTW-API shim (FFTW absent); "
              f"TransformConfig build {ref.config_s:.2f} s excluded")
    print(json.dumps({
        "metric": "fp64 DLT coeffs/sec", "value": v, "unit": "coeffs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "ms_per_step_basis": f"one step = {cols} columns (the timed sample)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": config_dict(args.config, world, total),
        "cpu_baseline": {"value": v, "unit": "coeffs/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "coeffs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def _timer(stream):
    import torch

    def timed(fn, reps=3, warm=1):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    return timed


def ndct_flops_per_coef(n: int, terms: int) -> float:
    """L (2.5 log2 N + 3) flop per coefficient (power-of-two N)."""
    return terms * (2.5 * math.log2(n) + 3)


def sub_configs(args, dist, rank: int, world: int, local: int) -> dict:
    """C1, C2, the C3 sweep and C5 (BASELINE.json configs), device-resident,
    CUDA events on the launching stream; the plan / TransformConfig is built
    once per size and timed separately. At world > 1 only C5
    (the one config that is sharded as a single transform) runs, over all
    ranks; the batched configs shard like C4."""
    import ctypes as C
    import torch
    import paper_1505_00354_b200 as fl
    from paper_1505_00354_b200 import _lib
    from paper_1505_00354_b200 import distributed as D
    from paper_1505_00354_b200.shard import max_over_ranks
    vp = C.c_void_p
    stream = torch.cuda.current_stream()
    sp = vp(stream.cuda_stream)
    timed = _timer(stream)
    peak = hbm_peak()
    out = {}

    def single(n, x, reps):
        t0 = time.perf_counter()
        cfg = fl.TransformConfig(n)
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        y, z = torch.empty_like(x), torch.empty_like(x)
        dlt = timed(lambda: _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, sp)), reps)
        idlt = timed(lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(y.data_ptr()), vp(z.data_ptr()), 1, n, sp)), reps)
        rt = float((z - x).abs().max() / x.abs().max())
        return cfg, {"N": n, "plan_s": plan_s, "dlt_ms": dlt, "idlt_ms": idlt,
                     "dlt_coeffs_per_s": n / dlt * 1e3, "idlt_coeffs_per_s": n / idlt * 1e3,
                     # single vector: the per-size tables are read too:
                     # +8 B (delta) for the DLT, +16 B (delta, w) for the IDLT
                     "dlt_hbm_frac": 24.0 * n / (dlt / 1e3) / 1e9 / peak,
                     "idlt_hbm_frac": 32.0 * n / (idlt / 1e3) / 1e9 / peak,
                     "leg2cheb": l2c_method(cfg, n),
                     "round_trip_rel": rt}

    def l2c_method(cfg, n):
        if n >= (1 << 16) and n & (n - 1) == 0:
            return "asymptotic expansion " + json.dumps(cfg.leg2cheb_asy_info())
        return "toeplitz-hankel" if cfg.leg2cheb_rank(0) else "direct"

    def conversions(n, reps):
        """The conversion alone, one vector: the asymptotic expansion against
        Toeplitz-Hankel (both directions)."""
        cfg = fl.TransformConfig(n)
        x = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
        y = torch.empty_like(x)
        r = {}
        for mode, name in ((fl.LEG2CHEB_TOEPLITZ, "toeplitz_hankel"), (fl.LEG2CHEB_ASYMPTOTIC, "asymptotic")):
            cfg.set_leg2cheb_mode(mode)
            for t in (0, 1):
                r[f"{name}{'_T' if t else ''}_ms"] = timed(lambda: _lib.check(_lib.LIB.fl_plan_leg2cheb(
                    cfg.handle, t, vp(x.data_ptr()), vp(y.data_ptr()), 1, n, sp)), reps)
        r["asymptotic_shape"] = cfg.leg2cheb_asy_info()
        return r

    if world == 1:
        # C1: one N = 1024 vector (latency-bound: one CTA runs all NDCT terms)
        n = 1024
        c = make_inputs("c1", n, 0, 1)
        _, r = single(n, torch.from_numpy(c[0].copy()).cuda(), 200)
        try:
            ref = RefBatch(n)
            y = np.empty_like(c)
            ref.dlt(c, y, 1)
            r["cpu_reference_dlt_ms_1core"] = 1e3 * float(np.median([ref.dlt(c, y, 1) for _ in range(20)]))
            ref.close()
        except RuntimeError:
            pass
        r["workload"] = CONFIGS["c1"][3]
        r["bound"] = "latency (one column: the direct method as two fp64 table row products, 4 MiB table in L2)"
        out["c1"] = r

        # C2: NDCT only, N = 65536 x 64 columns, iid N(0,1), the node kernel's grid
        n, cols = 65536, 64
        c2 = fl.random_decaying(n, 0.0, 1000, batch=cols)
        grid = fl.legendre_nodes_weights(n)
        x = torch.from_numpy(c2).cuda()
        y = torch.empty_like(x)
        r = {"workload": "C2 NDCT N=65536 x 64 cols, iid N(0,1), node-kernel grid", "N": n, "columns": cols}
        for kind in (fl.GridKind.chebstar, fl.GridKind.cheb1):
            plan = fl.plan_ndct(grid, kind, fl.default_tolerance)
            d = torch.from_numpy(np.asarray(plan.reference.delta_theta)).cuda()
            L = plan.num_terms
            f = timed(lambda: _lib.check(_lib.LIB.fl_ndct(0, int(kind), n, L, vp(d.data_ptr()), vp(x.data_ptr()),
                                                          vp(y.data_ptr()), cols, n, sp)), 5)
            t = timed(lambda: _lib.check(_lib.LIB.fl_ndct(1, int(kind), n, L, vp(d.data_ptr()), vp(x.data_ptr()),
                                                          vp(y.data_ptr()), cols, n, sp)), 5)
            r[kind.name] = {"L": L, "ndct_ms": f, "ndct_T_ms": t, "ndct_coeffs_per_s": n * cols / f * 1e3,
                            "ndct_T_coeffs_per_s": n * cols / t * 1e3,
                            "hbm_frac": 16.0 * n * cols / (f / 1e3) / 1e9 / peak,
                            "api": "free functions ndct_apply / _transpose (ndct.hpp:98-143): the "
                                   "expansion's tables are planned on every call"}
        # the same NDCT through a TransformConfig (planned once: the dlt's NDCT step)
        cfg2 = fl.TransformConfig(n)
        f = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg2.handle, 0, vp(x.data_ptr()), vp(y.data_ptr()),
                                                            cols, n, sp)), 5)
        t = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg2.handle, 1, vp(x.data_ptr()), vp(y.data_ptr()),
                                                            cols, n, sp)), 5)
        r["planned_chebstar"] = {"ndct_ms": f, "ndct_T_ms": t, "ndct_coeffs_per_s": n * cols / f * 1e3,
                                 "ndct_T_coeffs_per_s": n * cols / t * 1e3,
                                 "api": "fl_plan_ndct (TransformConfig planned once)"}
        out["c2"] = r

        # C3: the sweep N = 2^10 .. 2^20 (headline 2^20)
        sweep = []
        for lg in range(10, 21):
            n = 1 << lg
            c = fl.random_decaying(n, 1.0, 3)
            _, r = single(n, torch.from_numpy(c).cuda(), max(3, min(100, (1 << 22) // n)))
            sweep.append(r)
        out["c3"] = {"workload": CONFIGS["c3"][3] + ", sweep 2^10..2^20", "sweep": sweep}
        # the two fast conversions timed against each other (north-star subsystem 2)
        out["leg2cheb_methods"] = {"2^17": conversions(1 << 17, 20), "2^20": conversions(1 << 20, 5),
                                   "2^26": conversions(1 << 26, 2)}

    # C5: one 2^26 vector; term-parallel over the ranks (all ranks take part)
    n = CONFIGS["c5"][0]
    t0 = time.perf_counter()
    cfg = fl.TransformConfig(n)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    x = torch.from_numpy(make_inputs("c5", n, 0, 1)[0]).cuda()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    res = {}
    for name, fn in (("dlt", D.dlt), ("idlt", D.idlt)):
        for _ in range(2):
            fn(cfg, x, dist, scatter=True)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            fn(cfg, x, dist, scatter=True)
        e1.record(stream)
        barrier()
        res[name] = max_over_ranks(e0.elapsed_time(e1) / 3, dist, f"cuda:{local}")
    # the sharded form: coefficients / values in natural blocks of N/P per
    # rank, the NDCT as the distributed four-step (one NCCL all-to-all per
    # term group), the conversion term-parallel (distributed.dlt_four_step)
    fs = D.FourStep(cfg, world, rank)
    blk = x[rank * fs.B:(rank + 1) * fs.B].contiguous()
    fs_res = {}
    for name, fn in (("dlt", D.dlt_four_step), ("idlt", D.idlt_four_step)):
        for _ in range(2):
            fn(cfg, blk, dist, fs)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            fn(cfg, blk, dist, fs)
        e1.record(stream)
        barrier()
        fs_res[name] = max_over_ranks(e0.elapsed_time(e1) / 3, dist, f"cuda:{local}")
    del fs
    out["c5"] = {"workload": CONFIGS["c5"][3], "N": n, "n_gpus": world, "plan_s": plan_s,
                 "dlt_ms": res["dlt"], "idlt_ms": res["idlt"],
                 "four_step": {"dlt_ms": fs_res["dlt"], "idlt_ms": fs_res["idlt"],
                               "note": "sharded in / out (N/P per rank); NDCT as the distributed "
                                       "four-step with one all-to-all per term group"},
                 "dlt_coeffs_per_s": n / res["dlt"] * 1e3, "idlt_coeffs_per_s": n / res["idlt"] * 1e3,
                 "dlt_hbm_frac_per_gpu": 24.0 * n / (res["dlt"] / 1e3) / 1e9 / peak / world,
                 "leg2cheb": l2c_method(cfg, n),
                 "stage_terms": [D.stage_terms(cfg, 0), D.stage_terms(cfg, 1)]}
    return out if rank == 0 else {}


def run_c5(args, rank: int, world: int, local: int) -> None:
    """--config c5: one 2^26 DLT, its conversion (the asymptotic expansion's
    (level, m) terms and recurrence bands, split by cost) and NDCT
    (Chebyshev-expansion terms) split over the ranks, partials
    combined by NCCL all-reduce / reduce-scatter (distributed.py). Fixed N:
    strong scaling."""
    import torch
    import paper_1505_00354_b200 as fl
    from paper_1505_00354_b200 import distributed as D
    from paper_1505_00354_b200.shard import max_over_ranks
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = CONFIGS["c5"][0]
    cfg = fl.TransformConfig(n)
    xh = torch.from_numpy(make_inputs("c5", n, 0, 1)[0]).pin_memory()
    x = xh.cuda()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if args.c5_mode == "four_step":
        fs = D.FourStep(cfg, world, rank)
        sl = slice(rank * fs.B, (rank + 1) * fs.B)
        xh = xh[sl].contiguous().pin_memory()
        x = xh.cuda()

        def step(v):
            return D.dlt_four_step(cfg, v, dist, fs)
    else:
        def step(v):
            return D.dlt(cfg, v, dist, scatter=True)
    for _ in range(max(args.warmup, 3)):
        step(x)
    barrier()
    l0 = fl.launch_count()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(s)
        for _ in range(args.steps):
            step(x)
        e1.record(s)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, f"cuda:{local}")
    launches = fl.launch_count() - l0
    # e2e: the host vector in, this rank's block of f back to the host
    e0.record(s)
    for _ in range(2):
        xd = xh.cuda(non_blocking=True)
        part = step(xd)
        back = part.cpu()
    e1.record(s)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / 2, dist, f"cuda:{local}")
    if rank == 0:
        print(json.dumps({
            "metric": "fp64 DLT coeffs/sec", "value": n / (ms / 1e3), "unit": "coeffs/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict("c5", world, 1),
            "roofline": {"bound": "hbm", "achieved": 24.0 * n / (ms / 1e3) / 1e9, "peak": hbm_peak() * world,
                         "unit": "GB/s", "frac": 24.0 * n / (ms / 1e3) / 1e9 / (hbm_peak() * world),
                         "traffic": None, "note": "24 B/coef (c, f, delta) over the job"},
            "e2e": {"value": n / (e2e_ms / 1e3), "unit": "coeffs/s", "h2d_bytes_per_step": int(8 * xh.numel()),
                    "d2h_bytes_per_step": int(8 * back.numel())},
            "leg2cheb": "asymptotic expansion " + json.dumps(cfg.leg2cheb_asy_info()),
            "c5_mode": args.c5_mode,
            "gpu_launches": launches, "clocks": clk.summary()}))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_batched(args, rank: int, world: int, local: int) -> None:
    import ctypes
    import torch
    import paper_1505_00354_b200 as fl
    from paper_1505_00354_b200 import _lib
    from paper_1505_00354_b200.shard import column_shard, max_over_ranks

    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: rank {rank} needs cuda:{local}; only {torch.cuda.device_count()} GPU(s) visible")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, total, _, _ = CONFIGS[args.config]
    if args.cols:
        total = args.cols
    col0, cols = column_shard(total, world, rank)
    stream = torch.cuda.current_stream()
    vp = ctypes.c_void_p
    sp = vp(stream.cuda_stream)

    cfg = fl.TransformConfig(n)  # chebstar, tol 2^-52; plan built once, not timed
    x_host = make_inputs(args.config, n, col0, cols)
    x = torch.from_numpy(x_host).to(f"cuda:{local}")
    y = torch.empty_like(x)

    def step():
        _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()), cols, n, sp))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    l0 = fl.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    launches = fl.launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = max_over_ranks(ms, dist, f"cuda:{local}")
    value = n * total / (ms_max / 1e3)

    # ---- per-kernel split (same stream, CUDA events): the plan's two steps
    timed = _timer(stream)
    chat = torch.empty_like(x)
    # the plan's conversion step exactly as fl_dlt runs it (split-int8 tcgen05 GEMM)
    ms_l2c = timed(lambda: _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()),
                                                                vp(chat.data_ptr()), cols, n, sp)))
    # the plan's NDCT step exactly as fl_dlt runs it (fast mode: Chebyshev expansion)
    L1 = _lib.LIB.fl_plan_ndct_terms(cfg.handle)
    ms_ndct = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 0, vp(chat.data_ptr()),
                                                             vp(y.data_ptr()), cols, n, sp)))
    ms_dct = timed(lambda: _lib.check(_lib.LIB.fl_trig(0, fl.GridKind.cheb1, n, vp(x.data_ptr()),
                                                       vp(y.data_ptr()), cols, n, sp)))
    ms_dct_t = timed(lambda: _lib.check(_lib.LIB.fl_trig(2, fl.GridKind.cheb1, n, vp(x.data_ptr()),
                                                         vp(y.data_ptr()), cols, n, sp)))
    # the inverse on the same shard (DLT, IDLT and NDCT reported separately)
    ms_ndct_t = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 1, vp(x.data_ptr()),
                                                               vp(chat.data_ptr()), cols, n, sp)))
    ms_l2c_t = timed(lambda: _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 1, vp(chat.data_ptr()),
                                                                  vp(y.data_ptr()), cols, n, sp)))
    ms_idlt = timed(lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()),
                                                        cols, n, sp)))
    # the factored path (the reference's conversion + NDCT) on the same shard, as the ablation
    direct = cfg.uses_direct(cols)
    cfg.set_dlt_method(fl.DLT_FACTORED)
    ms_dlt_f = timed(lambda: _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()),
                                                        cols, n, sp)))
    ms_idlt_f = timed(lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()),
                                                          cols, n, sp)))
    cfg.set_dlt_method(fl.DLT_DIRECT)
    coef = n * cols
    l2c_flops = coef * (n / 2.0)                   # N^2/4 MACs per column = N/2 flop per coefficient
    ndct_flops = coef * ndct_flops_per_coef(n, L1)
    # int8 tensor work of the split product: 28 digit pairs x the 128-row-blocked
    # triangle (K from the diagonal block), 2 ops per MAC, both parities
    r_rows = n // 2
    rbs = r_rows // 128
    tri_macs = sum((r_rows - 128 * rb) * 128 for rb in range(rbs)) * 2 * cols
    i8_ops = 28 * 2 * tri_macs
    # the direct product: 28 digit pairs x 2 parities x (N/2)^2 MACs per column, 2 ops per MAC
    dense_ops = 28 * 2 * 2 * (n // 2) ** 2 * cols
    dense_tops = dense_ops / (ms / 1e3) / 1e12
    gemm_mode = cfg.gemm_mode()
    achieved = ndct_flops / (ms_ndct / 1e3) / 1e12
    peak = hbm_peak()
    # DRAM traffic of the NDCT kernel per launch, from the committed ncu
    # --set full capture (profiles/ncu_traffic.json: bytes per coefficient)
    traffic = dct_traffic = dense_traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        lg = int(math.log2(n))
        for name, rec in tj.items():
            if name.startswith("fast_ndct_fwd_kernel") and (f"<{lg}>" in name or f"<{lg}, 1>" in name):
                traffic = {"bytes_per_launch": rec["dram_bytes_per_coef"] * coef,
                           "bytes_per_coef": rec["dram_bytes_per_coef"],
                           "algorithmic_bytes_per_coef": 16.0, "source": rec["capture"]}
                break
        rec = tj.get(f"oz_gemm2_kernel(dense, N={n})")
        if rec:
            dense_traffic = {"bytes_per_launch": rec["dram_bytes_per_coef"] * coef,
                             "bytes_per_coef": rec["dram_bytes_per_coef"],
                             "algorithmic_bytes_per_coef": 16.0, "source": rec["capture"]}
        rec = tj.get(f"fast_dct_stream_fwd_kernel<{lg}>")
        if rec:
            dct_traffic = {"bytes_per_coef": rec["dram_bytes_per_coef"], "algorithmic_bytes_per_coef": 16.0,
                           "source": rec["capture"]}
    dct_gbs = 16.0 * coef / (ms_dct / 1e3) / 1e9
    dct_t_gbs = 16.0 * coef / (ms_dct_t / 1e3) / 1e9

    # ---- end to end through the public API with pinned host buffers
    xh = torch.from_numpy(x_host).pin_memory()
    yh = torch.empty_like(xh).pin_memory()

    def e2e_step():
        _lib.check(_lib.LIB.fl_dlt(cfg.handle, vp(xh.data_ptr()), vp(yh.data_ptr()), cols, n, sp))

    e2e_step()
    barrier()
    e_steps = max(1, min(args.steps, 5))
    e0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e_steps, dist, f"cuda:{local}")

    # parity spot check of this run's output against the oracle (not timed)
    parity = None
    if rank == 0 and cols:
        from oracle import ORACLE
        g = cfg.grid()
        j = cols - 1
        ref = ORACLE.dlt_grid(x_host[j], 1, cfg.tolerance(), g.theta, g.x, g.weights)
        parity = float(np.max(np.abs(yh[j].numpy() - ref)) / np.abs(x_host[j]).sum())
    subs = {}
    if not args.no_configs:
        subs = sub_configs(args, dist, rank, world, local)
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(args.config, n, args.cpu_seconds, os.cpu_count() or 1)
    if rank == 0:
        line = {
            "metric": "fp64 DLT coeffs/sec", "value": value, "unit": "coeffs/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(args.config, world, total),
            "method": {"dlt": ("direct: f = P c, one dense parity-split product per parity on the int8 "
                               "tcgen05 tensor cores (P_n(cos theta_k) in double-double at the reference's "
                               "angles; 7 8-bit digits/operand, exact int32 digit products, fp64 "
                               "recombination); idlt: c = D_s P^T D_w f likewise")
                       if direct else "factored: conversion + NDCT",
                       "factored_ablation": {"ndct": f"the chebstar nodes evaluated about cheb1 by the {L1}-term "
                                                     "Chebyshev (Jacobi-Anger) expansion, fused on chip",
                                             "conversion": "exact int8 digit-split triangular GEMM (tcgen05)"
                                             if gemm_mode == fl.GEMM_INT8_SPLIT else "fp64 DMMA"}},
            "roofline": {"bound": "tensor", "kernel": "oz_split_b_kernel + oz_gemm2_kernel (direct product)",
                         "achieved": dense_tops, "peak": INT8_PEAK_TOPS, "unit": "TOP/s int8",
                         "frac": dense_tops / INT8_PEAK_TOPS, "traffic": dense_traffic,
                         "timed": "the whole DLT step (digit split + GEMM) with CUDA events; "
                                  "the GEMM alone is the ncu share in profiles/",
                         "peak_source": "dense int8 tcgen05 peak measured by tools/tc_i8_peak.cu "
                                        "(profiles/r01_tc_i8_peak.log); MEASURED_PEAKS.json has no int8 entry",
                         "algorithmic": "28 digit pairs x 2 parities x (N/2)^2 MACs per column, 2 ops/MAC "
                                        f"(fp64-equivalent N flop/coef = {n * n * cols / (ms / 1e3) / 1e12:.1f} TFLOP/s)"}
            if direct else
                        {"bound": "fp64", "kernel": "fast_ndct_fwd_kernel",
                         "achieved": achieved, "peak": DFMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / DFMA_PEAK_TFLOPS, "traffic": traffic,
                         "peak_source": "measured DFMA (fp64 CUDA-core) peak, tools/fp64_peak.cu (profiles/r01_fp64_peak.log)",
                         "algorithmic": f"NDCT L(2.5 log2N + 3) flop/coef, L = {L1} transforms "
                                        "(Chebyshev expansion about cheb1, 2^-52)"},
            "roofline_fp64_factored_ndct": {"bound": "fp64", "kernel": "fast_ndct_fwd_kernel", "achieved": achieved,
                                            "peak": DFMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                                            "frac": achieved / DFMA_PEAK_TFLOPS, "traffic": traffic,
                                            "algorithmic": f"NDCT L(2.5 log2N + 3) flop/coef, L = {L1}"},
            "roofline_tensor": {"bound": "tensor", "kernel": "oz_split_b_kernel + oz_gemm2_kernel",
                                "gemm_mode": "int8_split" if gemm_mode == fl.GEMM_INT8_SPLIT else "fp64",
                                "achieved": i8_ops / (ms_l2c / 1e3) / 1e12, "peak": INT8_PEAK_TOPS,
                                "unit": "TOP/s int8", "frac": i8_ops / (ms_l2c / 1e3) / 1e12 / INT8_PEAK_TOPS,
                                "tile_cap": INT8_N64_CAP_TOPS,
                                "fp64_equivalent_tflops": l2c_flops / (ms_l2c / 1e3) / 1e12,
                                "peak_source": "tools/tc_i8_peak.cu (profiles/r01_tc_i8_peak.log)",
                                "algorithmic": "28 digit pairs (7 signed 8-bit digits per operand) x blocked triangle, 2 ops/MAC; fp64-equivalent N/2 flop/coef"},
            "roofline_hbm": {"bound": "hbm", "achieved": 16.0 * value / 1e9 / world, "peak": peak, "unit": "GB/s",
                             "frac": 16.0 * value / 1e9 / world / peak,
                             "note": "16 B/coef algorithmic (one fp64 read + one write), whole DLT, per GPU",
                             "dct_pass_gbs": dct_gbs, "dct_pass_frac": dct_gbs / peak,
                             "dct_pass_kernel": "fast_dct_stream_fwd_kernel (fl_trig DCT-III, same shard)",
                             "dct_pass_traffic": dct_traffic,
                             "dct_t_pass_gbs": dct_t_gbs, "dct_t_pass_frac": dct_t_gbs / peak},
            "kernels_ms": {"dlt_step": ms, "idlt_step": ms_idlt,
                           "factored_dlt_step": ms_dlt_f, "factored_idlt_step": ms_idlt_f,
                           "leg2cheb_split_int8": ms_l2c, "ndct": ms_ndct, "dct_iii_pass": ms_dct,
                           "dct_iii_t_pass": ms_dct_t,
                           "ndct_transpose": ms_ndct_t, "leg2cheb_transpose_split_int8": ms_l2c_t},
            "idlt": {"value": n * cols / (ms_idlt / 1e3) * world, "unit": "coeffs/s"},
            "e2e": {"value": n * total / (e2e_ms / 1e3), "unit": "coeffs/s",
                    "h2d_bytes_per_step": int(8 * n * cols), "d2h_bytes_per_step": int(8 * n * cols)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "parity_check": {"column": col0 + cols - 1, "rel_err_vs_oracle": parity,
                             "tolerance": 1e-13 * math.log2(n)},
        }
        if subs:
            line["configs"] = subs
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        dry_run(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == "c5":
        run_c5(args, rank, world, local)
    else:
        run_batched(args, rank, world, local)


if __name__ == "__main__":
    main()
