"""Benchmark: fp64 DLT coefficients/sec on B200 (BASELINE.json metric), with
the reference CPU path timed beside it.

Workload (BASELINE.json configs[3], "C4"): batched DLT, N = 4096, 65536
independent columns (2 GiB fp64 input), coefficients iid U[-1,1) from
std::mt19937_64(4000 + j), columns sharded evenly over the
ranks with no collective. One step = one DLT of this rank's shard through
the C ABI (fl_dlt) on device-resident input. `e2e` is the same call with
pinned HOST buffers (H2D + D2H inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4|c1|c3] [--cols C]

Multi-GPU: launched by torchrun, one rank per GPU (NCCL only for the barrier
and the max-over-ranks timing; the data path has no collective).
"""
from __future__ import annotations

import argparse
import json
import math
import os
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

CONFIGS = {
    # name: (N, total columns, generator, description)
    "c4": (4096, 65536, "uniform", "C4 batched DLT N=4096 x 65536 cols, U[-1,1)"),
    "c1": (1024, 1, "decay0.5", "C1 DLT N=1024, c_n = g_n/(n+1)^0.5"),
    "c3": (1 << 20, 1, "decay1", "C3 DLT N=2^20, c_n = g_n/(n+1)"),
    "c5": (1 << 26, 1, "c5", "C5 DLT N=2^26 (512 MiB), c_n = g_n e^{-n/N}, term-parallel over ranks"),
}


def run_c5(args, rank: int, world: int, local: int) -> None:
    """C5: one 2^26 DLT, its Taylor terms and Toeplitz-Hankel rank terms split
    over the ranks, partial sums combined by NCCL all-reduce / reduce-scatter
    (paper_1505_00354_b200/distributed.py). Fixed N: strong scaling."""
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
    c = fl.random_decaying(n, 0.0, 5) * np.exp(-np.arange(n) / n)
    x = torch.from_numpy(c).cuda()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        D.dlt(cfg, x, dist, scatter=True)
    barrier()
    l0 = fl.launch_count()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(s)
        for _ in range(args.steps):
            D.dlt(cfg, x, dist, scatter=True)
        e1.record(s)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, f"cuda:{local}")
    if rank == 0:
        print(json.dumps({
            "metric": "fp64 DLT coeffs/sec", "value": n / (ms / 1e3), "unit": "coeffs/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIGS["c5"][3], "N": n, "parallelism": f"term-parallel x{world}",
                       "leg2cheb_rank": [cfg.leg2cheb_rank(0), cfg.leg2cheb_rank(1)],
                       "l2": "512 MiB vectors > L2"},
            "gpu_launches": fl.launch_count() - l0, "clocks": clk.summary()}))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


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
    return ap.parse_args()


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
    import paper_1505_00354_b200 as fl
    gen = CONFIGS[cfg][2]
    if cols == 0:
        return np.empty((0, n))
    if gen == "uniform":
        return fl.random_uniform_pm1(n, 4000 + col0, batch=cols).reshape(cols, n)
    decay = 0.5 if gen == "decay0.5" else 1.0
    seed = 1 if cfg == "c1" else 3
    return fl.random_decaying(n, decay, seed + col0, batch=cols).reshape(cols, n)


def cpu_baseline(cfg: str, n: int, budget_s: float, threads: int) -> dict:
    """The reference's own CPU path (reference headers compiled in place,
    oracle/_ref) on a bounded sample of the workload, all host threads."""
    import ctypes as C
    from oracle import _ref
    if _ref is None:
        return {"value": None, "unit": "coeffs/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    vp, sz, i, d = C.c_void_p, C.c_size_t, C.c_int, C.c_double
    _ref.fr_config_create.argtypes = [sz, d, i, C.POINTER(vp)]
    _ref.fr_config_create.restype = i
    _ref.fr_batch.argtypes = [vp, i, sz, sz, vp, vp, i]
    _ref.fr_batch.restype = i
    _ref.fr_config_destroy.argtypes = [vp]
    h = vp()
    t0 = time.perf_counter()
    assert _ref.fr_config_create(n, 2.0 ** -52, 1, C.byref(h)) == 0
    t_cfg = time.perf_counter() - t0
    cols = max(threads, 1) if n <= 8192 else 1
    x = make_inputs(cfg, n, 0, cols)
    y = np.empty_like(x)
    done, elapsed = 0, 0.0
    while elapsed < budget_s:
        t0 = time.perf_counter()
        rc = _ref.fr_batch(h, 0, cols, n, vp(x.ctypes.data), vp(y.ctypes.data), threads)
        elapsed += time.perf_counter() - t0
        assert rc == 0
        done += cols
        if n > 8192:
            break
    _ref.fr_config_destroy(h)
    return {"value": done * n / elapsed, "unit": "coeffs/s", "cores": threads, "kind": "reference",
            "sample": f"{done} columns of N={n} ({elapsed:.1f} s, TransformConfig build {t_cfg:.2f} s "
                      f"excluded); reference headers + FFTW-API shim (FFTW absent)"}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    n, total, _, desc = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    vals = []
    for s in range(args.warmup + args.steps):
        b = cpu_baseline(args.config, n, max(args.cpu_seconds / max(args.steps, 1), 1.0), threads)
        if s >= args.warmup:
            vals.append(b["value"])
    v = float(np.median(vals))
    # a step of the full workload (all columns), at the sampled rate; each timed step
    # itself is a bounded sample (cpu_baseline.sample says how many columns)
    ms = n * total / v * 1e3
    line = {"metric": "fp64 DLT coeffs/sec", "value": v, "unit": "coeffs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_step_basis": "full workload at the sampled rate", "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": desc, "N": n, "columns": total, "parallelism": f"{threads} host threads"},
            "cpu_baseline": {**b, "value": v},
            "e2e": {"value": v, "unit": "coeffs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main() -> None:
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == "c5":
        run_c5(args, rank, world, local)
        return

    import torch
    import paper_1505_00354_b200 as fl
    from paper_1505_00354_b200 import _lib

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, total, _, desc = CONFIGS[args.config]
    if args.cols:
        total = args.cols
    from paper_1505_00354_b200.shard import column_shard, max_over_ranks
    col0, cols = column_shard(total, world, rank)
    per = (total + world - 1) // world
    stream = torch.cuda.current_stream()
    sp = __import__("ctypes").c_void_p(stream.cuda_stream)

    cfg = fl.TransformConfig(n)  # chebstar, tol 2^-52; plan built once, not timed
    x_host = make_inputs(args.config, n, col0, cols)
    x = torch.from_numpy(x_host).to(f"cuda:{local}")
    y = torch.empty_like(x)
    vp = __import__("ctypes").c_void_p

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
    chat = torch.empty_like(x)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    # the plan's conversion step exactly as fl_dlt runs it (split-int8 tcgen05 GEMM)
    ms_l2c = timed(lambda: _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 0, vp(x.data_ptr()),
                                                                vp(chat.data_ptr()), cols, n, sp)))
    # the plan's NDCT step exactly as fl_dlt runs it (fast mode: Chebyshev expansion)
    L1 = _lib.LIB.fl_plan_ndct_terms(cfg.handle)
    ms_ndct = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 0, vp(chat.data_ptr()),
                                                             vp(y.data_ptr()), cols, n, sp)))
    ms_dct = timed(lambda: _lib.check(_lib.LIB.fl_trig(0, fl.GridKind.cheb1, n, vp(x.data_ptr()),
                                                       vp(y.data_ptr()), cols, n, sp)))
    # the inverse on the same shard (DLT, IDLT and NDCT reported separately)
    # the IDLT's two steps (transpose = 1): NDCT^T, then the transposed conversion
    ms_ndct_t = timed(lambda: _lib.check(_lib.LIB.fl_plan_ndct(cfg.handle, 1, vp(x.data_ptr()),
                                                               vp(chat.data_ptr()), cols, n, sp)))
    ms_l2c_t = timed(lambda: _lib.check(_lib.LIB.fl_plan_leg2cheb(cfg.handle, 1, vp(chat.data_ptr()),
                                                                  vp(y.data_ptr()), cols, n, sp)))
    ms_idlt = timed(lambda: _lib.check(_lib.LIB.fl_idlt(cfg.handle, vp(x.data_ptr()), vp(y.data_ptr()),
                                                        cols, n, sp)))
    coef = n * cols
    l2c_flops = coef * (n / 2.0)                   # N^2/4 MACs per column = N/2 flop per coefficient
    ndct_flops = coef * L1 * (2.5 * math.log2(n) + 3)  # L (2.5 log2 N + 3)
    # int8 tensor work of the split product: 28 digit pairs x the 128-row-blocked
    # triangle (K from the diagonal block), 2 ops per MAC, both parities
    r_rows = n // 2
    rbs = r_rows // 128
    tri_macs = sum((r_rows - 128 * rb) * 128 for rb in range(rbs)) * 2 * cols
    i8_ops = 28 * 2 * tri_macs
    gemm_mode = cfg.gemm_mode()
    dom = "fast_ndct_fwd_kernel" if ms_ndct >= ms_l2c else "oz_gemm_kernel"
    achieved = ndct_flops / (ms_ndct / 1e3) / 1e12
    hbm_peak = json.load(open(MEASURED))["hbm_gbs"] if os.path.exists(MEASURED) else 6650.0
    # DRAM traffic of the NDCT kernel per launch, from the committed ncu
    # --set full capture (profiles/ncu_traffic.json: bytes per coefficient)
    traffic = dct_traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        for name, rec in tj.items():
            lg = int(math.log2(n))
            if name.startswith("fast_ndct_fwd_kernel") and (f"<{lg}>" in name or f"<{lg}, 1>" in name):
                traffic = {"bytes_per_launch": rec["dram_bytes_per_coef"] * coef,
                           "bytes_per_coef": rec["dram_bytes_per_coef"],
                           "algorithmic_bytes_per_coef": 16.0, "source": rec["capture"]}
                break
        rec = tj.get(f"fast_dct_stream_fwd_kernel<{int(math.log2(n))}>")
        if rec:
            dct_traffic = {"bytes_per_coef": rec["dram_bytes_per_coef"], "algorithmic_bytes_per_coef": 16.0,
                           "source": rec["capture"]}
    dct_gbs = 16.0 * coef / (ms_dct / 1e3) / 1e9

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
    if rank == 0:
        from oracle import ORACLE
        g = cfg.grid()
        j = cols - 1
        ref = ORACLE.dlt_grid(x_host[j], 1, cfg.tolerance(), g.theta, g.x, g.weights)
        parity = float(np.max(np.abs(yh[j].numpy() - ref)) / np.abs(x_host[j]).sum())
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(args.config, n, args.cpu_seconds, os.cpu_count() or 1)
    if rank == 0:
        line = {
            "metric": "fp64 DLT coeffs/sec", "value": value, "unit": "coeffs/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "N": n, "columns": total, "columns_per_rank": per,
                       "grid": "chebstar (default TransformConfig), NDCT evaluated about cheb1 (fast mode, "
                               "14-term Chebyshev expansion)",
                       "arithmetic": "fp64 throughout; the Legendre->Chebyshev product as an exact "
                                     "int8 digit-split GEMM on the tcgen05 tensor cores (7 8-bit digits/operand, "
                                     "int32 accumulation, fp64 recombination; fl_plan_set_gemm_mode "
                                     "selects the fp64 DMMA product instead)",
                       "parallelism": f"column shards x{world}, no collective",
                       "l2": "inputs (2 GiB) larger than L2 (126 MB); no flush"},
            "roofline": {"bound": "fp64", "kernel": "fast_ndct_fwd_kernel", "dominant": dom,
                         "achieved": achieved, "peak": DFMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / DFMA_PEAK_TFLOPS, "traffic": traffic,
                         "peak_source": "measured DFMA (fp64 CUDA-core) peak, tools/fp64_peak.cu (profiles/r01_fp64_peak.log)",
                         "algorithmic": f"NDCT L(2.5 log2N + 3) flop/coef, L = {L1} transforms "
                                        "(Chebyshev expansion about cheb1, 2^-52)"},
            "roofline_tensor": {"bound": "tensor", "kernel": "oz_split_b_kernel + oz_gemm2_kernel",
                                "gemm_mode": "int8_split" if gemm_mode == fl.GEMM_INT8_SPLIT else "fp64",
                                "achieved": i8_ops / (ms_l2c / 1e3) / 1e12, "peak": INT8_PEAK_TOPS,
                                "unit": "TOP/s int8", "frac": i8_ops / (ms_l2c / 1e3) / 1e12 / INT8_PEAK_TOPS,
                                "tile_cap": INT8_N64_CAP_TOPS,
                                "fp64_equivalent_tflops": l2c_flops / (ms_l2c / 1e3) / 1e12,
                                "peak_source": "tools/tc_i8_peak.cu (profiles/r01_tc_i8_peak.log)",
                                "algorithmic": "28 digit pairs (7 signed 8-bit digits per operand) x blocked triangle, 2 ops/MAC; fp64-equivalent N/2 flop/coef"},
            "roofline_hbm": {"bound": "hbm", "achieved": 16.0 * value / 1e9, "peak": hbm_peak, "unit": "GB/s",
                             "frac": 16.0 * value / 1e9 / hbm_peak,
                             "note": "16 B/coef algorithmic (one fp64 read + one write), whole DLT",
                             "dct_pass_gbs": dct_gbs, "dct_pass_frac": dct_gbs / hbm_peak,
                             "dct_pass_kernel": "fast_dct_stream_fwd_kernel (fl_trig DCT-III, same shard)",
                             "dct_pass_traffic": dct_traffic},
            "kernels_ms": {"leg2cheb_split_int8": ms_l2c, "ndct": ms_ndct, "dct_iii_pass": ms_dct,
                           "dlt_step": ms, "idlt_step": ms_idlt,
                           "ndct_transpose": ms_ndct_t, "leg2cheb_transpose_split_int8": ms_l2c_t},
            "e2e": {"value": n * total / (e2e_ms / 1e3), "unit": "coeffs/s",
                    "h2d_bytes_per_step": int(8 * n * cols), "d2h_bytes_per_step": int(8 * n * cols)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "parity_check": {"column": col0 + cols - 1, "rel_err_vs_oracle": parity,
                             "tolerance": 1e-13 * math.log2(n)},
        }
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
