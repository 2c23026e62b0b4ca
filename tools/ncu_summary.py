"""Summarise ncu evidence for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches gpurun_out/launches.csv   # per-kernel share of a launch list
  python tools/ncu_summary.py full gpurun_out/hot_full.ncu-rep    # key metrics of a --set full capture
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
]


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list {path}: gpu__time_duration.sum, cold-cache serialised (compare shares)")
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.1f}%")


def full(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full {path}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"\n## {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:82s} {d[k]:>16s} {units[h.index(k)]}")
        stalls = [(float(d[k].replace(',', '')), k) for k in h
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d.get(k, "").replace(",", "").replace(".", "").isdigit()]
        tot = sum(x for x, _ in stalls) or 1.0
        print("  top stall reasons (pc sampling):")
        for x, k in sorted(stalls, reverse=True)[:6]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f}%")


def traffic_json(path: str, coefs: int, out: str) -> None:
    """DRAM bytes per transformed coefficient of each kernel in a capture
    (read by bench.py for the roofline `traffic` field)."""
    import json
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("unnamed>::", "")
        b = sum(float(d[k].replace(",", "")) * scale[units[h.index(k)]]
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res[name] = {"dram_bytes_per_coef": b / coefs, "capture": path, "coefs_per_launch": coefs}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic_json(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
