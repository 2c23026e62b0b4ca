"""Pinned host <-> device copy rates on this box (development tool): H2D alone,
D2H alone, both at once on two streams, and the e2e DLT pipeline's
per-chunk overlap, to bound bench.py's e2e number.

  python tools/pcie_probe.py [GiB]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def rate(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    n = int(gib * (1 << 30)) // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_in = torch.empty(n, dtype=torch.float64, device="cuda")
    d_out = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = n * 8
    print(f"h2d alone: {rate(lambda: d_in.copy_(h_in, non_blocking=True), nb):.1f} GB/s")
    print(f"d2h alone: {rate(lambda: h_out.copy_(d_out, non_blocking=True), nb):.1f} GB/s")

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    print(f"h2d + d2h concurrently: {rate(both, 2 * nb):.1f} GB/s total")


if __name__ == "__main__":
    main()
