"""Per-instruction shared-memory excess and stall samples from an ncu report
(development tool): python tools/sass_hot.py report.ncu-rep [top]"""
import csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: h.index(k) for k in ["Address", "Source", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared",
                              "Warp Stall Sampling (All Samples)"]}
data = rows[2:]
f = lambda r, k: float(r[ix[k]] or 0)
print("shared wavefronts", sum(f(r, "L1 Wavefronts Shared") for r in data),
      "excessive", sum(f(r, "L1 Wavefronts Shared Excessive") for r in data),
      "samples", sum(f(r, "Warp Stall Sampling (All Samples)") for r in data))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
print("-- top excessive")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:top]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(r[ix["Address"]][-5:], r[ix["Source"]][:60].strip(), int(f(r, "L1 Wavefronts Shared")),
              int(f(r, "L1 Wavefronts Shared Excessive")))
print("-- top stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    print(r[ix["Address"]][-5:], r[ix["Source"]][:60].strip(), int(f(r, "Warp Stall Sampling (All Samples)")))
