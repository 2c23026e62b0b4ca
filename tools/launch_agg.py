"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel
(development tool): total ms and launch count per kernel name."""
import collections, csv, sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].replace("(anonymous namespace)::", "")[:100]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-6)
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1]:10.3f} ms {v[0]:6d}  {v[1] / v[0] * 1e3:9.1f} us/launch  {k}")
print(f"total {tot:.3f} ms")
