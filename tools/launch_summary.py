"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
if mi is not None:
    data = [r for r in data if r[mi] == "gpu__time_duration.sum"]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data[skip:]:
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':42s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:42s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:8.2f} {v[1] / tot:6.3f}")
print(f"total_us {tot:.1f} launches {sum(v[0] for v in agg.values())}")
