"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    us = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | total ms | mean ms/launch | share |\n|---|---:|---:|---:|---:|")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {us / 1e3:.3f} | {us / 1e3 / n:.4f} | {100 * us / tot:.1f} % |")
