"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per kernel:
launches, summed device time, share, mean).

    python tools/launchlist_summary.py gpurun_out/launches.csv "header line" > profiles/X.txt
"""
import collections
import csv
import sys

path = sys.argv[1]
head = sys.argv[2] if len(sys.argv) > 2 else ""
rows = []
with open(path) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    us = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "second": 1e6, "s": 1e6}[unit]
    rows.append((r["Kernel Name"], us))
agg = collections.defaultdict(lambda: [0, 0.0])
for k, us in rows:
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(v[1] for v in agg.values())
print(f"# {head}")
print("# cold-cache, serialised launches under ncu: compare shares, not absolutes")
print(f"launches {len(rows)} summed device time ms {tot / 1e3:.3f}")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    name = k if len(k) < 60 else k[:57] + "..."
    print(f"{name:60s} n={c:6d} {us / 1e3:9.3f} ms {100 * us / tot:5.1f}%  mean {us / c:9.2f} us")
