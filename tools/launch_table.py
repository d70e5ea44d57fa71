"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_table.py launches.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg[name].append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for k, v in agg.items() if "leo::" in k)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:top]:
    share = 100 * sum(v) / tot if "leo::" in k else 0.0
    print(f"{k:44s} n={len(v):3d} total={sum(v) / 1e3:8.1f}us mean={sum(v) / len(v) / 1e3:7.1f}us "
          f"max={max(v) / 1e3:7.1f}us share={share:5.1f}%")
