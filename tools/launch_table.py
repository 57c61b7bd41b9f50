"""Per-kernel mean/total of an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv).

  python tools/launch_table.py gpurun_out/launches.csv
"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
lines = [l for l in text.splitlines() if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"][:90]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    us = v / 1000.0 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1000.0
    agg.setdefault(name, []).append(us)
tot = sum(sum(v) for v in agg.values())
print(f"{'count':>6} {'mean us':>9} {'total us':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):6d} {sum(v) / len(v):9.2f} {sum(v):10.1f} {100 * sum(v) / tot:5.1f}%  {k}")
