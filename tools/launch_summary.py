"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum --csv launch list.

usage: python tools/launch_summary.py <launches.csv> [title] > profiles/rNN/<name>.txt
"""
import collections
import csv
import sys

rows = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(rows) if l.startswith('"ID"'))
times = collections.OrderedDict()
for r in csv.DictReader(rows[start:]):
    if r.get("Metric Name") != "gpu__time_duration.sum" or "lutgpu" not in r["Kernel Name"]:
        continue
    v = float(r["Metric Value"].replace(",", ""))
    v = v / 1000.0 if r["Metric Unit"] == "ns" else (v * 1000.0 if r["Metric Unit"] == "ms" else v)
    times.setdefault(r["Kernel Name"].split("(")[0], []).append(v)
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
for k, v in times.items():
    print(f"{k[:72]:<72} n={len(v):4d} mean={sum(v) / len(v):9.2f} us min={min(v):9.2f} us total={sum(v):10.1f} us")
