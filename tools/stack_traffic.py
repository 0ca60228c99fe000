"""DRAM bytes per step of the caller stacks from ncu launch lists
(tools/gpu_stack_traffic.sh): the hot-path kernels (encode / gather / one-hot) of
every step the bench ran are summed and divided by the number of steps.

usage: python tools/stack_traffic.py <dir with traffic_cfgN.csv> > ncu_traffic_stacks.json
"""
import collections
import csv
import json
import os
import re
import sys

HOT = re.compile(r"^(void )?(lutgpu::)?(<unnamed>::)?(encode_\w+_kernel|gather_(f32|i8)_|onehot_(pair|stream|gemm)_kernel)")
LAYERS = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 60}  # LUT layers per step (2 launches each)

out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (cold cache, serialised), "
                 "bench.py --workload cfgN --steps 1 --warmup 1", "workloads": {}}
for tag, nl in LAYERS.items():
    path = os.path.join(sys.argv[1], f"traffic_{tag}.csv")
    if not os.path.exists(path):
        continue
    rows = open(path).read().splitlines()
    start = next(i for i, l in enumerate(rows) if l.startswith('"ID"'))
    by = collections.OrderedDict()
    for r in csv.DictReader(rows[start:]):
        name = r["Kernel Name"]
        if not HOT.search(name):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        d = by.setdefault(name.split("(")[0], {"launches": 0, "dram_bytes": 0.0, "us": 0.0})
        if r["Metric Name"].startswith("dram__bytes"):
            d["dram_bytes"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            if r["Metric Name"] == "dram__bytes_read.sum":
                d["launches"] += 1
        elif r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] += v * {"ns": 1e-3, "us": 1.0, "ms": 1e3}[u]
    launches = sum(d["launches"] for d in by.values())
    steps = launches / (2.0 * nl)
    out["workloads"][tag] = {
        "hot_launches": launches, "steps_profiled": steps,
        "dram_bytes_per_step": sum(d["dram_bytes"] for d in by.values()) / steps if steps else None,
        "kernels": {k: {"launches_per_step": d["launches"] / steps, "dram_bytes_per_launch": d["dram_bytes"] / d["launches"],
                        "us_per_launch_cold": d["us"] / d["launches"]} for k, d in by.items()}}
print(json.dumps(out, indent=1))
