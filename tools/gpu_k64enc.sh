#!/bin/bash
# configs[4] K=64 encode: HEAD build (a) vs new (b) vs probe build with 2/3/4 consumer groups
cd "$(dirname "$0")/.."
run() { timeout 120 python bench.py --k 64 --no-cpu --no-e2e --no-variants --no-ties --steps 6 --warmup 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$1', round(d['roofline']['kernel_ms']['encode'],3), round(d['roofline']['kernel_ms']['gather'],3))"; }
for i in 1 2; do
  LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_a.so run a
  LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_b.so run b
  for g in 2 3 4; do LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_probe.so LUTGPU_ENC_TC_GROUPS=$g run probe_g$g; done
done
