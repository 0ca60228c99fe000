#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "LUTGPU_OH_DEBUG=7" "LUTGPU_OH_DEBUG=23" "LUTGPU_OH_DEBUG=16" "LUTGPU_OH_DEBUG=17"; do
  env $cfg timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl4.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl4.json'));print('$cfg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))"
done
LUTGPU_OH_DEBUG=23 LUTGPU_OH_TRACE=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
