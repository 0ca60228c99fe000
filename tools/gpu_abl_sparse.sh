#!/bin/bash
cd "$(dirname "$0")/.."
for dbg in 0 1 2 4 8 3 5 6 7; do
  LUTGPU_OH_DEBUG=$dbg timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl_$dbg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl_$dbg.json'));print('debug $dbg gather_ms', round(d['roofline']['kernel_ms']['gather'],3))"
done
LUTGPU_OH_TRACE=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -2
