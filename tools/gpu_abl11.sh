#!/bin/bash
cd "$(dirname "$0")/.."
for dbg in 0 1 2 4 3 6; do
  LUTGPU_OH_KB=4 LUTGPU_OH_DEBUG=$dbg timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl11.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl11.json'));print('KB4 debug $dbg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))" 2>/dev/null || echo "$dbg failed"
done
LUTGPU_OH_KB=4 LUTGPU_OH_TRACE=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
LUTGPU_OH_KB=4 LUTGPU_OH_ACC1=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl11.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/abl11.json'));print('KB4 acc1', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))"
