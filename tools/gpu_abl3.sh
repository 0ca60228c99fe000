#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "LUTGPU_OH_SPIN=0" "LUTGPU_OH_SPIN=2" "LUTGPU_OH_SPIN=2 LUTGPU_OH_DEBUG=7" "LUTGPU_OH_SPIN=0 LUTGPU_OH_DEBUG=7"; do
  env $cfg timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl3.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl3.json'));print('$cfg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))"
done
