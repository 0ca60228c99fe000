#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "LUTGPU_OH_DEBUG=0" "LUTGPU_OH_DEBUG=7" "LUTGPU_OH_DEBUG=199" "LUTGPU_OH_DEBUG=0"; do
  env $cfg timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl7.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl7.json'));print('$cfg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3), 'enc', round(d['roofline']['kernel_ms']['encode'],3), d['clocks'])" 2>/dev/null || echo "$cfg failed"
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
