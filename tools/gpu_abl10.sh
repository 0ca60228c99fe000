#!/bin/bash
cd "$(dirname "$0")/.."
LUTGPU_OH_KB=4 timeout 600 python -m pytest tests -m gpu -x -q -k "tc or onehot or tensor or ffn or lutn" 2>&1 | tail -2
for cfg in "LUTGPU_OH_KB=2" "LUTGPU_OH_KB=4" "LUTGPU_OH_KB=4 LUTGPU_OH_DEBUG=7"; do
  env $cfg timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl10.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl10.json'));print('$cfg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))" 2>/dev/null || echo "$cfg failed"
done
