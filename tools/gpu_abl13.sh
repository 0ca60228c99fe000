#!/bin/bash
cd "$(dirname "$0")/.."
LUTGPU_OH_TMAOUT=0 timeout 600 python -m pytest tests -m gpu -x -q -k "tc or onehot or tensor or ffn or lutn" 2>&1 | tail -2
for cfg in "LUTGPU_OH_TMAOUT=1" "LUTGPU_OH_TMAOUT=0"; do
  env $cfg timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl13.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl13.json'));print('$cfg', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))" 2>/dev/null || echo "$cfg failed"
done
LUTGPU_OH_TMAOUT=0 LUTGPU_OH_TRACE=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
