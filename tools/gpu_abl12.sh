#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/abl12.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/abl12.json'));print('default', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))"
LUTGPU_OH_TRACE=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
