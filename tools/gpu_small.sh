#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/small
for s in 0 8192 65536; do
  for w in "cfg1 --table f32" "cfg2" "cfg4"; do
    LUTGPU_ENC_SMALL_ROWS=$s timeout 120 python bench.py --workload $w --steps 10 --warmup 2 > gpurun_out/small/s.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/small/s.json'));print('small=$s $w', round(d['ms_per_step'],4))" || echo "fail $s $w"
  done
done
