#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/enc
for cfg in "LUTGPU_ENC_CHAIN=2" "LUTGPU_ENC_CHAIN=1" "LUTGPU_ENC_CHAIN=2 LUTGPU_ENC_GEOM=4" "LUTGPU_ENC_CHAIN=2 LUTGPU_ENC_GEOM=12"; do
  env $cfg timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/enc/pytest.log 2>&1; echo "$cfg pytest rc=$? $(tail -1 gpurun_out/enc/pytest.log)"
  env $cfg timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/enc/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/enc/b.json'));print('$cfg', d['roofline']['kernel_ms'], d['near_ties'])"
  env $cfg timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --k 64 > gpurun_out/enc/b64.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/enc/b64.json'));print('K=64 $cfg', d['roofline']['kernel_ms'])"
done
