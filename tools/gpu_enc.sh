#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/enc
for g in 2 3 4; do
  LUTGPU_ENC_TC_GROUPS=$g timeout 300 python -m pytest tests -m gpu -x -q -k "encode or ties or crit1 or cfg or large or screen" > gpurun_out/enc/pytest.log 2>&1; echo "groups=$g pytest rc=$? $(tail -1 gpurun_out/enc/pytest.log)"
  LUTGPU_ENC_TC_GROUPS=$g timeout 120 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/enc/b.json 2>gpurun_out/enc/b.err
  python -c "import json;d=json.load(open('gpurun_out/enc/b.json'));print('groups=$g', d['roofline']['kernel_ms'], d['near_ties'])" || tail -3 gpurun_out/enc/b.err
done


