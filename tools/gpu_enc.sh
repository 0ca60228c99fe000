#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/enc
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/enc/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/enc/pytest.log)"; grep -m5 "Error\|assert\|FAIL" gpurun_out/enc/pytest.log
for g in 2 3; do
  for k in 16 64; do
    LUTGPU_ENC_TC_GROUPS=$g timeout 120 python bench.py --no-cpu --no-e2e --steps 3 --k $k > gpurun_out/enc/b.json 2>gpurun_out/enc/b.err
    python -c "import json;d=json.load(open('gpurun_out/enc/b.json'));print('groups=$g k=$k', d['roofline']['kernel_ms'], d['near_ties'])" || tail -3 gpurun_out/enc/b.err
  done
done
