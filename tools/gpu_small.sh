#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/small
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/small/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/small/pytest.log)"
for env in "X=0" "LUTGPU_GATHER_MINROWS=0"; do
  for w in "cfg1 --table f32" "cfg3 --table f32" "cfg2" "cfg4"; do
    env $env timeout 120 python bench.py --workload $w --steps 10 --warmup 2 > gpurun_out/small/s.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/small/s.json'));print('$env | $w', round(d['ms_per_step'],4))" || echo "fail $env $w"
  done
done
