#!/bin/bash
# Caller-stack epilogue (FAST 6) check: its parity tests, the full GPU suite, and
# an A/B of the configs[1]/[3] stacks against the generic epilogue (LUTGPU_OH_EPI=0).
cd "$(dirname "$0")/.."
OUT=gpurun_out/stackepi
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k stack_epilogue > $OUT/pytest_new.log 2>&1; echo "new rc=$? $(tail -1 $OUT/pytest_new.log)"
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "gpu rc=$? $(tail -1 $OUT/pytest_gpu.log)"
for r in 1 2; do
  for w in cfg2 cfg4; do
    timeout 300 python bench.py --workload $w --steps 20 > $OUT/${w}_fast6_$r.json 2>/dev/null
    LUTGPU_OH_EPI=0 timeout 300 python bench.py --workload $w --steps 20 > $OUT/${w}_generic_$r.json 2>/dev/null
  done
done
for f in $OUT/*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" 2>&1)"; done
