#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/rlx
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_ or onehot or tensor or large" > gpurun_out/rlx/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/rlx/pytest.log)"
run() {
  env "$@" timeout 120 python bench.py --no-cpu --no-e2e --steps 5 --warmup 2 > gpurun_out/rlx/b.json 2>gpurun_out/rlx/b.err
  python -c "import json;d=json.load(open('gpurun_out/rlx/b.json'));print('$*', d['roofline']['kernel_ms'])" 2>/dev/null || { echo "$* failed"; tail -2 gpurun_out/rlx/b.err; }
}
run X=0
run X=1
run LUTGPU_OH_DEBUG=5
