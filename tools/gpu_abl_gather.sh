#!/bin/bash
# Gather (pair kernel) ablations at configs[4]: kernel ms per env setting + role trace.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/abl
run() {
  env "$@" timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 2 > gpurun_out/abl/b.json 2>gpurun_out/abl/b.err
  python -c "import json;d=json.load(open('gpurun_out/abl/b.json'));print('$*', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))" 2>/dev/null || { echo "$* failed"; tail -2 gpurun_out/abl/b.err; }
}
run X=0
run LUTGPU_OH_DEBUG=1
run LUTGPU_OH_DEBUG=2
run LUTGPU_OH_DEBUG=4
run LUTGPU_OH_DEBUG=8
run LUTGPU_OH_DEBUG=32
run LUTGPU_OH_DEBUG=3
run LUTGPU_OH_DEBUG=7
run LUTGPU_OH_DEBUG=6
run LUTGPU_OH_DEBUG=5
run LUTGPU_OH_TMAOUT=0
run LUTGPU_OH_KB=2
run LUTGPU_OH_SPIN=0
run LUTGPU_OH_SPIN=1
LUTGPU_OH_TRACE=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
