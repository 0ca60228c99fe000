#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/abl
run() {
  env "$@" timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 2 > gpurun_out/abl/b.json 2>gpurun_out/abl/b.err
  python -c "import json;d=json.load(open('gpurun_out/abl/b.json'));print('$*', 'gather_ms', round(d['roofline']['kernel_ms']['gather'],3))" 2>/dev/null || { echo "$* failed"; tail -2 gpurun_out/abl/b.err; }
}
run X=0
run LUTGPU_OH_DEBUG=64
run LUTGPU_OH_DEBUG=128
run LUTGPU_OH_DEBUG=192
run LUTGPU_OH_DEBUG=2
run LUTGPU_OH_DEBUG=6
run LUTGPU_OH_DEBUG=70
run LUTGPU_OH_DEBUG=134
