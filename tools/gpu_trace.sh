#!/bin/bash
cd "$(dirname "$0")/.."
for dbg in 0 7 1; do
  echo "debug $dbg"; LUTGPU_OH_DEBUG=$dbg LUTGPU_OH_TRACE=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 >/dev/null | grep trace | tail -1
done
