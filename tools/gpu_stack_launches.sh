#!/bin/bash
# Launch lists (ncu gpu__time_duration, cold, serialised) for the configs[0..3] stacks.
# usage: tools/gpu_stack_launches.sh [cfg...]   (default: all four)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/stack
for tag in ${@:-cfg1 cfg2 cfg3 cfg4}; do
  extra=""; [ $tag = cfg1 ] || [ $tag = cfg3 ] && extra="--table f32"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stack/launch_$tag.csv \
      python bench.py --workload $tag $extra --steps 1 --warmup 1 > gpurun_out/stack/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
