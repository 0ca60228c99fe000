#!/bin/bash
# Launch lists (ncu gpu__time_duration, cold, serialised) for the configs[0..3] stacks.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/stack
for w in "cfg1 --table f32" "cfg2" "cfg3 --table f32" "cfg4"; do
  tag=$(echo $w | cut -d' ' -f1)
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stack/launch_$tag.csv \
      python bench.py --workload $w --steps 1 --warmup 1 > gpurun_out/stack/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
