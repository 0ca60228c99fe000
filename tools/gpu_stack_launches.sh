#!/bin/bash
# Launch lists (ncu gpu__time_duration, cold, serialised) for the configs 1-4 stacks.
cd "$(dirname "$0")/.."
for w in cfg1 cfg2 cfg3; do
  python bench.py --workload $w --table f32 --steps 2 --warmup 3 > gpurun_out/st_$w.json 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$w.csv \
      python bench.py --workload $w --table f32 --steps 1 --warmup 3 > gpurun_out/ncu_$w.log 2>&1
done
