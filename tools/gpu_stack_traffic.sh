#!/bin/bash
# DRAM bytes per launch (ncu, cold-cache, serialised) of the configs[0..3] caller stacks,
# summarised into gpurun_out/stack/ncu_traffic_stacks.json (copy to profiles/rNN/).
# usage: tools/gpu_stack_traffic.sh [cfg...]   (default: all four)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/stack
for tag in ${@:-cfg1 cfg2 cfg3 cfg4}; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:"^(encode_|gather_f32|gather_i8|onehot_)" \
      --log-file gpurun_out/stack/traffic_$tag.csv \
      python bench.py --workload $tag --steps 1 --warmup 1 --no-cpu > gpurun_out/stack/ncu_traffic_$tag.log 2>&1
  echo "$tag rc=$?"
done
python tools/stack_traffic.py gpurun_out/stack > gpurun_out/stack/ncu_traffic_stacks.json
cat gpurun_out/stack/ncu_traffic_stacks.json
