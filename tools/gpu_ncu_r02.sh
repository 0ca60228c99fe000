#!/bin/bash
# ncu --set full of the headline kernels (configs[4] geometry, 131072 rows): the
# plain run first (must exit 0), then one capture of encode + gather.
cd "$(dirname "$0")/.."
CMD="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants --no-ties"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"onehot_pair|encode_tc" -s 2 -c 2 \
    -o gpurun_out/prof_r02 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
