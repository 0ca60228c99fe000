#!/bin/bash
# Round-2 final evidence (one gpurun call): the refresh (tests, smoke, default bench,
# reference arm, stacks, torchrun), then the ncu launch list of the default bench
# command, the --set full captures of the headline kernels and the conv encodes, and
# the stack launch lists.  Everything lands under gpurun_out/ (copy to profiles/r02/).
cd "$(dirname "$0")/.."
bash tools/gpu_refresh_r02.sh
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants --no-ties"
timeout 300 $CMD > gpurun_out/r02/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv $CMD > gpurun_out/r02/ncu_launch.log 2>&1
echo "launch list rc=$?"
bash tools/gpu_ncu_r02.sh
bash tools/gpu_ncu_conv.sh
bash tools/gpu_stack_launches.sh cfg1 cfg2 cfg3
