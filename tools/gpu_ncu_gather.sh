#!/bin/bash
# One --set full capture (source-correlated) of the pair gather + encode at 131072 rows.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
CMD="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/ncu/plain.json 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onehot_pair|encode_tma" -s 2 -c 2 -o gpurun_out/ncu/full $CMD > gpurun_out/ncu/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu/ncu.log
