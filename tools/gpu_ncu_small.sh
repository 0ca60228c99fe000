#!/bin/bash
# ncu --set full of the small-config hot kernels: configs[0] f32 gather + encode,
# configs[1] FFN1 gather (FAST 6) and FFN2 gather (FAST 4).
cd "$(dirname "$0")/.."
OUT=gpurun_out/small
mkdir -p $OUT
timeout 120 python bench.py --workload cfg1 --table f32 --steps 2 --warmup 1 > $OUT/cfg1.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gather_f32_tiled|encode_tma" -s 2 -c 2 -o $OUT/cfg1 \
    python bench.py --workload cfg1 --table f32 --steps 1 --warmup 1 > $OUT/ncu_cfg1.log 2>&1
echo "cfg1 rc=$?"
timeout 120 python bench.py --workload cfg2 --steps 2 --warmup 1 > $OUT/cfg2.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"onehot_pair" -s 2 -c 2 -o $OUT/cfg2 \
    python bench.py --workload cfg2 --steps 1 --warmup 1 > $OUT/ncu_cfg2.log 2>&1
echo "cfg2 rc=$?"
