#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q -k "conv or resnet or lutn" 2>&1 | tail -3
python bench.py --workload cfg3 --table f32 --steps 20 > gpurun_out/st_cfg3.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_cfg3.csv python bench.py --workload cfg3 --table f32 --steps 1 --warmup 3 > gpurun_out/ncu_cfg3.log 2>&1
echo done
