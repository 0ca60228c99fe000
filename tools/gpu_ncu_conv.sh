#!/bin/bash
# ncu --set full of the configs[2] conv encodes (tools/conv_bench.py), after a plain run.
cd "$(dirname "$0")/.."
python tools/conv_bench.py > gpurun_out/conv_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"encode_conv" -c 24 \
    -o gpurun_out/prof_conv python tools/conv_bench.py > gpurun_out/ncu_conv.log 2>&1
echo "ncu rc=$?"
