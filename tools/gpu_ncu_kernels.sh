#!/bin/bash
# ncu --set full of the secondary kernels (tools/ncu_kernels.py), after a plain run.
cd "$(dirname "$0")/.."
python tools/ncu_kernels.py > gpurun_out/ncuk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"gather_f32_rows|gather_i8_rows|encode_tma|encode_hash|onehot_pair_kernel|encode_conv" \
    -o gpurun_out/prof_kernels python tools/ncu_kernels.py > gpurun_out/ncuk.log 2>&1
echo "ncu rc=$?"
