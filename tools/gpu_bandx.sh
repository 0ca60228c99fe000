#!/bin/bash
# Headline gather vs the pair kernel's band width (probe build, LUTGPU_OH_BANDX),
# alternating settings on one box.
cd "$(dirname "$0")/.."
for i in 1 2; do
  for bx in ${BXS:-1 2 4 8 16}; do
    LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_probe.so LUTGPU_OH_BANDX=$bx timeout 120 python bench.py --no-cpu --no-e2e --no-variants --no-ties --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('bandx=$bx', round(d['roofline']['kernel_ms']['gather'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
