#!/bin/bash
# A/B two in-tree builds on the same box (alternating runs): _lib/liblutgpu_a.so vs _lib/liblutgpu_b.so
# usage: tools/ab_lib.sh [extra bench.py args]
cd "$(dirname "$0")/.."
for i in 1 2 3 4; do
  for v in a b; do
    LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_$v.so timeout 120 python bench.py --no-cpu --no-e2e --no-variants --no-ties --steps 10 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v', round(d['roofline']['kernel_ms']['encode'],3), round(d['roofline']['kernel_ms']['gather'],3))"
  done
done
