#!/bin/bash
# A/B two builds (_lib/liblutgpu_a.so vs _b.so) on the caller stacks, alternating, one box.
# usage: tools/ab_stack.sh cfg1 [cfg3 ...]
cd "$(dirname "$0")/.."
for w in "$@"; do
  for i in 1 2 3; do
    for v in a b; do
      LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_$v.so timeout 300 python bench.py --workload $w --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w $v', round(d['ms_per_step']*1e3,2), 'us/step')"
    done
  done
done
