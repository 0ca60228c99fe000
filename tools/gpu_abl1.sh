cd $GRAFT_REPO_ROOT
for dbg in 0 1 2 4 3 5 6 7; do
  echo "debug=$dbg" >> gpurun_out/abl1.log
  LUTGPU_OH_DEBUG=$dbg timeout 300 python bench.py --rows 262144 --steps 3 --warmup 1 --no-cpu --no-e2e --table i8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('gather_ms', d['roofline']['kernel_ms'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/abl1.log
done
