cd $GRAFT_REPO_ROOT
rm -f gpurun_out/abl.log
for tbl in i8; do for dbg in 0 1 2 4 5 6 7; do
  echo "table=$tbl debug=$dbg" >> gpurun_out/abl.log
  LUTGPU_OH_DEBUG=$dbg timeout 300 python bench.py --rows 262144 --steps 3 --warmup 1 --no-cpu --no-e2e --table $tbl 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('kernel_ms', d['roofline']['kernel_ms'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/abl.log
done; done
