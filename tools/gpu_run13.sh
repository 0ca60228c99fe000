cd $GRAFT_REPO_ROOT
rm -f gpurun_out/dimtest.log
for cfg in "262144 4096" "1048576 1024" "4194304 256"; do set -- $cfg
  echo "rows=$1 dim=$2" >> gpurun_out/dimtest.log
  timeout 300 python bench.py --rows $1 --dim $2 --steps 3 --warmup 1 --no-cpu --no-e2e --table i8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; n=d['config']['rows_per_gpu']; dd=d['config']['d']
        print('encode_ms %.3f  GB/s %.0f' % (r['kernel_ms']['encode'], 4*n*dd/r['kernel_ms']['encode']/1e6))" >> gpurun_out/dimtest.log
done
