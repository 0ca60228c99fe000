cd $GRAFT_REPO_ROOT
rm -f gpurun_out/enc.log
for cfg in "0 3" "1 3" "0 2" "1 2"; do set -- $cfg
  echo "debug=$1 stages=$2" >> gpurun_out/enc.log
  LUTGPU_ENC_DEBUG=$1 LUTGPU_ENC_STAGES=$2 timeout 300 python bench.py --rows 262144 --steps 3 --warmup 1 --no-cpu --no-e2e --table i8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; n=d['config']['rows_per_gpu']; dd=d['config']['d']
        print('encode_ms %.3f  GB/s %.0f' % (r['kernel_ms']['encode'], 4*n*dd/r['kernel_ms']['encode']/1e6))" >> gpurun_out/enc.log
done
