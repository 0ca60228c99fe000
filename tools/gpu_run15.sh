cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "tc_ or cfg1 or crit1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/abl.log
for tbl in i8 f32; do for cfg in "0 0" "1 0" "0 1" "1 1"; do set -- $cfg
  echo "table=$tbl spin=$1 acc1=$2" >> gpurun_out/abl.log
  LUTGPU_OH_SPIN=$1 LUTGPU_OH_ACC1=$2 timeout 300 python bench.py --rows 262144 --steps 3 --warmup 1 --no-cpu --no-e2e --table $tbl 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('kernel_ms', d['roofline']['kernel_ms'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/abl.log
done; done
