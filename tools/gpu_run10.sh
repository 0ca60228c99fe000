cd $GRAFT_REPO_ROOT
rm -f gpurun_out/trace.log
for tbl in i8 f32; do
  echo "$tbl" >> gpurun_out/trace.log
  LUTGPU_OH_TRACE=1 timeout 300 python bench.py --rows 262144 --steps 1 --warmup 0 --no-cpu --no-e2e --table $tbl 2>&1 | grep -E 'trace|Error' | tail -1 >> gpurun_out/trace.log
done
