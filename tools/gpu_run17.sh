cd $GRAFT_REPO_ROOT
rm -f gpurun_out/trace.log
for dbg in 0 7; do
  echo "i8 debug=$dbg" >> gpurun_out/trace.log
  LUTGPU_OH_DEBUG=$dbg LUTGPU_OH_TRACE=1 timeout 300 python bench.py --rows 262144 --steps 1 --warmup 0 --no-cpu --no-e2e --table i8 2>&1 | grep -E 'trace|Error' | tail -1 >> gpurun_out/trace.log
done
