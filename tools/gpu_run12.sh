cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_i8_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_i8_full.log
timeout 900 python bench.py --steps 5 --warmup 3 --table f32 --no-cpu --no-e2e > gpurun_out/bench_f32_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_f32_full.log
CMD="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e --table i8"
$CMD > gpurun_out/prof5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:encode_tma -s 1 -c 1 -o gpurun_out/prof_encode $CMD > gpurun_out/prof5_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof5_ncu.log
