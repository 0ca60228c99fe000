cd $GRAFT_REPO_ROOT
CMD="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e --table i8"
$CMD > gpurun_out/prof4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:onehot_pair -s 1 -c 1 -o gpurun_out/prof_pair_i8_v2 $CMD > gpurun_out/prof4_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof4_ncu.log
