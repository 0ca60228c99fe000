cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/p6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_i8.csv $CMD > gpurun_out/p6_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/p6_ncu_launch.log
CMD2="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/p6_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"onehot_pair|encode_tma" -s 2 -c 2 -o gpurun_out/prof_r01_full $CMD2 > gpurun_out/p6_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/p6_ncu_full.log
