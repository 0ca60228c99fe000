cd $GRAFT_REPO_ROOT
CMD2="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/ps_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"onehot_pair" -s 1 -c 1 -o gpurun_out/prof_sparse $CMD2 > gpurun_out/ps_ncu.log 2>&1
echo "full rc=$?"
