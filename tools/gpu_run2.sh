cd $GRAFT_REPO_ROOT
timeout 180 python tools/tc_sanity.py > gpurun_out/tc_sanity.log 2>&1; echo "rc=$?" >> gpurun_out/tc_sanity.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --table i8 > gpurun_out/bench_i8_tc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_i8_tc.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --table f32 > gpurun_out/bench_f32_tc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_f32_tc.log
