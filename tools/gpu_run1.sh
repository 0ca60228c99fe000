cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_f32.log 2>&1; echo "rc=$?" >> gpurun_out/bench_f32.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --table i8 --no-e2e > gpurun_out/bench_i8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_i8.log
