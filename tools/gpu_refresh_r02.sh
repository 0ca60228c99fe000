#!/bin/bash
# Round-2 evidence refresh (one gpurun call): GPU tests, smoke, the default bench,
# the reference arm, the caller stacks, the torchrun/NCCL path; logs under gpurun_out/r02/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r02/bench_default.json 2> gpurun_out/r02/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02/bench_reference.json 2>&1; echo "ref rc=$?"
for w in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --workload $w --steps 30 --warmup 5 > gpurun_out/r02/stack_$w.json 2>&1; echo "$w rc=$?"
done
timeout 300 python bench.py --workload cfg2 --per-table-scales --steps 30 --warmup 5 > gpurun_out/r02/stack_cfg2_mtile.json 2>&1
timeout 300 python bench.py --workload cfg2 --cmtile-tensor --steps 30 --warmup 5 > gpurun_out/r02/stack_cfg2_cmtile_tensor.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu --no-variants --gather-out --e2e-steps 1 \
  > gpurun_out/r02/bench_torchrun.json 2>&1; echo "torchrun rc=$?"
