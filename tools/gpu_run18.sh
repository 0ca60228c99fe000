cd $GRAFT_REPO_ROOT
timeout 600 python tools/san_small.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/san_small.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu --rows 262144 > gpurun_out/torchrun1.log 2>&1; echo "torchrun rc=$?" >> gpurun_out/torchrun1.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.log 2>&1; echo "ref rc=$?" >> gpurun_out/ref_arm.log
