#!/bin/bash
# Round evidence: GPU parity suite, smoke, default bench line, ncu launch list of
# the same command, one --set full capture (131072 rows, configs[4] geometry) of
# encode + gather, the configs[0..3] stacks and the f32 / K=64 variants.
cd "$(dirname "$0")/.."
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err || { echo bench failed; tail $OUT/bench_default.err; }
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 200 $CMD > $OUT/plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD2="python bench.py --rows 131072 --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 200 $CMD2 > $OUT/plain2.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onehot_pair|encode_tc" -s 2 -c 2 -o $OUT/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
timeout 300 python bench.py --workload cfg3 --table f32 --steps 20 > $OUT/stack_cfg3.json 2>/dev/null
timeout 300 python bench.py --workload cfg2 --steps 20 > $OUT/stack_cfg2.json 2>/dev/null
timeout 300 python bench.py --workload cfg1 --table f32 --steps 20 > $OUT/stack_cfg1.json 2>/dev/null
timeout 300 python bench.py --workload cfg4 --steps 10 > $OUT/stack_cfg4.json 2>/dev/null
timeout 300 python bench.py --table f32 --no-cpu --steps 5 > $OUT/bench_f32.json 2>/dev/null
timeout 300 python bench.py --k 64 --no-cpu --no-e2e --steps 5 > $OUT/bench_k64.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2>/dev/null
echo done
