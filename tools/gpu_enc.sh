#!/bin/bash
# Encode geometry A/B: parity (both RPL settings) + bench kernel times.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/enc
for rpl in 4 2; do
  LUTGPU_ENC_RPL=$rpl timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/enc/pytest_rpl$rpl.log 2>&1; echo "rpl=$rpl pytest rc=$? $(tail -1 gpurun_out/enc/pytest_rpl$rpl.log)"
  LUTGPU_ENC_RPL=$rpl timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/enc/b_rpl$rpl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/enc/b_rpl$rpl.json'));print('rpl=$rpl', d['roofline']['kernel_ms'], d['ms_per_step'], d['near_ties'])"
  LUTGPU_ENC_RPL=$rpl timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --k 64 > gpurun_out/enc/b64_rpl$rpl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/enc/b64_rpl$rpl.json'));print('K=64 rpl=$rpl', d['roofline']['kernel_ms'])"
done
