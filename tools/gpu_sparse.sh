#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/b_sparse.json 2> gpurun_out/b_sparse.err
LUTGPU_OH_DENSE=1 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/b_dense.json 2> gpurun_out/b_dense.err
python - <<'PY'
import json
for f in ("b_sparse", "b_dense"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["ms_per_step"], 3), d["roofline"]["kernel_ms"], round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(f, "failed", e, open(f"gpurun_out/{f}.err").read()[-500:])
PY
