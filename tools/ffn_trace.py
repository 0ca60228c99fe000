"""configs[1] FFN pair gathers with the pair-kernel role counters (needs the probe
build, tools/build_probes.sh): prints cycles per unit for each role, per layer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2302_03213_b200 import workloads as W

ffn, x = W.ffn_pair("cuda")
with torch.no_grad():
    for _ in range(3):
        ffn(x)
    torch.cuda.synchronize()
    os.environ["LUTGPU_OH_TRACE"] = "1"
    for _ in range(2):
        ffn(x)
        torch.cuda.synchronize()
