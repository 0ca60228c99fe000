"""configs[0] layer (1024 x 768 -> 768, f32) once, for an ncu capture of its two kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_03213_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda", 0)
layer, a = W.linear(dev, 1024, 768, 768, 16, 16, False)
for _ in range(3):
    layer.forward_device(a, False)
torch.cuda.synchronize()
print("ok")
