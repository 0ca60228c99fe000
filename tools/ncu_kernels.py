"""One launch of each secondary kernel at a BASELINE shape, for an ncu --set full
capture (tools/gpu_ncu_kernels.sh): the CUDA-core gathers at configs[4] geometry,
the TMA FFMA2 encode (configs[0]), the hash encoder, the caller-stack pair
epilogue (configs[1] FFN1: bias + GELU + per-m-tile scales) and the conv-plane
encode (configs[2] stage 1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03213_b200 as L  # noqa: E402
from paper_2302_03213_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
# CUDA-core gathers, configs[4] geometry (65536 rows)
for integer in (False, True):
    layer, a = W.linear(dev, 65536, 4096, 4096, 32, 16, integer, gather="cuda")
    layer.forward_device(a, integer)
# configs[0]: encode_tma (V = 16) + f32 gather
layer, a = W.linear(dev, 1024, 768, 768, 16, 16, False)
layer.forward_device(a, False)
# hash encoder (depth 4 trees) on configs[0] rows
rng = np.random.default_rng(3)
trees = [(rng.integers(0, 16, 4), rng.standard_normal(15).astype(np.float32), rng.integers(0, 16, 16).astype(np.uint8))
         for _ in range(48)]
L.encode_hash(a, trees)
# configs[1] FFN1: pair kernel with the caller-stack epilogue (bias, GELU, m-tile scales)
ffn, x = W.ffn_pair(dev, tokens=4096, scale_mtile=128)
ffn(x)
# configs[2] stage 1 conv
convs = W.resnet_convs(dev, batch=256)
convs[0][0](convs[0][1])
torch.cuda.synchronize()
print("ok")
