"""Small shapes through every kernel, for compute-sanitizer memcheck."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_03213_b200 as L
from oracle import lut_oracle as O

rng = O.make_rng(3)
for (n, c, k, v, m) in [(600, 8, 16, 32, 40), (300, 12, 8, 4, 33), (70, 5, 16, 9, 7), (513, 16, 64, 16, 130)]:
    a, books, b = O.random_instance(rng, n, c, k, v, m)
    for gather in ("cuda", "tensor"):
        layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=b, bias=np.ones(m, np.float32), qat=True,
                           gather=gather)
        y8 = L.lut_layer_infer(a, layer, integer=True)
        yf = L.lut_layer_infer(a, layer, integer=False)
x = np.abs(rng.standard_normal((2, 8, 6, 6))).astype(np.float32)
bk = np.abs(rng.standard_normal((8, 16, 9))).astype(np.float32)
lay = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=bk, weight=rng.standard_normal((72, 8)).astype(np.float32))
y, _ = L.LutConv(8, 3, 1, 1, lay).forward(x)
torch.cuda.synchronize()
print("sanitizer workload ok")
