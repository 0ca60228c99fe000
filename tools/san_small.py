"""Small shapes through every kernel, for compute-sanitizer memcheck."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_03213_b200 as L
from oracle import lut_oracle as O

rng = O.make_rng(3)
for (n, c, k, v, m) in [(600, 8, 16, 32, 40), (300, 12, 8, 4, 33), (70, 5, 16, 9, 7), (513, 16, 64, 16, 130),
                        (700, 20, 16, 32, 260), (333, 3, 64, 32, 64), (1000, 128, 16, 32, 256)]:
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
# plain int8 pair-gather epilogue (no bias), the configs[4] call, on a partial tile
from paper_2302_03213_b200._lib import load
lib = load()
n, c, k, v, m = 777, 128, 16, 32, 384
g = torch.Generator(device="cuda").manual_seed(5)
lay = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=torch.randn((c, k, v), generator=g, device="cuda"),
                 weight=torch.randn((c * v, m), generator=g, device="cuda") * 0.02, qat=True, gather="tensor")
a = torch.randn((n, c * v), generator=g, device="cuda")
cs = int(lib.lut_code_stride(c))
codes = torch.empty((n, cs), dtype=torch.uint8, device="cuda")
out = torch.empty((n, m), device="cuda")
sp = torch.cuda.current_stream().cuda_stream
assert lib.lut_encode_f32(a.data_ptr(), n, c * v, lay.books_prep.data_ptr(), c, k, v, codes.data_ptr(), 8, cs, None, sp) == 0
assert lib.lut_gather_onehot(codes.data_ptr(), cs, n, c, k, m, 1, lay.onehot_image(True).data_ptr(),
                             lay.qtable.scales_tensor("cuda").data_ptr(), 0, None, 0, out.data_ptr(), None, 0, sp) == 0
torch.cuda.synchronize()
print("sanitizer workload ok")
