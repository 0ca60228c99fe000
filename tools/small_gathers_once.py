"""One lut_gather_f32 call per small BASELINE shape (configs[1] FFN pair, configs[0],
the three configs[2] convs) — the launch list an ncu capture of the small gathers needs.

usage: ncu ... python tools/small_gathers_once.py [lib.so]
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_03213_b200._lib import SIGNATURES  # noqa: E402

h = C.CDLL(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2302_03213_b200/_lib/liblutgpu.so"))
for name, (res, args) in SIGNATURES.items():
    if hasattr(h, name):
        f = getattr(h, name)
        f.restype, f.argtypes = res, args
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
sp = torch.cuda.current_stream().cuda_stream
for name, n, c, k, m, hw, epi in [
    ("ffn1", 4096, 24, 16, 3072, 0, True),
    ("ffn2", 4096, 96, 16, 768, 0, True),
    ("cfg1", 1024, 48, 16, 768, 0, False),
    ("conv1", 256 * 1024, 16, 16, 16, 1024, True),
    ("conv2", 256 * 256, 32, 16, 32, 256, True),
    ("conv3", 256 * 64, 64, 16, 64, 64, True),
]:
    codes = torch.randint(0, k, (n, c), generator=g, device=dev, dtype=torch.uint8)
    table = torch.randn((c, k, m), generator=g, device=dev)
    bias = torch.randn(m, generator=g, device=dev) if epi else None
    out = torch.empty(n * m, device=dev)
    torch.cuda.synchronize()
    assert h.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, table.data_ptr(),
                            bias.data_ptr() if bias is not None else None, 1 if epi else 0, out.data_ptr(), hw,
                            None, sp) == 0
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
