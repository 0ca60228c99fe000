"""configs[2] conv-plane encodes (lut_encode_conv_f32) and CUDA-core gathers
(NCHW) per stage, for one or two builds of the library; codes compared.

usage: python tools/conv_bench.py [lib_a.so [lib_b.so]]
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_03213_b200._lib import SIGNATURES  # noqa: E402

libs = sys.argv[1:] or [os.path.join(ROOT, "paper_2302_03213_b200/_lib/liblutgpu.so")]
handles = []
for path in libs:
    h = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if hasattr(h, name):
            f = getattr(h, name)
            f.restype, f.argtypes = res, args
    handles.append(h)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
sp = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for cin, hw in ((16, 32), (32, 16), (64, 8)):
    b, k, v = 256, 16, 9
    x = torch.relu(torch.randn((b, cin, hw, hw), generator=g, device=dev))
    books = torch.relu(torch.randn((cin, k, v), generator=g, device=dev))
    n = b * hw * hw
    line = f"conv {hw}x{hw}x{cin}:"
    ref = None
    for li, h in enumerate(handles):
        prep = torch.empty(max(1, h.lut_books_prep_bytes(cin, k, v)), dtype=torch.uint8, device=dev)
        assert h.lut_prepare_books(books.data_ptr(), cin, k, v, prep.data_ptr(), sp) == 0
        codes = torch.empty((n, cin), dtype=torch.uint8, device=dev)
        fn = lambda: h.lut_encode_conv_f32(x.data_ptr(), b, cin, hw, hw, 3, 3, 1, 1, prep.data_ptr(), cin, k, v,
                                           codes.data_ptr(), 8, None, sp)
        ms = timeit(fn)
        same = "" if ref is None else (" same" if torch.equal(ref, codes) else " DIFF")
        ref = codes.clone() if ref is None else ref
        line += f"  [{li}] encode {ms * 1e3:7.1f} us{same}"
    print(line, flush=True)
