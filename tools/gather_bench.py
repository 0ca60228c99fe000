"""CUDA-core gather kernels on the BASELINE shapes: times lut_gather_f32 /
lut_gather_i8 (C ABI, CUDA events) for one or two builds of the library and
checks that both give the same bytes.

usage: python tools/gather_bench.py [lib_a.so [lib_b.so]]
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

SHAPES = [  # name, n, C, K, M, out_hw, bias+relu
    ("cfg5_f32/i8 (2^18 rows)", 1 << 18, 128, 16, 4096, 0, False),
    ("cfg1 1024x768->768", 1024, 48, 16, 768, 0, False),
    ("cfg3 conv1 32x32x16", 256 * 1024, 16, 16, 16, 1024, True),
    ("cfg3 conv2 16x16x32", 256 * 256, 32, 16, 32, 256, True),
    ("cfg3 conv3 8x8x64", 256 * 64, 64, 16, 64, 64, True),
    ("k64 C=128 M=512", 1 << 16, 128, 64, 512, 0, False),
]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
sp = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, device=dev)  # read after the write: dirty lines written back untimed


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for name, n, c, k, m, hw, epi in SHAPES:
    codes = torch.randint(0, k, (n, c), generator=g, device=dev, dtype=torch.uint8)
    table = torch.randn((c, k, m), generator=g, device=dev)
    q = torch.randint(-127, 128, (c, k, m), generator=g, device=dev, dtype=torch.int8)
    scale = torch.tensor([0.01], device=dev)
    bias = torch.randn(m, generator=g, device=dev) if epi else None
    act = 1 if epi else 0
    outs = {}
    for kind in ("f32", "i8"):
        line = f"{name:28s} {kind}:"
        ref = None
        for li, h in enumerate(handles):
            out = torch.empty(n * m, device=dev)
            if kind == "f32":
                fn = lambda: h.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, table.data_ptr(),
                                              bias.data_ptr() if bias is not None else None, act, out.data_ptr(),
                                              hw, None, sp)
            else:
                fn = lambda: h.lut_gather_i8(codes.data_ptr(), 8, n, c, k, m, q.data_ptr(), scale.data_ptr(), 0,
                                             bias.data_ptr() if bias is not None else None, act, out.data_ptr(),
                                             None, hw, None, sp)
            ms = timeit(fn)
            same = "" if ref is None else (" same" if torch.equal(ref, out) else " DIFF")
            ref = out if ref is None else ref
            lookups = n * m * c * (4 if kind == "f32" else 1)
            line += f"  [{li}] {ms * 1e3:9.1f} us ({lookups / (ms / 1e3) / 1e12:6.2f} TB/s lookups){same}"
        print(line, flush=True)
