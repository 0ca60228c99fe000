"""configs[0] (1024 x 768 -> 768, V = 16, K = 16, f32 table): the encode and the gather
timed separately and together, each as a CUDA graph replayed after an L2 flush (the
stack bench's conditions)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03213_b200 as L  # noqa: E402
from paper_2302_03213_b200 import workloads as W  # noqa: E402
from paper_2302_03213_b200._lib import load  # noqa: E402

dev = torch.device("cuda", 0)
lib = load()
layer, a = W.linear(dev, 1024, 768, 768, 16, 16, False)
n, c, k, v, m = 1024, 48, 16, 16, 768
stride = int(lib.lut_code_stride(c))
codes = torch.empty((n, stride), dtype=torch.uint8, device=dev)
out = torch.empty((n, m), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)


def sp():
    return torch.cuda.current_stream().cuda_stream


def enc():
    assert lib.lut_encode_f32(a.data_ptr(), n, c * v, layer.books_prep.data_ptr(), c, k, v, codes.data_ptr(), 8, stride,
                              None, sp()) == 0


def gat():
    assert lib.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, layer.table.data_ptr(), None, 0, out.data_ptr(), 0,
                              None, sp()) == 0


def both():
    layer.forward_device(a, False, out=out, codes=codes)


def timed(fn, name, steps=30):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(steps):
        flush.zero_()
        flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{name:28s} median {ts[len(ts) // 2]:6.2f} us  min {ts[0]:6.2f} us", flush=True)


timed(lambda: None if torch.zeros(1, device=dev).add_(1) is None else None, "tiny torch kernel (floor)")
timed(enc, "encode only")
timed(gat, "gather only (codes in L2?)")
timed(lambda: (enc(), gat()), "encode + gather, no PDL")
timed(both, "layer (encode + PDL gather)")
