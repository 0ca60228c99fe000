"""Encode / gather split of the small caller layers (configs[0] LUT Linear,
configs[2] conv stages) as CUDA graphs with the stack bench's L2 flush: the
whole layer, the encode alone and the gather alone (from stored codes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_03213_b200 import workloads as W  # noqa: E402
from paper_2302_03213_b200._lib import check, load  # noqa: E402

dev = torch.device("cuda", 0)
lib = load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, device=dev)


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        flush.zero_()
        flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def sp():
    return torch.cuda.current_stream().cuda_stream


layer, a = W.linear(dev, 1024, 768, 768, 16, 16, False)
n, c, k, v, m = 1024, layer.c, layer.k, layer.v, layer.m
cs = layer.code_stride
codes = torch.empty((n, cs), dtype=torch.uint8, device=dev)
out = torch.empty((n, m), device=dev)
enc = lambda: check(lib.lut_encode_f32(a.data_ptr(), n, c * v, layer.books_prep.data_ptr(), c, k, v, codes.data_ptr(),
                                       8, cs, None, sp()))
gat = lambda: check(lib.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, layer.table.data_ptr(), None, 0,
                                       out.data_ptr(), 0, None, sp()))
# lut_gather_f32 expects stride C codes: use a compact copy for the gather-only timing
codes_c = torch.empty((n, c), dtype=torch.uint8, device=dev)
enc()
codes_c.copy_(codes[:, :c])
gat_c = lambda: check(lib.lut_gather_f32(codes_c.data_ptr(), 8, n, c, k, m, layer.table.data_ptr(), None, 0,
                                         out.data_ptr(), 0, None, sp()))
print(f"cfg1 layer {graph_time(lambda: layer.forward_device(a, False, out=out, codes=codes)):7.1f} us  "
      f"encode {graph_time(enc):7.1f} us  gather {graph_time(gat_c):7.1f} us", flush=True)
for conv, x in W.resnet_convs(dev, batch=256):
    lut = conv.lut
    print(f"cfg3 conv Cin={lut.c:3d} layer {graph_time(lambda: conv(x)):7.1f} us", flush=True)
