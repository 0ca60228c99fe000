"""Probe-build sweep of the row-parallel f32 gather geometry (LUTGPU_F32_NP /
LUTGPU_F32_T) on the small BASELINE shapes; L2 flushed between timed calls.

usage: python tools/f32_sweep.py path/to/liblutgpu_probe.so
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_03213_b200._lib import SIGNATURES  # noqa: E402

h = C.CDLL(sys.argv[1])
for name, (res, args) in SIGNATURES.items():
    if hasattr(h, name):
        f = getattr(h, name)
        f.restype, f.argtypes = res, args
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
sp = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, device=dev)


def graph_time(fn, launches=20, reps=5):
    """Device time per launch: `launches` back-to-back launches captured in one CUDA graph."""
    global sp
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        sp = side.cuda_stream
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=side):
            sp = torch.cuda.current_stream().cuda_stream
            for _ in range(launches):
                fn()
    sp = torch.cuda.current_stream().cuda_stream
    gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / launches)
    return sorted(ts)[len(ts) // 2]


def timeit(fn, reps=7, cold=True):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
            flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


SHAPES = [
    ("ffn1", 4096, 24, 16, 3072, 0, True),
    ("ffn2", 4096, 96, 16, 768, 0, True),
    ("cfg1", 1024, 48, 16, 768, 0, False),
    ("conv1", 256 * 1024, 16, 16, 16, 1024, True),
    ("conv2", 256 * 256, 32, 16, 32, 256, True),
    ("conv3", 256 * 64, 64, 16, 64, 64, True),
]
for name, n, c, k, m, hw, epi in SHAPES:
    codes = torch.randint(0, k, (n, c), generator=g, device=dev, dtype=torch.uint8)
    table = torch.randn((c, k, m), generator=g, device=dev)
    bias = torch.randn(m, generator=g, device=dev) if epi else None
    act = 1 if epi else 0
    out = torch.empty(n * m, device=dev)
    fn = lambda: h.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, table.data_ptr(),
                                  bias.data_ptr() if bias is not None else None, act, out.data_ptr(), hw, None, sp)
    timeit = lambda f, cold=True: graph_time(f) if cold else 0.0
    for key in ("LUTGPU_F32_NP", "LUTGPU_F32_T"):
        os.environ.pop(key, None)
    base_cold, base_hot = timeit(fn), timeit(fn, cold=False)
    ref = out.clone()
    print(f"{name}: default cold {base_cold * 1e3:7.1f} us hot {base_hot * 1e3:7.1f} us", flush=True)
    for npair in (1, 2, 4, 8):
        if 2 * npair > 2 * m:
            continue
        for th in (128, 256, 512, 1024):
            os.environ["LUTGPU_F32_NP"] = str(npair)
            os.environ["LUTGPU_F32_T"] = str(th)
            out.zero_()
            try:
                cold, hot = timeit(fn), timeit(fn, cold=False)
            except Exception as e:  # noqa: BLE001
                print(f"  NP={npair} T={th}: {e}")
                continue
            same = torch.equal(out, ref)
            print(f"  NP={npair} T={th:4d}: cold {cold * 1e3:7.1f} us hot {hot * 1e3:7.1f} us {'same' if same else 'DIFF'}",
                  flush=True)
    for key in ("LUTGPU_F32_NP", "LUTGPU_F32_T"):
        os.environ.pop(key, None)
