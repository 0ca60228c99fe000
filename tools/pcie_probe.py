"""Pinned-host <-> HBM copy bandwidth on this box: H2D alone, D2H alone, both at once
(two streams) — the link roofline of bench.py's e2e number."""
import json
import time

import torch

nbytes = 4 << 30
h_in = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
d_out = torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


bi = timed(both)
print(json.dumps({"bytes": nbytes, "h2d_GBps": nbytes / h2d / 1e9, "d2h_GBps": nbytes / d2h / 1e9,
                  "concurrent_each_GBps": nbytes / bi / 1e9}))
