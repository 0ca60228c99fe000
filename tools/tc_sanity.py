"""Quick tensor-core one-hot gather sanity check (tiny shapes) against numpy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_03213_b200 as L

rng = np.random.default_rng(0)
for (n, c, k, m) in [(128, 8, 16, 64), (200, 16, 16, 100), (1000, 128, 16, 256), (130, 3, 4, 17), (64, 4, 64, 40)]:
    q = rng.integers(-127, 128, size=(c, k, m)).astype(np.int8)
    enc = rng.integers(0, k, size=(n, c)).astype(np.uint8)
    want = np.zeros((n, m), np.int64)
    for ci in range(c):
        want += q[ci, enc[:, ci]]
    got = L.kernels.lut_gather_i32_tc(enc, q)
    torch.cuda.synchronize()
    ok = np.array_equal(got, want)
    print((n, c, k, m), "ok" if ok else "MISMATCH", flush=True)
    if not ok:
        bad = np.argwhere(got != want)
        print(" first bad", bad[:5], got[tuple(bad[0])], want[tuple(bad[0])], flush=True)
