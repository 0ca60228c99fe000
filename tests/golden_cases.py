"""Regenerate the inputs of every golden case from its seed (no /root/reference
needed) and expose the reference's recorded outputs.  Shared by the CPU oracle
pin tests and the GPU parity tests, so both check against the same bytes."""

from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from oracle import lut_oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F32 = np.float32


def sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


@dataclass
class Golden:
    meta: dict
    arrays: dict

    @classmethod
    def load(cls) -> "Golden":
        with open(os.path.join(HERE, "golden.json")) as f:
            meta = json.load(f)
        with np.load(os.path.join(HERE, "golden.npz")) as z:
            arrays = {k: z[k] for k in z.files}
        return cls(meta, arrays)

    def cases(self, family):
        return self.meta["cases"][family]


def encode25_inputs(case):
    rng = O.make_rng(case["seed"])
    n = int(rng.integers(1, 50))
    c = int(rng.integers(1, 7))
    k = int(rng.choice([4, 8, 16]))
    v = int(rng.choice([2, 3, 4, 9]))
    assert (n, c, k, v) == (case["n"], case["c"], case["k"], case["v"])
    a, books, _ = O.random_instance(rng, n, c, k, v, 1)
    return a, books


def ties_dup_inputs():
    rng = O.make_rng(99)
    books = rng.standard_normal((2, 8, 3)).astype(F32)
    books[0, 5] = books[0, 2]
    books[1, 7] = books[1, 0]
    a = np.repeat(np.hstack([books[0, 2][None], books[1, 0][None]]).astype(F32), 4, axis=0)
    return a, books


def crit1_inputs():
    """Yields (case_index, a, books, b) for the 200 acceptance shapes."""
    rng = O.make_rng(20250101)
    for trial in range(200):
        k = int(rng.choice([4, 8, 16]))
        v = int(rng.choice([2, 3, 4, 9, 16]))
        c = int(rng.integers(1, max(2, 144 // v) + 1))
        d = c * v
        n = int(rng.integers(1, 65))
        m = int(rng.integers(1, 97))
        a = rng.standard_normal((n, d)).astype(F32)
        books = rng.standard_normal((c, k, v)).astype(F32)
        b = rng.standard_normal((d, m)).astype(F32)
        if trial % 5 == 0:
            books[0, k - 1] = books[0, 0]
            a[0, :v] = books[0, 0]
        rng.integers(1, 65)
        rng.integers(1, k + 1)
        yield trial, a, books, b


def gather15_inputs(case):
    rng = O.make_rng(100 + case["seed"])
    n = int(rng.integers(1, 40))
    c = int(rng.integers(1, 30))
    k = int(rng.choice([4, 8, 16]))
    m = int(rng.integers(1, 25))
    q = rng.integers(-127, 128, size=(c, k, m)).astype(np.int8)
    enc = rng.integers(0, k, size=(n, c)).astype(np.uint8)
    return enc, q


def gather_c300_inputs():
    rng = O.make_rng(7)
    q = rng.integers(-127, 128, size=(300, 4, 6)).astype(np.int8)
    enc = rng.integers(0, 4, size=(9, 300)).astype(np.uint8)
    return enc, q


def scale_once_inputs():
    rng = O.make_rng(8)
    t = rng.standard_normal((5, 4, 3)).astype(F32)
    enc = rng.integers(0, 4, size=(7, 5)).astype(np.uint8)
    return enc, t


def pqamm_inputs(case):
    rng = O.make_rng(200 + case["seed"])
    c = int(rng.integers(1, 6))
    v = int(rng.integers(1, 4))
    k = int(rng.integers(1, 9))
    n = int(rng.integers(1, 12))
    m = int(rng.integers(1, 9))
    return O.random_instance(rng, n, c, k, v, m)


def im2col_inputs(case):
    rng = O.make_rng(100 + case["trial"])
    cin = int(rng.integers(1, 4))
    rng.integers(1, 4)
    h = int(rng.integers(3, 7))
    w = int(rng.integers(3, 7))
    kh = int(rng.integers(1, min(4, h + 1)))
    kw = int(rng.integers(1, min(4, w + 1)))
    stride = int(rng.integers(1, 3))
    pad = int(rng.integers(0, 2))
    x = rng.standard_normal((2, cin, h, w)).astype(F32)
    return x, kh, kw, stride, pad


def cfg1_inputs():
    """BASELINE configs[0]: N=1024, D=M=768, V=16 -> C=48, K=16; W ~ N(0, 1/D)."""
    rng = O.make_rng(1)
    n, d, m, v, k = 1024, 768, 768, 16, 16
    a = rng.standard_normal((n, d)).astype(F32)
    books = rng.standard_normal((d // v, k, v)).astype(F32)
    w = (rng.standard_normal((d, m)) / np.sqrt(d)).astype(F32)
    return a, books, w


def cfg5s_inputs(k):
    rng = O.make_rng(5000 + k)
    n, d, v = 2048, 4096, 32
    a = rng.standard_normal((n, d)).astype(F32)
    books = rng.standard_normal((d // v, k, v)).astype(F32)
    return a, books


def conv_inputs():
    rng = O.make_rng(33)
    bsz, cin, hh, ww = 2, 16, 8, 8
    x = np.abs(rng.standard_normal((bsz, cin, hh, ww))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    wconv = (rng.standard_normal((cin * 9, cin)) * np.sqrt(2.0 / (9 * cin))).astype(F32)
    return x, books, wconv


def hash_inputs(g: Golden):
    case = g.cases("hash")
    rng = O.make_rng(case["seed"])
    c, v, k = case["c"], case["v"], case["k"]
    samples = rng.standard_normal((800, c * v)).astype(F32)
    trees = [(g.arrays[f"hash_dims_{i}"], g.arrays[f"hash_thr_{i}"], g.arrays[f"hash_leaves_{i}"])
             for i in range(c)]
    return samples[: case["rows"]], trees
