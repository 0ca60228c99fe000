"""Generate golden vectors by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the read-only reference package `lutkit` from /root/reference and
records its outputs on seeded inputs.  Inputs are NOT stored: every case is
regenerated from its seed with Philox4x64-10 (`np.random.Philox`, identical
on every platform — pinned by the seed-42 golden stream below), so the GPU box
(which has no /root/reference) rebuilds the same bytes.  Outputs are stored as
full arrays where small (codes, i32 sums) and as SHA-256 of the raw bytes for
f32 results that must match bitwise.

Case families mirror the reference's own tests for the path:
  encode25   tests/test_kernels.py:46-57   centroid_search_fast == encode_hard
  ties       tests/test_kernels.py:59-75, test_pq.py:82-88
  crit1      tests/test_acceptance.py:53-103 (200 shapes, every 5th with a crafted tie)
  gather15   tests/test_kernels.py:79-91 (+ :93-117 widening / bound / hand cases)
  quant      tests/test_quant.py:16-68
  pqamm      tests/test_pq.py:145-157
  im2col     tests/test_tensor.py:41-98
  cfg1       BASELINE.json configs[0] (N=1024, 768->768, V=16, K=16)
  cfg5s      configs[4] encode geometry (D=4096, V=32, K=16 and 64) on a 2048-row subsample
  conv       configs[2] geometry on a batch-2 sample (16ch 8x8, V=9, K=16)
  hash       hashing.py:171-196 trees built by the reference on a seeded sample
  lutn_*     container.py:1-23 models written by the reference (bytes stored) and
             its predict_fast outputs on the loaded model (pipeline.py:206-225)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import lutkit  # noqa: E402
from lutkit import hashing, kernels, pq, quant, tensor  # noqa: E402
from lutkit.rng import make_rng  # noqa: E402
from lutkit.softpq import LutLayer  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def inst(rng, n, c, k, v, m):
    d = c * v
    a = rng.standard_normal((n, d)).astype(F32)
    books = rng.standard_normal((c, k, v)).astype(F32)
    b = rng.standard_normal((d, m)).astype(F32)
    return a, books, b


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": "lutkit " + lutkit.__version__, "cases": {}}

    # Philox golden stream (tests/test_tensor.py:175-187)
    g = make_rng(42).integers(0, 2**64, size=16, dtype=np.uint64, endpoint=False)
    meta["philox42"] = [int(x) for x in g]

    # encode25: tests/test_kernels.py:46-57
    enc25 = []
    for seed in range(25):
        rng = make_rng(seed)
        n = int(rng.integers(1, 50))
        c = int(rng.integers(1, 7))
        k = int(rng.choice([4, 8, 16]))
        v = int(rng.choice([2, 3, 4, 9]))
        a, books, _ = inst(rng, n, c, k, v, 1)
        nb = int(rng.integers(1, 20))
        kb = int(rng.integers(1, 8))
        plan = kernels.KernelPlan(n_block=nb, k_block=kb)
        codes = kernels.centroid_search_fast(a, books, plan)
        assert np.array_equal(codes, pq.encode_hard(a, books))
        arrays[f"encode25_{seed}"] = codes
        enc25.append({"seed": seed, "n": n, "c": c, "k": k, "v": v, "n_block": nb, "k_block": kb})
    meta["cases"]["encode25"] = enc25

    # ties
    rng = make_rng(99)
    books = rng.standard_normal((2, 8, 3)).astype(F32)
    books[0, 5] = books[0, 2]
    books[1, 7] = books[1, 0]
    a = np.repeat(np.hstack([books[0, 2][None], books[1, 0][None]]).astype(F32), 4, axis=0)
    arrays["ties_dup"] = kernels.centroid_search_fast(a, books)
    books = np.array([[[0.0, 0.0], [2.0, 0.0]]], dtype=F32)
    arrays["ties_equi"] = kernels.centroid_search_fast(np.array([[1.0, 5.0]], F32), books,
                                                       kernels.KernelPlan(k_block=1))
    books = np.array([[[0.0], [2.0], [2.0]]], dtype=F32)
    arrays["ties_lowest"] = np.concatenate([
        pq.encode_hard(np.array([[1.0]], F32), books),
        pq.encode_hard(np.array([[2.0]], F32), books)])

    # crit1: tests/test_acceptance.py:53-103
    rng = make_rng(20250101)
    crit = []
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
        tie = trial % 5 == 0
        if tie:
            books[0, k - 1] = books[0, 0]
            a[0, :v] = books[0, 0]
        nb = int(rng.integers(1, 65))
        kb = int(rng.integers(1, k + 1))
        plan = kernels.KernelPlan(n_block=nb, k_block=kb)
        codes = pq.encode_hard(a, books)
        assert np.array_equal(codes, kernels.centroid_search_fast(a, books, plan))
        table = pq.build_table(b, books)
        layer = LutLayer(cfg=pq.PqConfig(v=v, k=k), books=books, weight=b,
                         bias=np.zeros(m, F32))
        fout = kernels.lut_layer_infer(a, layer, plan, integer=False)
        qt = quant.quantize_table(table)
        i32 = kernels.lut_gather_i32(codes, qt.q, plan)
        arrays[f"crit1_codes_{trial}"] = codes
        arrays[f"crit1_i32_{trial}"] = i32
        crit.append({"trial": trial, "n": n, "c": c, "k": k, "v": v, "m": m, "tie": tie,
                     "table_sha": sha(table), "out_f32_sha": sha(fout), "q_sha": sha(qt.q),
                     "scale": float(qt.scale)})
    meta["cases"]["crit1"] = crit

    # gather15 + widening / bound / hand
    g15 = []
    for seed in range(15):
        rng = make_rng(100 + seed)
        n = int(rng.integers(1, 40))
        c = int(rng.integers(1, 30))
        k = int(rng.choice([4, 8, 16]))
        m = int(rng.integers(1, 25))
        q = rng.integers(-127, 128, size=(c, k, m)).astype(np.int8)
        enc = rng.integers(0, k, size=(n, c)).astype(np.uint8)
        gs = int(rng.integers(1, 10))
        arrays[f"gather15_{seed}"] = kernels.lut_gather_i32(enc, q, kernels.KernelPlan(group_size=gs))
        g15.append({"seed": seed, "n": n, "c": c, "k": k, "m": m, "group_size": gs})
    meta["cases"]["gather15"] = g15
    rng = make_rng(7)
    q = rng.integers(-127, 128, size=(300, 4, 6)).astype(np.int8)
    enc = rng.integers(0, 4, size=(9, 300)).astype(np.uint8)
    arrays["gather_c300"] = kernels.lut_gather_i32(enc, q, kernels.KernelPlan(group_size=128))
    arrays["gather_bound258"] = kernels.lut_gather_i32(
        np.zeros((4, 258), np.uint8), np.full((258, 2, 3), 127, np.int8), kernels.KernelPlan(group_size=258))
    arrays["gather_hand200"] = kernels.lut_gather_i32(
        np.zeros((1, 200), np.uint8), np.full((200, 1, 1), 127, np.int8), kernels.KernelPlan(group_size=128))
    qt = quant.LookupTableI8(q=np.array([[[1, -2], [3, 4]]], np.int8), scale=np.float32(0.5))
    arrays["gather_single"] = kernels.lut_gather_accumulate(np.array([[1]], np.uint8), qt)
    rng = make_rng(8)
    t = rng.standard_normal((5, 4, 3)).astype(F32)
    qt = quant.quantize_table(t)
    enc = rng.integers(0, 4, size=(7, 5)).astype(np.uint8)
    meta["cases"]["scale_once"] = {"out_sha": sha(kernels.lut_gather_accumulate(enc, qt)),
                                   "q_sha": sha(qt.q), "scale": float(qt.scale)}

    # quant KATs: tests/test_quant.py
    qk = {}
    for name, vals in {"scale127": [1.27, 0.50, -0.25], "endpoint": [3.7, -1.0],
                       "endpoint_neg": [-3.7, 1.0]}.items():
        qt = quant.quantize_table(np.asarray(vals, F32).reshape(1, 1, -1))
        qk[name] = {"vals": vals, "q": qt.q.ravel().tolist(), "scale": float(qt.scale)}
    s = 2.0 / 127.0
    hv = np.array([2.0, s * 0.5, s * 1.5], dtype=F32)
    qt = quant.quantize_table(hv.reshape(1, 1, -1))
    qk["half_even"] = {"vals": [float(x) for x in hv], "q": qt.q.ravel().tolist(), "scale": float(qt.scale)}
    qz = quant.quantize_table(np.zeros((2, 3, 4), F32))
    qk["zero"] = {"scale": float(qz.scale)}
    qr = []
    for seed in range(20):
        rng = make_rng(seed)
        t = (rng.standard_normal((2, 4, 6)) * rng.uniform(0.01, 100)).astype(F32)
        qt = quant.quantize_table(t)
        qr.append({"seed": seed, "q_sha": sha(qt.q), "scale": float(qt.scale)})
    qk["random20"] = qr
    meta["cases"]["quant"] = qk

    # pq_amm composed pipeline: tests/test_pq.py:145-157
    pa = []
    for seed in range(100):
        rng = make_rng(200 + seed)
        c = int(rng.integers(1, 6))
        v = int(rng.integers(1, 4))
        k = int(rng.integers(1, 9))
        n = int(rng.integers(1, 12))
        m = int(rng.integers(1, 9))
        a, books, b = inst(rng, n, c, k, v, m)
        out = pq.pq_amm(a, b, pq.PqConfig(v=v, k=k), books)
        pa.append({"seed": seed, "c": c, "v": v, "k": k, "n": n, "m": m, "out_sha": sha(out),
                   "table_sha": sha(pq.build_table(b, books))})
    meta["cases"]["pqamm"] = pa

    # im2col
    im = []
    for trial in range(8):
        rng = make_rng(100 + trial)
        cin = int(rng.integers(1, 4))
        cout = int(rng.integers(1, 4))
        h = int(rng.integers(3, 7))
        w = int(rng.integers(3, 7))
        kh = int(rng.integers(1, min(4, h + 1)))
        kw = int(rng.integers(1, min(4, w + 1)))
        stride = int(rng.integers(1, 3))
        pad = int(rng.integers(0, 2))
        x = rng.standard_normal((2, cin, h, w)).astype(F32)
        cols = tensor.im2col(x, kh, kw, stride=stride, pad=pad)
        im.append({"trial": trial, "cin": cin, "cout": cout, "h": h, "w": w, "kh": kh, "kw": kw,
                   "stride": stride, "pad": pad, "shape": list(cols.shape), "sha": sha(cols)})
    meta["cases"]["im2col"] = im

    # cfg1: BASELINE configs[0]
    rng = make_rng(1)
    n, d, m, v, k = 1024, 768, 768, 16, 16
    c = d // v
    a = rng.standard_normal((n, d)).astype(F32)
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((d, m)) / np.sqrt(d)).astype(F32)
    layer = LutLayer(cfg=pq.PqConfig(v=v, k=k), books=books, weight=w, bias=np.zeros(m, F32), qat=True)
    codes = kernels.centroid_search_fast(a, books)
    arrays["cfg1_codes"] = codes
    meta["cases"]["cfg1"] = {
        "seed": 1, "n": n, "d": d, "m": m, "v": v, "k": k,
        "table_sha": sha(layer.table), "q_sha": sha(layer.qtable.q), "scale": float(layer.qtable.scale),
        "out_f32_sha": sha(kernels.lut_layer_infer(a, layer, integer=False)),
        "out_i8_sha": sha(kernels.lut_layer_infer(a, layer, integer=True)),
        "near_ties_1e6": int(np.sum(_gaps(a, books) < 1e-6)),
    }

    # cfg5 geometry subsample (K=16 and K=64 codes)
    for k in (16, 64):
        rng = make_rng(5000 + k)
        n, d, v = 2048, 4096, 32
        a = rng.standard_normal((n, d)).astype(F32)
        books = rng.standard_normal((d // v, k, v)).astype(F32)
        arrays[f"cfg5s_k{k}_codes"] = kernels.centroid_search_fast(a, books, kernels.KernelPlan(n_block=2048))
        meta["cases"][f"cfg5s_k{k}"] = {"seed": 5000 + k, "n": n, "d": d, "v": v, "k": k}

    # conv (configs[2] geometry, small batch): x=|N(0,1)|, V=9, C=Cin, K=16
    rng = make_rng(33)
    bsz, cin, hh, ww = 2, 16, 8, 8
    x = np.abs(rng.standard_normal((bsz, cin, hh, ww))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    wconv = (rng.standard_normal((cin * 9, cin)) * np.sqrt(2.0 / (9 * cin))).astype(F32)
    cols = tensor.im2col(x, 3, 3, 1, 1)
    layer = LutLayer(cfg=pq.PqConfig(v=9, k=16), books=books, weight=wconv, bias=np.zeros(cin, F32))
    arrays["conv_codes"] = kernels.centroid_search_fast(cols, books)
    y = kernels.lut_layer_infer(cols, layer, integer=False)
    meta["cases"]["conv"] = {"seed": 33, "b": bsz, "cin": cin, "h": hh, "w": ww, "cols_sha": sha(cols),
                             "table_sha": sha(layer.table), "out_f32_sha": sha(y),
                             "nchw_sha": sha(np.ascontiguousarray(y.reshape(bsz, hh, ww, cin).transpose(0, 3, 1, 2)))}

    # hash trees
    rng = make_rng(77)
    c, v, k, lv = 3, 4, 16, 6
    samples = rng.standard_normal((800, c * v)).astype(F32)
    books = rng.standard_normal((c, k, v)).astype(F32)
    trees = [hashing.build_hash_tree(samples[:, i * v:(i + 1) * v], books[i], lv) for i in range(c)]
    for i, t in enumerate(trees):
        arrays[f"hash_dims_{i}"] = np.asarray(t.dims, np.int64)
        arrays[f"hash_thr_{i}"] = np.asarray(t.thresholds, F32)
        arrays[f"hash_leaves_{i}"] = np.asarray(t.leaves, np.uint8)
    arrays["hash_codes"] = hashing.encode_hash(samples[:64], trees)
    meta["cases"]["hash"] = {"seed": 77, "c": c, "v": v, "k": k, "levels": lv, "rows": 64}

    _lutn_cases(arrays, meta)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays")


def _lut(rng, c, k, v, m, qat, bias=True, tree_levels=0, samples=None):
    books = rng.standard_normal((c, k, v)).astype(F32)
    weight = rng.standard_normal((c * v, m)).astype(F32)
    b = rng.standard_normal(m).astype(F32) if bias else np.zeros(m, F32)
    lut = LutLayer(cfg=pq.PqConfig(v=v, k=k), books=books, weight=weight, bias=b, qat=qat)
    if tree_levels:
        lut.trees = [hashing.build_hash_tree(samples[:, i * v:(i + 1) * v], books[i], tree_levels) for i in range(c)]
    return lut


def _lutn_cases(arrays, meta):
    """Containers written by the reference + predict_fast of the loaded model."""
    from lutkit import container, pipeline
    from lutkit.model import Conv, Dense, LutConv, LutDense, Model, Relu

    # A: LutDense(f32, bias, trees) -> relu -> LutDense(i8, bias, trees) -> relu -> Dense
    rng = make_rng(501)
    x = rng.standard_normal((96, 16)).astype(F32)
    l1 = _lut(rng, 4, 8, 4, 12, qat=False, tree_levels=3, samples=x)
    h = np.maximum(kernels.lut_layer_infer(x, l1), 0)
    l2 = _lut(rng, 3, 16, 4, 7, qat=True, tree_levels=4, samples=np.pad(h, ((0, 0), (0, 0))))
    head = Dense(7, 3, rng)
    head.bias = rng.standard_normal(3).astype(F32)
    model = Model([LutDense(l1), Relu(), LutDense(l2), Relu(), head])
    raw = container.model_bytes(model)
    loaded = container.model_from_bytes(raw)
    arrays["lutn_a_bytes"] = np.frombuffer(raw, np.uint8)
    arrays["lutn_a_x"] = x
    arrays["lutn_a_dist"] = pipeline.predict_fast(loaded, x)
    arrays["lutn_a_f32"] = pipeline.predict_fast(loaded, x, integer=False)
    arrays["lutn_a_hash"] = pipeline.predict_fast(loaded, x, encoder="hash")
    arrays["lutn_a_hidden"] = pipeline.predict_fast(Model(loaded.layers[:4]), x)

    # B: LutConv(i8) -> relu -> Conv -> relu -> Dense(flatten)
    rng = make_rng(502)
    x = rng.standard_normal((2, 3, 8, 8)).astype(F32)
    lc = _lut(rng, 3, 16, 9, 8, qat=True)
    conv = Conv(8, 4, kernel=3, stride=2, pad=1, rng=rng)
    conv.bias = rng.standard_normal(4).astype(F32)
    head = Dense(4 * 4 * 4, 10, rng)
    model = Model([LutConv(3, 3, 1, 1, lc), Relu(), conv, Relu(), head])
    raw = container.model_bytes(model)
    loaded = container.model_from_bytes(raw)
    arrays["lutn_b_bytes"] = np.frombuffer(raw, np.uint8)
    arrays["lutn_b_x"] = x
    arrays["lutn_b_dist"] = pipeline.predict_fast(loaded, x)
    arrays["lutn_b_f32"] = pipeline.predict_fast(loaded, x, integer=False)
    arrays["lutn_b_conv"] = pipeline.predict_fast(Model(loaded.layers[:2]), x)
    meta["cases"]["lutn"] = {"a_seed": 501, "b_seed": 502, "a_len": int(arrays["lutn_a_bytes"].size),
                             "b_len": int(arrays["lutn_b_bytes"].size)}


def _gaps(a, books):
    d = pq.subvector_distances(a, books)
    part = np.partition(d, 1, axis=2)
    return (part[..., 1] - part[..., 0]) / np.maximum(np.abs(part[..., 1]), 1e-300)


if __name__ == "__main__":
    main()
