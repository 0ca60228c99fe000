"""GPU: per-(codebook, m-tile) int8 scales — BASELINE configs[1]'s table
format ("int8 with per-(c, m-tile) fp32 scale").  An extension with no
reference counterpart (SPEC.md:361 rejects per-codebook scales; parity
UNPINNED): checked bitwise against the oracle restatement
(quantize_table_cmtile, lut_gather_accumulate_cmtile)."""

import numpy as np
import pytest

from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


@pytest.mark.parametrize("c,k,m,mtile", [(24, 16, 3072, 128), (96, 16, 768, 128), (5, 8, 100, 32), (3, 16, 40, 64)])
def test_cmtile_quantize_and_gather(L, c, k, m, mtile):
    rng = O.make_rng(c * m + mtile)
    table = (rng.standard_normal((c, k, m)) * rng.uniform(0.01, 3.0, (c, 1, 1))).astype(F32)
    qt = L.quantize_table(table, scale_mtile=mtile, per_codebook=True)
    q_ref, s_ref = O.quantize_table_cmtile(table, mtile)
    assert qt.per_codebook and np.asarray(qt.scale).shape == s_ref.shape
    assert np.array_equal(qt.q, q_ref) and np.asarray(qt.scale).tobytes() == s_ref.tobytes()
    enc = rng.integers(0, k, (777, c)).astype(np.uint8)
    got = L.lut_gather_accumulate(enc, qt)
    want = O.lut_gather_accumulate_cmtile(enc, q_ref, s_ref, mtile)
    assert got.tobytes() == want.tobytes()


def test_cmtile_layer_and_ffn(L):
    """A LUT layer with per-(c, m-tile) scales through lut_layer_infer (bias,
    GELU fused) == oracle; the configs[1] FFN pair builds and runs with them."""
    import torch

    rng = O.make_rng(31)
    n, c, k, v, m, mt = 600, 24, 16, 32, 384, 128
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
    bias = rng.standard_normal(m).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias, qat=True, scale_mtile=mt,
                       scale_per_codebook=True)
    assert not layer.uses_tensor_cores(True)
    got = L.lut_layer_infer(a, layer, integer=True)
    q, s = O.quantize_table_cmtile(O.build_table(w, books), mt)
    enc = O.encode_hard(a, books)
    want = O.lut_gather_accumulate_cmtile(enc, q, s, mt) + bias
    assert got.tobytes() == want.astype(F32).tobytes()
    gl = layer.with_act("gelu")
    got_g = L.lut_layer_infer(a, gl, integer=True)
    np.testing.assert_allclose(got_g, O.gelu_erf(want), rtol=1e-5, atol=1e-5)
    from paper_2302_03213_b200 import workloads as W

    ffn, x = W.ffn_pair(torch.device("cuda", 0), tokens=512, scale_mtile=128, per_codebook=True)
    y = ffn(x)
    assert y.shape == (512, 768) and torch.isfinite(y).all()


def test_cmtile_not_storable_in_lutn(L):
    """The version-1 .lutn container holds one scale per table (container.py):
    per-(codebook, m-tile) scales are refused with ContainerError, not dropped."""
    rng = O.make_rng(5)
    books = rng.standard_normal((4, 16, 8)).astype(F32)
    w = rng.standard_normal((32, 64)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=8, k=16), books=books, weight=w, qat=True, scale_mtile=32,
                       scale_per_codebook=True)
    dense = L.LutDense(layer)
    with pytest.raises(L.ContainerError):
        L.model_bytes(L.Model([dense]))


def test_cmtile_tensor_digit_planes(L):
    """gather="tensor" opts a per-(codebook, m-tile) layer into the tensor cores: the
    dequantized table as 4 int8 digit planes (no exact integer sum exists across
    codebooks), within the north star's fp tolerance (rtol / atol 1e-5) of the bitwise
    f32 sum; bias + GELU through the same call."""
    rng = O.make_rng(77)
    n, c, k, v, m, mt = 900, 24, 16, 32, 3072, 128
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
    bias = rng.standard_normal(m).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    mk = lambda g: L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias, qat=True, scale_mtile=mt,
                              scale_per_codebook=True, gather=g)
    lt, lc = mk("tensor"), mk("auto")
    assert lt.uses_tensor_cores(True) and not lc.uses_tensor_cores(True)
    got = L.lut_layer_infer(a, lt, integer=True)
    ref = L.lut_layer_infer(a, lc, integer=True)
    q, s = O.quantize_table_cmtile(O.build_table(w, books), mt)
    want = (O.lut_gather_accumulate_cmtile(O.encode_hard(a, books), q, s, mt) + bias).astype(F32)
    assert ref.tobytes() == want.tobytes()
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(L.lut_layer_infer(a, lt.with_act("gelu"), integer=True), O.gelu_erf(want),
                               rtol=1e-5, atol=1e-5)
