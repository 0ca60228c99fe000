"""Callers either side of the path, layer by layer against
the oracle on activations captured from our own forward: configs[1] FFN pair
(int8 + GELU, per-table and per-m-tile scales), configs[2] ResNet20 3x3 convs,
configs[3] BERT encoder (LUT layers 3+)."""

import numpy as np
import pytest
import torch

from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32
DEV = "cuda"


def _np(t):
    return t.detach().cpu().numpy()


def _oracle_linear(lut, a_np, integer=True):
    """Oracle of one LUT linear incl. its epilogue (bias, act)."""
    books = _np(lut.books)
    codes = O.centroid_search_fast(a_np, books)
    if integer:
        q = _np(lut.qtable.q)
        scales = _np(lut.qtable.scales_tensor(lut.device))
        if lut.qtable.scale_mtile:
            out = O.lut_gather_accumulate_mtile(codes, q, scales, lut.qtable.scale_mtile)
        else:
            out = O.lut_gather_accumulate(codes, q, scales[0])
    else:
        out = O.lut_gather_f32(codes, _np(lut.table))
    if lut.bias.numel():
        out = out + _np(lut.bias)
    if lut.act == "gelu":
        out = O.gelu_erf(out)
    elif lut.act == "relu":
        out = np.maximum(out, 0)
    return out


def _check(lut, a, got, integer=True):
    want = _oracle_linear(lut, _np(a).reshape(-1, lut.d), integer)
    got = _np(got).reshape(want.shape)
    if lut.act == "gelu":  # f32 erff in the epilogue vs f64 erf rounded: contract rtol/atol 1e-5
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    else:
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("scale_mtile", [0, 128])
@pytest.mark.parametrize("gather", ["cuda", "tensor"])
def test_ffn_pair(scale_mtile, gather):
    from paper_2302_03213_b200 import workloads as W

    ffn, x = W.ffn_pair(torch.device(DEV), tokens=192, scale_mtile=scale_mtile, held_rows=512, gather=gather)
    assert ffn.up.lut.c == 24 and ffn.down.lut.c == 96 and ffn.up.lut.act == "gelu"
    h = ffn.up(x)
    y = ffn.down(h)
    _check(ffn.up.lut, x, h)
    _check(ffn.down.lut, h, y)
    torch.testing.assert_close(ffn(x), y, rtol=0, atol=0)


def test_resnet_convs():
    from paper_2302_03213_b200 import workloads as W

    for conv, x in W.resnet_convs(torch.device(DEV), batch=2):
        lut = conv.lut
        assert (lut.v, lut.c, lut.m) == (9, conv.in_channels, conv.in_channels)
        got = _np(conv(x))
        xn = _np(x)
        cols = O.im2col(xn, 3, 3, 1, 1)
        want = O.lut_layer_infer(cols, _np(lut.books), table=_np(lut.table), integer=False)
        b, _, h, w = xn.shape
        want = want.reshape(b, h, w, -1).transpose(0, 3, 1, 2)
        np.testing.assert_array_equal(got, want)


def test_bert_encoder_layer_by_layer():
    from paper_2302_03213_b200 import workloads as W

    cfg = W.BertConfig(layers=4, dense_layers=2)
    model, tokens = W.bert_encoder(torch.device(DEV), batch=2, seq=16, cfg=cfg, calib_batch=2)
    luts = model.lut_linears()
    assert len(luts) == 12 and {i for i, _, _ in luts} == {2, 3}
    seen = []
    hooks = [mod.register_forward_hook(lambda m_, inp, out_, key=(i, n): seen.append((key, m_, inp[0], out_)))
             for i, n, mod in luts]
    out = model(tokens)
    for hk in hooks:
        hk.remove()
    assert out.shape == tokens.shape and torch.isfinite(out).all()
    assert len(seen) == 12
    for (_, name), mod, a, y in seen:
        _check(mod.lut, a, y)
