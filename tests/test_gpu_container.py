"""`.lutn` models written by the reference, loaded straight into HBM and run
through predict_fast, against the reference's own predict_fast outputs on the
loaded model (pipeline.py:206-225; make_golden.py `lutn_*`)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


def _load(golden, name, **kw):
    from paper_2302_03213_b200.container import model_from_bytes

    return model_from_bytes(golden.arrays[f"lutn_{name}_bytes"].tobytes(), **kw)


def test_layers_resident_in_hbm(L, golden):
    model = _load(golden, "a")
    names = [type(layer).__name__ for layer in model.layers]
    assert names == ["LutDense", "Relu", "LutDense", "Relu", "Dense"]
    lut2 = model.layers[2].lut
    assert lut2.books.is_cuda and lut2.qtable.q.is_cuda and lut2.table.is_cuda
    assert lut2.bias.abs().sum().item() == 0          # bias folded into the table (container.py:102-104)


@pytest.mark.parametrize("gather", ["auto", "cuda", "tensor"])
def test_lut_stack_bitwise(L, golden, gather):
    """LUT -> relu -> LUT(int8) -> relu: no dense layer, so bit-identical."""
    from paper_2302_03213_b200.nn import Model, predict_fast

    model = _load(golden, "a", gather=gather)
    x = golden.arrays["lutn_a_x"]
    np.testing.assert_array_equal(predict_fast(Model(model.layers[:4]), x), golden.arrays["lutn_a_hidden"])


def test_model_a_dist_and_f32(L, golden):
    from paper_2302_03213_b200.nn import predict_fast

    model = _load(golden, "a")
    x = golden.arrays["lutn_a_x"]
    # the final Dense is a cuBLAS fp32 GEMM vs numpy's sgemm: f32 association only
    np.testing.assert_allclose(predict_fast(model, x), golden.arrays["lutn_a_dist"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(predict_fast(model, x, integer=False), golden.arrays["lutn_a_f32"], rtol=1e-5,
                               atol=1e-5)
    np.testing.assert_allclose(model.predict_logits(x), golden.arrays["lutn_a_dist"], rtol=1e-5, atol=1e-5)


def test_model_a_hash(L, golden):
    from paper_2302_03213_b200.nn import predict_fast

    model = _load(golden, "a")
    x = golden.arrays["lutn_a_x"]
    np.testing.assert_allclose(predict_fast(model, x, encoder="hash"), golden.arrays["lutn_a_hash"], rtol=1e-5,
                               atol=1e-5)


def test_model_b_conv(L, golden):
    from paper_2302_03213_b200.nn import Model, predict_fast

    model = _load(golden, "b")
    x = golden.arrays["lutn_b_x"]
    np.testing.assert_array_equal(predict_fast(Model(model.layers[:2]), x), golden.arrays["lutn_b_conv"])
    np.testing.assert_allclose(predict_fast(model, x), golden.arrays["lutn_b_dist"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(predict_fast(model, x, integer=False), golden.arrays["lutn_b_f32"], rtol=1e-5,
                               atol=1e-5)
    got = predict_fast(model, torch.from_numpy(x).cuda())
    assert got.is_cuda
    np.testing.assert_allclose(got.cpu().numpy(), golden.arrays["lutn_b_dist"], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("name", ["a", "b"])
def test_write_back_byte_identical(L, golden, name, tmp_path):
    from paper_2302_03213_b200.container import load_model, model_bytes, save_model

    raw = golden.arrays[f"lutn_{name}_bytes"].tobytes()
    model = _load(golden, name)
    assert model_bytes(model) == raw
    save_model(tmp_path / "m.lutn", model)
    assert load_model(tmp_path / "m.lutn") is not None and (tmp_path / "m.lutn").read_bytes() == raw


def test_bias_folded_on_write(L, golden):
    """A layer with a bias writes table + bias/C (container.py:102-104)."""
    from oracle import lut_oracle as O
    from paper_2302_03213_b200.container import model_bytes, parse_records
    from paper_2302_03213_b200.nn import LutDense, Model

    rng = O.make_rng(7)
    books = rng.standard_normal((4, 8, 2)).astype(np.float32)
    w = rng.standard_normal((8, 6)).astype(np.float32)
    b = rng.standard_normal(6).astype(np.float32)
    for qat in (False, True):
        lut = L.LutLayer(cfg=L.PqConfig(v=2, k=8), books=books, weight=w, bias=b, qat=qat)
        rec = parse_records(model_bytes(Model([LutDense(lut)])))[0][0]
        folded = O.build_table(w, books) + (b / np.float32(4)).astype(np.float32)[None, None, :]
        if qat:
            q, s = O.quantize_table(folded)
            np.testing.assert_array_equal(rec.q, q)
            assert np.float32(rec.scale) == np.float32(s)
        else:
            np.testing.assert_array_equal(rec.table, folded)
