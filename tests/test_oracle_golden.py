"""Pin the CPU oracle against golden vectors recorded from the reference itself.

If these pass, every GPU parity test that compares against `oracle/` is
transitively a comparison against the reference's own outputs."""

import numpy as np
import pytest

import golden_cases as G
from oracle import lut_oracle as O

F32 = np.float32


def test_philox_stream_seed42(golden):
    draws = O.make_rng(42).integers(0, 2**64, size=16, dtype=np.uint64, endpoint=False)
    assert [int(x) for x in draws] == golden.meta["philox42"]


def test_encode25(golden):
    for case in golden.cases("encode25"):
        a, books = G.encode25_inputs(case)
        want = golden.arrays[f"encode25_{case['seed']}"]
        np.testing.assert_array_equal(O.encode_hard(a, books), want)
        np.testing.assert_array_equal(
            O.centroid_search_fast(a, books, case["n_block"], case["k_block"]), want)


def test_ties(golden):
    a, books = G.ties_dup_inputs()
    np.testing.assert_array_equal(O.centroid_search_fast(a, books), golden.arrays["ties_dup"])
    assert golden.arrays["ties_dup"][0, 0] == 2 and golden.arrays["ties_dup"][0, 1] == 0
    books = np.array([[[0.0, 0.0], [2.0, 0.0]]], dtype=F32)
    np.testing.assert_array_equal(
        O.centroid_search_fast(np.array([[1.0, 5.0]], F32), books, k_block=1), golden.arrays["ties_equi"])
    books = np.array([[[0.0], [2.0], [2.0]]], dtype=F32)
    got = np.concatenate([O.encode_hard(np.array([[1.0]], F32), books),
                          O.encode_hard(np.array([[2.0]], F32), books)])
    np.testing.assert_array_equal(got, golden.arrays["ties_lowest"])


def test_crit1_all_paths(golden):
    meta = golden.cases("crit1")
    for trial, a, books, b in G.crit1_inputs():
        case = meta[trial]
        codes = O.encode_hard(a, books)
        np.testing.assert_array_equal(codes, golden.arrays[f"crit1_codes_{trial}"])
        table = O.build_table(b, books)
        assert G.sha(table) == case["table_sha"], trial
        out = O.lut_layer_infer(a, books, table=table, bias=np.zeros(b.shape[1], F32), integer=False)
        assert G.sha(out) == case["out_f32_sha"], trial
        q, scale = O.quantize_table(table)
        assert G.sha(q) == case["q_sha"] and float(scale) == case["scale"]
        np.testing.assert_array_equal(O.lut_gather_i32(codes, q), golden.arrays[f"crit1_i32_{trial}"])


def test_gather_cases(golden):
    for case in golden.cases("gather15"):
        enc, q = G.gather15_inputs(case)
        np.testing.assert_array_equal(O.lut_gather_i32(enc, q, case["group_size"]),
                                      golden.arrays[f"gather15_{case['seed']}"])
    enc, q = G.gather_c300_inputs()
    np.testing.assert_array_equal(O.lut_gather_i32(enc, q, 128), golden.arrays["gather_c300"])
    got = O.lut_gather_i32(np.zeros((4, 258), np.uint8), np.full((258, 2, 3), 127, np.int8), 258)
    np.testing.assert_array_equal(got, golden.arrays["gather_bound258"])
    assert (got == 32766).all()
    got = O.lut_gather_i32(np.zeros((1, 200), np.uint8), np.full((200, 1, 1), 127, np.int8), 128)
    np.testing.assert_array_equal(got, golden.arrays["gather_hand200"])
    got = O.lut_gather_accumulate(np.array([[1]], np.uint8), np.array([[[1, -2], [3, 4]]], np.int8), 0.5)
    np.testing.assert_array_equal(got, golden.arrays["gather_single"])
    enc, t = G.scale_once_inputs()
    q, s = O.quantize_table(t)
    case = golden.cases("scale_once")
    assert G.sha(q) == case["q_sha"] and float(s) == case["scale"]
    assert G.sha(O.lut_gather_accumulate(enc, q, s)) == case["out_sha"]


def test_bad_index_raises():
    with pytest.raises(O.OracleError) as e:
        O.lut_gather_i32(np.array([[7]], np.uint8), np.zeros((1, 4, 2), np.int8))
    assert e.value.kind == "CorruptionError"
    with pytest.raises(O.OracleError):
        O.lut_matmul_ref(np.array([[4]], np.uint8), np.zeros((1, 4, 2), F32))


def test_quant_kats(golden):
    qk = golden.cases("quant")
    for name in ("scale127", "endpoint", "endpoint_neg", "half_even"):
        q, s = O.quantize_table(np.asarray(qk[name]["vals"], F32).reshape(1, 1, -1))
        assert q.ravel().tolist() == qk[name]["q"] and float(s) == qk[name]["scale"], name
    _, s = O.quantize_table(np.zeros((2, 3, 4), F32))
    assert float(s) == qk["zero"]["scale"] == 1.0
    for case in qk["random20"]:
        rng = O.make_rng(case["seed"])
        t = (rng.standard_normal((2, 4, 6)) * rng.uniform(0.01, 100)).astype(F32)
        q, s = O.quantize_table(t)
        assert G.sha(q) == case["q_sha"] and float(s) == case["scale"]


def test_pqamm(golden):
    for case in golden.cases("pqamm"):
        a, books, b = G.pqamm_inputs(case)
        table = O.build_table(b, books)
        assert G.sha(table) == case["table_sha"]
        assert G.sha(O.lut_matmul_ref(O.encode_hard(a, books), table)) == case["out_sha"]


def test_im2col(golden):
    for case in golden.cases("im2col"):
        x, kh, kw, stride, pad = G.im2col_inputs(case)
        cols = O.im2col(x, kh, kw, stride, pad)
        assert list(cols.shape) == case["shape"] and G.sha(cols) == case["sha"]


def test_cfg1(golden):
    case = golden.cases("cfg1")
    a, books, w = G.cfg1_inputs()
    codes = O.centroid_search_fast(a, books)
    np.testing.assert_array_equal(codes, golden.arrays["cfg1_codes"])
    table = O.build_table(w, books)
    assert G.sha(table) == case["table_sha"]
    q, s = O.quantize_table(table)
    assert G.sha(q) == case["q_sha"] and float(s) == case["scale"]
    bias = np.zeros(w.shape[1], F32)
    assert G.sha(O.lut_layer_infer(a, books, table=table, bias=bias, integer=False)) == case["out_f32_sha"]
    assert G.sha(O.lut_layer_infer(a, books, q=q, scale=s, bias=bias)) == case["out_i8_sha"]


@pytest.mark.parametrize("k", [16, 64])
def test_cfg5_subsample_codes(golden, k):
    a, books = G.cfg5s_inputs(k)
    np.testing.assert_array_equal(O.centroid_search_fast(a, books, n_block=2048),
                                  golden.arrays[f"cfg5s_k{k}_codes"])


def test_conv(golden):
    case = golden.cases("conv")
    x, books, wconv = G.conv_inputs()
    cols = O.im2col(x, 3, 3, 1, 1)
    assert G.sha(cols) == case["cols_sha"]
    np.testing.assert_array_equal(O.centroid_search_fast(cols, books), golden.arrays["conv_codes"])
    table = O.build_table(wconv, books)
    assert G.sha(table) == case["table_sha"]
    y = O.lut_layer_infer(cols, books, table=table, bias=np.zeros(16, F32), integer=False)
    assert G.sha(y) == case["out_f32_sha"]


def test_hash_encode(golden):
    a, trees = G.hash_inputs(golden)
    np.testing.assert_array_equal(O.encode_hash(a, trees), golden.arrays["hash_codes"])


def test_flop_counter_examples():
    c = O.flop_counter(100, 64, 128, 16, 8)
    assert (c["encode"], c["lookup_aggregate"], c["dense"]) == (102400, 102400, 819200)
    c = O.flop_counter(1, 768, 768, 16, 32)
    assert c["dense"] / (c["encode"] + c["lookup_aggregate"]) == pytest.approx(19.2)
