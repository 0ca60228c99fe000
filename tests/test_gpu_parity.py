"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the pinned oracle, on the reference's own test cases."""

import numpy as np
import pytest

import golden_cases as G
from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


def test_encode25(L, golden):
    for case in golden.cases("encode25"):
        a, books = G.encode25_inputs(case)
        plan = L.KernelPlan(n_block=case["n_block"], k_block=case["k_block"])
        np.testing.assert_array_equal(L.centroid_search_fast(a, books, plan), golden.arrays[f"encode25_{case['seed']}"])


def test_ties(L, golden):
    a, books = G.ties_dup_inputs()
    for plan in (L.KernelPlan(), L.KernelPlan(n_block=1, k_block=2), L.KernelPlan(k_block=3)):
        got, ties = L.centroid_search_fast(a, books, plan, return_near_ties=True)
        np.testing.assert_array_equal(got, golden.arrays["ties_dup"])
        assert got[0, 0] == 2 and got[0, 1] == 0
        assert ties == 8  # every (row, codebook) is an exact tie -> fp64 re-decision
    books = np.array([[[0.0, 0.0], [2.0, 0.0]]], dtype=F32)
    got = L.centroid_search_fast(np.array([[1.0, 5.0]], F32), books, L.KernelPlan(k_block=1))
    np.testing.assert_array_equal(got, golden.arrays["ties_equi"])
    books = np.array([[[0.0], [2.0], [2.0]]], dtype=F32)
    got = np.concatenate([L.encode_hard(np.array([[1.0]], F32), books), L.encode_hard(np.array([[2.0]], F32), books)])
    np.testing.assert_array_equal(got, golden.arrays["ties_lowest"])


def test_crit1_equivalence(L, golden):
    """Acceptance criterion 1 (tests/test_acceptance.py:53-103) on the GPU:
    indices exact, f32 path bitwise, i32 bitwise, table/quant bitwise."""
    meta = golden.cases("crit1")
    for trial, a, books, b in G.crit1_inputs():
        case = meta[trial]
        codes = L.centroid_search_fast(a, books)
        np.testing.assert_array_equal(codes, golden.arrays[f"crit1_codes_{trial}"], err_msg=str(trial))
        table = L.build_table(b, books)
        assert G.sha(table) == case["table_sha"], trial
        layer = L.LutLayer(cfg=L.PqConfig(v=case["v"], k=case["k"]), books=books, weight=b,
                           bias=np.zeros(case["m"], F32))
        out = L.lut_layer_infer(a, layer, integer=False)
        assert out.dtype == np.float32 and G.sha(out) == case["out_f32_sha"], trial
        qt = L.quantize_table(table)
        assert G.sha(qt.q) == case["q_sha"] and float(qt.scale) == case["scale"], trial
        np.testing.assert_array_equal(L.lut_gather_i32(codes, qt.q), golden.arrays[f"crit1_i32_{trial}"])


def test_gather_cases(L, golden):
    for case in golden.cases("gather15"):
        enc, q = G.gather15_inputs(case)
        got = L.lut_gather_i32(enc, q, L.KernelPlan(group_size=case["group_size"]))
        assert got.dtype == np.int32
        np.testing.assert_array_equal(got, golden.arrays[f"gather15_{case['seed']}"])
    enc, q = G.gather_c300_inputs()
    np.testing.assert_array_equal(L.lut_gather_i32(enc, q), golden.arrays["gather_c300"])
    got = L.lut_gather_i32(np.zeros((4, 258), np.uint8), np.full((258, 2, 3), 127, np.int8), L.KernelPlan(group_size=258))
    assert (got == 258 * 127).all()
    got = L.lut_gather_i32(np.zeros((1, 200), np.uint8), np.full((200, 1, 1), 127, np.int8))
    assert got[0, 0] == 25400
    qt = L.LookupTableI8(q=np.array([[[1, -2], [3, 4]]], np.int8), scale=np.float32(0.5))
    np.testing.assert_array_equal(L.lut_gather_accumulate(np.array([[1]], np.uint8), qt), [[1.5, 2.0]])
    enc, t = G.scale_once_inputs()
    qt = L.quantize_table(t)
    case = golden.cases("scale_once")
    assert G.sha(qt.q) == case["q_sha"] and float(qt.scale) == case["scale"]
    assert G.sha(L.lut_gather_accumulate(enc, qt)) == case["out_sha"]


def test_bad_index_raises(L):
    with pytest.raises(L.CorruptionError):
        L.lut_gather_i32(np.array([[7]], np.uint8), np.zeros((1, 4, 2), np.int8))
    with pytest.raises(L.CorruptionError):
        L.lut_gather_f32(np.array([[4]], np.uint8), np.zeros((1, 4, 2), F32))
    # device-side detection (codes already on the GPU, u8 dtype)
    import torch

    enc = torch.tensor([[0, 9]], dtype=torch.uint8, device="cuda")
    with pytest.raises(L.CorruptionError):
        L.lut_gather_f32(enc, torch.zeros((2, 4, 3), device="cuda"))
    # and the flag is cleared: a valid call afterwards succeeds
    ok = L.lut_gather_f32(torch.tensor([[0, 3]], dtype=torch.uint8, device="cuda"), torch.ones((2, 4, 3), device="cuda"))
    assert ok.cpu().numpy().tolist() == [[2.0, 2.0, 2.0]]


def test_integer_without_qtable_raises(L):
    rng = O.make_rng(12345)
    books = rng.standard_normal((4, 8, 3)).astype(F32)
    w = rng.standard_normal((12, 5)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=3, k=8), books=books, weight=w, bias=np.zeros(5, F32))
    with pytest.raises(L.ConfigError):
        L.lut_layer_infer(rng.standard_normal((3, 12)).astype(F32), layer, integer=True)


def test_quant_kats(L, golden):
    qk = golden.cases("quant")
    for name in ("scale127", "endpoint", "endpoint_neg", "half_even"):
        qt = L.quantize_table(np.asarray(qk[name]["vals"], F32).reshape(1, 1, -1))
        assert qt.q.ravel().tolist() == qk[name]["q"] and float(qt.scale) == qk[name]["scale"], name
    qt = L.quantize_table(np.zeros((2, 3, 4), F32))
    assert float(qt.scale) == 1.0 and not qt.q.any()
    for case in qk["random20"]:
        rng = O.make_rng(case["seed"])
        t = (rng.standard_normal((2, 4, 6)) * rng.uniform(0.01, 100)).astype(F32)
        qt = L.quantize_table(t)
        assert G.sha(qt.q) == case["q_sha"] and float(qt.scale) == case["scale"]
    with pytest.raises(L.DataError):
        L.quantize_table(np.array([[[np.nan, 1.0]]], F32))


def test_pqamm(L, golden):
    for case in golden.cases("pqamm"):
        a, books, b = G.pqamm_inputs(case)
        out = L.pq_amm(a, b, L.PqConfig(v=case["v"], k=case["k"]), books)
        assert G.sha(out) == case["out_sha"], case["seed"]


def test_im2col(L, golden):
    for case in golden.cases("im2col"):
        x, kh, kw, stride, pad = G.im2col_inputs(case)
        cols = L.im2col(x, kh, kw, stride, pad)
        assert list(cols.shape) == case["shape"] and G.sha(cols) == case["sha"]


def test_cfg1(L, golden):
    """BASELINE configs[0] end to end, bitwise against the reference."""
    case = golden.cases("cfg1")
    a, books, w = G.cfg1_inputs()
    np.testing.assert_array_equal(L.centroid_search_fast(a, books), golden.arrays["cfg1_codes"])
    layer = L.LutLayer(cfg=L.PqConfig(v=16, k=16), books=books, weight=w, bias=np.zeros(768, F32), qat=True)
    assert G.sha(layer.table.cpu().numpy()) == case["table_sha"]
    assert G.sha(layer.qtable.q.cpu().numpy()) == case["q_sha"]
    assert float(layer.qtable.scale) == case["scale"]
    assert G.sha(L.lut_layer_infer(a, layer, integer=False)) == case["out_f32_sha"]
    assert G.sha(L.lut_layer_infer(a, layer, integer=True)) == case["out_i8_sha"]


@pytest.mark.parametrize("k", [16, 64])
def test_cfg5_subsample_codes(L, golden, k):
    """configs[4] encode geometry (D=4096, V=32): the TMA kernel."""
    a, books = G.cfg5s_inputs(k)
    codes, ties = L.centroid_search_fast(a, books, return_near_ties=True)
    np.testing.assert_array_equal(codes, golden.arrays[f"cfg5s_k{k}_codes"])
    assert ties < codes.size * 1e-3


def test_conv_fused(L, golden):
    """configs[2] geometry: im2col fused into encode, NCHW fused into gather."""
    case = golden.cases("conv")
    x, books, wconv = G.conv_inputs()
    layer = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=books, weight=wconv, bias=np.zeros(16, F32))
    conv = L.LutConv(16, 3, 1, 1, layer)
    y, _ = conv.forward(x)
    assert y.shape == (2, 16, 8, 8)
    assert G.sha(y) == case["nchw_sha"]
    cols = L.im2col(x, 3, 3, 1, 1)
    np.testing.assert_array_equal(L.centroid_search_fast(cols, books), golden.arrays["conv_codes"])


# --------------------------------------------------------------- sweeps

SHAPES = [  # (n, c, k, v, m) — TMA encode path needs v in {4,8,16,32} and n >= 256
    (300, 8, 16, 32, 40), (1000, 24, 16, 16, 33), (777, 16, 64, 8, 17), (513, 12, 8, 4, 64),
    (256, 3, 128, 32, 5), (1, 5, 16, 32, 7), (70, 7, 256, 3, 9), (129, 4, 1, 9, 12),
    (200, 2, 16, 100, 6), (65, 9, 33, 64, 130), (600, 1, 16, 1, 1), (0, 4, 16, 4, 8),
]


@pytest.mark.parametrize("shape", SHAPES)
def test_sweep_against_oracle(L, shape):
    n, c, k, v, m = shape
    rng = O.make_rng(hash(shape) % (2**32))
    a, books, b = O.random_instance(rng, n, c, k, v, m)
    bias = rng.standard_normal(m).astype(F32)
    want_codes = O.encode_hard(a, books)
    codes = L.centroid_search_fast(a, books)
    np.testing.assert_array_equal(codes, want_codes)
    table = O.build_table(b, books)
    assert L.build_table(b, books).tobytes() == table.tobytes()
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=b, bias=bias, qat=True)
    out = L.lut_layer_infer(a, layer, integer=False)
    assert out.tobytes() == O.lut_layer_infer(a, books, table=table, bias=bias, integer=False).tobytes()
    q, s = O.quantize_table(table)
    out8 = L.lut_layer_infer(a, layer, integer=True)
    assert out8.tobytes() == O.lut_layer_infer(a, books, q=q, scale=s, bias=bias).tobytes()


def test_u4_codes_match_u8(L):
    import torch

    from paper_2302_03213_b200.kernels import encode_device, prepare_books

    rng = O.make_rng(4)
    for (n, c, v) in ((1000, 32, 32), (700, 15, 16), (90, 7, 3)):
        a, books, _ = O.random_instance(rng, n, c, 16, v, 1)
        a_d, b_d = torch.from_numpy(a).cuda(), torch.from_numpy(books).cuda()
        prep = prepare_books(b_d)
        u8 = encode_device(a_d, prep, c, 16, v, 8).cpu().numpy()
        u4 = encode_device(a_d, prep, c, 16, v, 4).cpu().numpy()
        lo, hi = u4 & 15, u4 >> 4
        unpacked = np.stack([lo, hi], axis=2).reshape(n, -1)[:, :c]
        np.testing.assert_array_equal(unpacked, u8)
        np.testing.assert_array_equal(u8, O.encode_hard(a, books))


def test_epilogues_extension(L):
    """GELU / ReLU epilogues and per-m-tile int8 scales (BASELINE configs[1]
    extensions; parity unpinned: oracle restatement, tolerance stated)."""
    rng = O.make_rng(21)
    n, c, k, v, m = 300, 24, 16, 32, 96
    a, books, b = O.random_instance(rng, n, c, k, v, m)
    b *= 0.02
    bias = rng.standard_normal(m).astype(F32) * 0.1
    table = O.build_table(b, books)
    codes = O.encode_hard(a, books)
    for act in ("relu", "gelu"):
        layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=b, bias=bias, act=act)
        got = L.lut_layer_infer(a, layer, integer=False)
        pre = O.lut_matmul_ref(codes, table) + bias
        want = np.maximum(pre, 0) if act == "relu" else O.gelu_erf(pre)
        if act == "relu":
            assert got.tobytes() == want.astype(F32).tobytes()
        else:
            np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=b, bias=bias, qat=True, scale_mtile=32)
    q, scales = O.quantize_table_mtile(table, 32)
    np.testing.assert_array_equal(layer.qtable.q.cpu().numpy(), q)
    np.testing.assert_array_equal(layer.qtable.scale.cpu().numpy(), scales)
    got = L.lut_layer_infer(a, layer, integer=True)
    want = O.lut_gather_accumulate_mtile(codes, q, scales, 32) + bias
    assert got.tobytes() == want.astype(F32).tobytes()


def test_large_rows_properties(L):
    """BASELINE configs[4] width at 64K rows (1 GiB of input): the pipelined
    host executor equals the device path bitwise, sampled rows equal the
    oracle, and outputs are row-permutation equivariant."""
    import torch

    n, d, m, v, k = 65536, 4096, 256, 32, 16
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((n, d), generator=g, device="cuda")
    rng = O.make_rng(55)
    books = rng.standard_normal((d // v, k, v)).astype(F32)
    w = (rng.standard_normal((d, m)) / np.sqrt(d)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, qat=True)
    out_dev = L.lut_layer_infer(a, layer, integer=False)
    out_host = L.lut_layer_infer(a.cpu().numpy(), layer, integer=False)  # > 32 MiB -> native executor
    assert out_dev.cpu().numpy().tobytes() == out_host.tobytes()
    idx = np.sort(rng.choice(n, 192, replace=False))
    a_s = a[torch.as_tensor(idx, device="cuda")].cpu().numpy()
    table = O.build_table(w, books)
    want = O.lut_layer_infer(a_s, books, table=table, integer=False)
    assert out_host[idx].tobytes() == want.tobytes()
    perm = torch.randperm(n, device="cuda", generator=g)
    out_perm = L.lut_layer_infer(a[perm], layer, integer=False)
    assert torch.equal(out_perm, out_dev[perm])
    o8 = L.lut_layer_infer(a, layer, integer=True)
    q, s = O.quantize_table(table)
    want8 = O.lut_layer_infer(a_s, books, q=q, scale=s)
    assert o8.cpu().numpy()[idx].tobytes() == want8.tobytes()


def test_reference_style_layer_object(L):
    """A duck-typed reference LutLayer (numpy arrays) is accepted as is."""
    from types import SimpleNamespace

    rng = O.make_rng(9)
    a, books, b = O.random_instance(rng, 50, 6, 8, 3, 7)
    table = O.build_table(b, books)
    q, s = O.quantize_table(table)
    ref_layer = SimpleNamespace(cfg=SimpleNamespace(v=3, k=8), books=books, table=table,
                                qtable=SimpleNamespace(q=q, scale=s), bias=np.zeros(7, F32), trees=None)
    got = L.lut_layer_infer(a, ref_layer)
    assert got.tobytes() == O.lut_layer_infer(a, books, q=q, scale=s, bias=np.zeros(7, F32)).tobytes()
    got = L.lut_layer_infer(a, ref_layer, integer=False)
    assert got.tobytes() == O.lut_layer_infer(a, books, table=table, bias=np.zeros(7, F32), integer=False).tobytes()


# --------------------------------------------------------- tensor-core path

def test_tc_int8_crit1_bitwise(L, golden):
    """tcgen05 one-hot int8 gather == reference i32 / accumulate, bitwise, on the
    200 acceptance shapes; f32 digit planes within rtol/atol 1e-5."""
    meta = golden.cases("crit1")
    for trial, a, books, b in G.crit1_inputs():
        case = meta[trial]
        codes = golden.arrays[f"crit1_codes_{trial}"]
        table = O.build_table(b, books)
        q, s = O.quantize_table(table)
        np.testing.assert_array_equal(L.kernels.lut_gather_i32_tc(codes, q), golden.arrays[f"crit1_i32_{trial}"],
                                      err_msg=str(trial))
        layer = L.LutLayer(cfg=L.PqConfig(v=case["v"], k=case["k"]), books=books, weight=b,
                           bias=np.zeros(case["m"], F32), qat=True, gather="tensor")
        assert layer.uses_tensor_cores(True) and layer.uses_tensor_cores(False)
        out8 = L.lut_layer_infer(a, layer, integer=True)
        want8 = O.lut_gather_accumulate(codes, q, s) + np.zeros(case["m"], F32)
        assert out8.tobytes() == want8.tobytes(), trial
        outf = L.lut_layer_infer(a, layer, integer=False)
        wantf = O.lut_matmul_ref(codes, table)
        np.testing.assert_allclose(outf, wantf, rtol=1e-5, atol=1e-5, err_msg=str(trial))


def test_tc_cfg1(L, golden):
    case = golden.cases("cfg1")
    a, books, w = G.cfg1_inputs()
    layer = L.LutLayer(cfg=L.PqConfig(v=16, k=16), books=books, weight=w, bias=np.zeros(768, F32), qat=True,
                       gather="tensor")
    assert G.sha(L.lut_layer_infer(a, layer, integer=True)) == case["out_i8_sha"]
    table = O.build_table(w, books)
    want = O.lut_matmul_ref(golden.arrays["cfg1_codes"], table)
    got = L.lut_layer_infer(a, layer, integer=False)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    # digits=4 is far tighter than the contract: error <= C * max|T| * 2^-31 + f32 rounding
    assert np.max(np.abs(got.astype(np.float64) - want)) < 2e-6


@pytest.mark.parametrize("shape", [(8192, 128, 16, 32, 4096), (5000, 24, 16, 32, 3072), (3000, 96, 16, 32, 768),
                                   (777, 33, 8, 4, 100), (300, 64, 64, 8, 130), (4096, 128, 64, 32, 512)])
def test_tc_matches_cuda_core(L, shape):
    """Tensor-core vs CUDA-core engines on the same device codes: int8 bitwise,
    f32 within rtol/atol 1e-5 (configs[1] and configs[4] geometries)."""
    import torch

    n, c, k, v, m = shape
    g = torch.Generator(device="cuda").manual_seed(n + m)
    a = torch.randn((n, c * v), generator=g, device="cuda")
    books = torch.randn((c, k, v), generator=g, device="cuda")
    w = torch.randn((c * v, m), generator=g, device="cuda") / np.sqrt(c * v)
    bias = torch.randn(m, generator=g, device="cuda") * 0.1
    lt = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias, qat=True, gather="tensor")
    lc = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias, qat=True, gather="cuda")
    assert lt.uses_tensor_cores(True)
    assert torch.equal(L.lut_layer_infer(a, lt, integer=True), L.lut_layer_infer(a, lc, integer=True))
    ft = L.lut_layer_infer(a, lt, integer=False)
    fc = L.lut_layer_infer(a, lc, integer=False)
    torch.testing.assert_close(ft, fc, rtol=1e-5, atol=1e-5)


def test_hash_encoder(L, golden):
    """encode_hash (hashing.py:171-196) on the GPU == reference codes; the hash
    encoder swaps only the indices (test_kernels.py:201-213)."""
    a, trees = G.hash_inputs(golden)
    np.testing.assert_array_equal(L.encode_hash(a, trees), golden.arrays["hash_codes"])
    case = golden.cases("hash")
    rng = O.make_rng(91)
    w = rng.standard_normal((case["c"] * case["v"], 6)).astype(F32)
    books = rng.standard_normal((case["c"], case["k"], case["v"])).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=case["v"], k=case["k"]), books=books, weight=w, bias=np.zeros(6, F32),
                       trees=trees)
    got = L.lut_layer_infer(a, layer, integer=False, encoder="hash")
    want = O.lut_matmul_ref(golden.arrays["hash_codes"], O.build_table(w, books))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n,m", [(3001, 4096), (1000, 640), (257, 200), (513, 132)])
def test_tc_plain_epilogue_bitwise(L, n, m):
    """The pair kernel's plain int8 epilogue (no bias / act, one scale: the
    configs[4] bench call) == the CUDA-core int8 gather, bitwise, on partial
    row tiles and on M not a multiple of the 128-column unit."""
    import torch

    from paper_2302_03213_b200._lib import load

    lib = load()
    c, k, v = 128, 16, 32
    g = torch.Generator(device="cuda").manual_seed(n * 7 + m)
    books = torch.randn((c, k, v), generator=g, device="cuda")
    w = torch.randn((c * v, m), generator=g, device="cuda") * 0.02
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, qat=True, gather="tensor")
    assert layer.uses_tensor_cores(True)
    a = torch.randn((n, c * v), generator=g, device="cuda")
    cstride = int(lib.lut_code_stride(c))
    codes = torch.empty((n, cstride), dtype=torch.uint8, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    assert lib.lut_encode_f32(a.data_ptr(), n, c * v, layer.books_prep.data_ptr(), c, k, v, codes.data_ptr(), 8,
                              cstride, None, sp) == 0
    scales = layer.qtable.scales_tensor("cuda")
    image = layer.onehot_image(True)
    out_tc = torch.full((n, m), float("nan"), device="cuda")
    out_cc = torch.empty((n, m), device="cuda")
    assert lib.lut_gather_onehot(codes.data_ptr(), cstride, n, c, k, m, 1, image.data_ptr(), scales.data_ptr(), 0,
                                 None, 0, out_tc.data_ptr(), None, 0, sp) == 0
    assert lib.lut_gather_i8(codes.data_ptr(), 8, n, c, k, m, layer.qtable.q.data_ptr(), scales.data_ptr(), 0, None,
                             0, out_cc.data_ptr(), None, 0, None, sp) == 0
    torch.cuda.synchronize()
    assert torch.equal(out_tc, out_cc)
    # fp32 tables through 4 digit planes (plain recombination epilogue) vs the bitwise f32 gather
    img_f = layer.onehot_image(False)
    out_tf = torch.full((n, m), float("nan"), device="cuda")
    out_cf = torch.empty((n, m), device="cuda")
    assert lib.lut_gather_onehot(codes.data_ptr(), cstride, n, c, k, m, 4, img_f.data_ptr(), None, 0,
                                 None, 0, out_tf.data_ptr(), None, 0, sp) == 0
    assert lib.lut_gather_f32(codes.data_ptr(), 8, n, c, k, m, layer.table.data_ptr(), None, 0,
                              out_cf.data_ptr(), 0, None, sp) == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(out_tf, out_cf, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("k", [16, 64])
def test_tc_screen_encode_exact(L, k):
    """configs[1,3,4] encode shapes (V=32, K=16 / 64) through the tensor-core
    screening kernel: exact centroid hits, duplicated centroids (tie -> lowest k),
    scaled near-duplicates and midpoints, plus random rows == encode_hard (oracle)."""
    rng = O.make_rng(2024 + k)
    c, v, n = 8, 32, 1000
    books = rng.standard_normal((c, k, v)).astype(F32)
    books[0, 9] = books[0, 3]                      # exact duplicate: lowest index wins
    books[1, 15] = books[1, 0]
    books[2, 7] = books[2, 6] * np.float32(1 + 2 ** -20)  # near duplicate
    books[3] *= np.float32(1e3)                    # large magnitudes
    books[4] *= np.float32(1e-3)                   # small magnitudes
    a = rng.standard_normal((n, c * v)).astype(F32)
    a[:, 3 * v:4 * v] *= np.float32(1e3)
    a[:, 4 * v:5 * v] *= np.float32(1e-3)
    for i in range(64):                            # exact hits and midpoints
        cb = i % c
        a[i, cb * v:(cb + 1) * v] = books[cb, i % k]
        a[64 + i, cb * v:(cb + 1) * v] = (books[cb, i % k] + books[cb, (i + 5) % k]) * np.float32(0.5)
    a[200:260, 0:v] = books[0, 3]                  # duplicated centroid hit
    a[260:320, v:2 * v] = books[1, 0]
    codes, ties = L.centroid_search_fast(a, books, return_near_ties=True)
    np.testing.assert_array_equal(codes, O.encode_hard(a, books))
    assert (codes[200:260, 0] == 3).all() and (codes[260:320, 1] == 0).all()
    assert ties >= 120  # the duplicated-centroid hits are exact ties -> f64 re-decision


def test_tc_screen_encode_random_shapes(L):
    """Tensor-core screening encode on random row counts / codebook counts (partial
    128-row tiles, partial 16-codebook groups, K in {16, 64}) and value scales,
    through both the numpy and the torch entry points == encode_hard."""
    import torch

    rng = O.make_rng(777)
    for trial in range(12):
        k = (16, 64)[trial % 2]
        n = int(rng.integers(128, 2500))
        c = int(rng.integers(1, 40))
        scale = np.float32(10.0 ** rng.integers(-2, 3))
        books = (rng.standard_normal((c, k, 32)) * scale).astype(F32)
        a = (rng.standard_normal((n, c * 32)) * scale).astype(F32)
        if trial % 3 == 0:  # rows sitting exactly on centroids
            idx = rng.integers(0, k, size=(n, c))
            a = books[np.arange(c)[None, :], idx].reshape(n, c * 32).copy()
        want = O.encode_hard(a, books)
        np.testing.assert_array_equal(L.centroid_search_fast(a, books), want, err_msg=f"trial {trial}")
        got_t = L.centroid_search_fast(torch.from_numpy(a).cuda(), torch.from_numpy(books).cuda())
        np.testing.assert_array_equal(got_t.cpu().numpy(), want, err_msg=f"trial {trial} (torch)")


@pytest.mark.parametrize("c,k,m", [(128, 16, 4096), (130, 16, 257), (64, 16, 130), (33, 64, 96), (17, 64, 200),
                                   (72, 16, 1000)])
def test_layer_configs4_family_vs_oracle(L, c, k, m):
    """configs[4]-family layers (V = 32) through lut_layer_infer on both table
    types, no bias (the plain epilogues): int8 output bytes-equal to the oracle's
    lut_layer_infer, fp32 tensor-core output within rtol/atol 1e-5 of it."""
    rng = O.make_rng(c * 1000 + k + m)
    n, v = 700, 32
    a = rng.standard_normal((n, c * v)).astype(F32)
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) / np.sqrt(c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, qat=True, gather="tensor")
    table = O.build_table(w, books)
    q, s = O.quantize_table(table)
    got8 = L.lut_layer_infer(a, layer, integer=True)
    assert got8.tobytes() == O.lut_layer_infer(a, books, q=q, scale=s).tobytes()
    gotf = L.lut_layer_infer(a, layer, integer=False)
    np.testing.assert_allclose(gotf, O.lut_layer_infer(a, books, table=table, integer=False), rtol=1e-5, atol=1e-5)


def test_conv_int8_tensor_nchw(L):
    """A 3x3 LUT conv with int8 tables through the tensor-core gather writing NCHW
    directly (out_hw > 0) == the oracle on the im2col matrix, bitwise."""
    import torch

    rng = O.make_rng(404)
    bsz, cin, hh, ww, cout = 3, 16, 10, 12, 48
    x = np.abs(rng.standard_normal((bsz, cin, hh, ww))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    wconv = (rng.standard_normal((cin * 9, cout)) * 0.1).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=books, weight=wconv, qat=True, gather="tensor")
    conv = L.LutConv(cin, 3, 1, 1, layer)
    y, _ = conv.forward(x, integer=True)
    cols = O.im2col(x, 3, 3, 1, 1)
    table = O.build_table(wconv, books)
    q, s = O.quantize_table(table)
    want = O.lut_layer_infer(cols, books, q=q, scale=s).reshape(bsz, hh, ww, cout).transpose(0, 3, 1, 2)
    got = y.cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
    assert got.tobytes() == np.ascontiguousarray(want).tobytes()


@pytest.mark.parametrize("m,mtile", [(3072, 0), (3072, 128), (768, 32), (200, 64), (1000, 40)])
@pytest.mark.parametrize("act", [None, "relu", "gelu"])
def test_tc_stack_epilogue_bitwise(L, m, mtile, act):
    """The pair kernel's compile-time caller-stack epilogue (int8 tables + bias,
    ReLU / GELU, per-m-tile scales: configs[1]/[3] layers) against the CUDA-core
    gather on the same device codes: bitwise (same fmul_rn, fadd_rn, activation
    per element). mtile 40 is not a multiple of 32 and takes the generic epilogue."""
    import torch

    n, c, k, v = 2000, 24, 16, 32
    g = torch.Generator(device="cuda").manual_seed(m + mtile)
    a = torch.randn((n, c * v), generator=g, device="cuda")
    books = torch.randn((c, k, v), generator=g, device="cuda")
    w = torch.randn((c * v, m), generator=g, device="cuda") * 0.02
    bias = torch.randn(m, generator=g, device="cuda") * 0.1
    kw = dict(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias, qat=True, act=act, scale_mtile=mtile)
    lt = L.LutLayer(gather="tensor", **kw)
    lc = L.LutLayer(gather="cuda", **kw)
    assert lt.uses_tensor_cores(True)
    got = L.lut_layer_infer(a, lt, integer=True)
    assert torch.equal(got, L.lut_layer_infer(a, lc, integer=True))
    if act is None and mtile == 0:  # and against the oracle restatement
        an, bn = a.cpu().numpy(), books.cpu().numpy()
        table = O.build_table(w.cpu().numpy(), bn)
        q, s = O.quantize_table(table)
        want = O.lut_layer_infer(an, bn, q=q, scale=s, bias=bias.cpu().numpy())
        assert got.cpu().numpy().tobytes() == want.tobytes()
