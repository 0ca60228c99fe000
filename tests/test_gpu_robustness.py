"""GPU: error behaviour and caching of the drop-in API (round-2 review items).

Each case mirrors a reference contract: a code >= K raises CorruptionError
(kernels.py:117-118, pq.py:209-210); the integer path without a quantized
table raises ConfigError (kernels.py:166-170); a layer converted from a
reference object follows in-place updates of its books / bias (train.py:162
updates parameters in place)."""

import types

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


def test_hash_leaf_out_of_range_raises(L, golden):
    """A corrupt hash tree (leaf >= K) raises, on both table kinds."""
    a, trees = G.hash_inputs(golden)
    case = golden.cases("hash")
    bad = [tuple(np.array(x, copy=True) for x in t) for t in trees]
    bad[0][2][:] = case["k"]  # every leaf of codebook 0 out of range
    rng = O.make_rng(5)
    w = rng.standard_normal((case["c"] * case["v"], 8)).astype(F32)
    books = rng.standard_normal((case["c"], case["k"], case["v"])).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=case["v"], k=case["k"]), books=books, weight=w, qat=True, trees=bad)
    for integer in (False, True):
        with pytest.raises(L.CorruptionError):
            L.lut_layer_infer(a, layer, integer=integer, encoder="hash")
    # the intact trees still work on the same layer object afterwards
    layer.trees = trees
    out = L.lut_layer_infer(a, layer, integer=False, encoder="hash")
    want = O.lut_matmul_ref(golden.arrays["hash_codes"], O.build_table(w, books))
    np.testing.assert_array_equal(out, want)


def test_conv_integer_without_qtable(L):
    rng = O.make_rng(3)
    books = rng.standard_normal((4, 16, 9)).astype(F32)
    w = rng.standard_normal((36, 8)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=books, weight=w)  # no qat -> no int8 table
    conv = L.LutConv(4, 3, 1, 1, layer)
    x = np.abs(rng.standard_normal((2, 4, 6, 6))).astype(F32)
    with pytest.raises(L.ConfigError):
        conv.forward(x, integer=True)


@pytest.mark.parametrize("gather", ["tensor", "cuda"])
def test_conv_int8_engines_bitwise(L, gather):
    """The int8 3x3 conv through each lookup engine (the tensor engine reads
    16-byte padded code rows and stores NCHW) == the oracle, bitwise."""
    rng = O.make_rng(44)
    cin, cout, b, h = 16, 32, 3, 10
    books = rng.standard_normal((cin, 16, 9)).astype(F32)
    wconv = (rng.standard_normal((cin * 9, cout)) * 0.1).astype(F32)
    x = np.abs(rng.standard_normal((b, cin, h, h))).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=books, weight=wconv, qat=True, gather=gather)
    assert layer.uses_tensor_cores(True) == (gather == "tensor")
    y, _ = L.LutConv(cin, 3, 1, 1, layer).forward(x, integer=True)
    cols = O.im2col(x, 3, 3, 1, 1)
    q, s = O.quantize_table(O.build_table(wconv, books))
    want = O.lut_layer_infer(cols, books, q=q, scale=s).reshape(b, h, h, cout).transpose(0, 3, 1, 2)
    np.testing.assert_array_equal(y, want)


def test_fresh_layer_large_numpy_int8(L):
    """First call of a fresh int8 tensor-core layer with a numpy input above the
    executor threshold: the B image is prepared on torch's stream before the
    executor's streams start (no half-built image)."""
    rng = O.make_rng(8)
    c, v, m = 16, 32, 2048
    n = (L.layer.PIPELINE_MIN_BYTES // (4 * c * v)) + 300
    books = rng.standard_normal((c, 16, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=16), books=books, weight=w, qat=True, gather="tensor")
    got = L.lut_layer_infer(a, layer, integer=True)  # first use of the layer
    q, s = O.quantize_table(O.build_table(w, books))
    idx = np.r_[0:256, n - 256:n]
    np.testing.assert_array_equal(got[idx], O.lut_layer_infer(a[idx], books, q=q, scale=s))


def test_foreign_layer_follows_in_place_updates(L):
    """A reference-style layer object is converted once; an in-place update of
    its books / bias (the reference SGD step) is picked up on the next call."""
    rng = O.make_rng(12)
    c, k, v, m = 6, 16, 4, 10
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = rng.standard_normal((c * v, m)).astype(F32)
    ref = types.SimpleNamespace(cfg=types.SimpleNamespace(v=v, k=k), books=books, bias=np.zeros(m, F32),
                                table=O.build_table(w, books), qtable=None, trees=None)
    a = rng.standard_normal((50, c * v)).astype(F32)
    first = L.lut_layer_infer(a, ref, integer=False)
    np.testing.assert_array_equal(first, O.lut_layer_infer(a, books, table=ref.table, bias=ref.bias, integer=False))
    assert L.layer.as_device_layer(ref) is L.layer.as_device_layer(ref)  # cached while unchanged
    ref.bias += 1.5          # in place, as train.py:162 does
    ref.books *= 0.5
    second = L.lut_layer_infer(a, ref, integer=False)
    np.testing.assert_array_equal(second, O.lut_layer_infer(a, ref.books, table=ref.table, bias=ref.bias,
                                                            integer=False))


def test_act_twin_has_own_pipelines(L):
    """with_act twins own their executor handles: dropping the parent's twins
    (rebuild) never frees a handle the parent still uses."""
    rng = O.make_rng(2)
    c, v, m = 8, 32, 256
    books = rng.standard_normal((c, 16, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=16), books=books, weight=w, qat=True)
    twin = layer.with_act("relu")
    assert twin._pipelines is not layer._pipelines


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2302_03213_b200 as L
    from paper_2302_03213_b200.dist import shard_range, sharded_forward

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rng = O.make_rng(77)
        n, c, v, m = 3001, 16, 32, 512
        books = rng.standard_normal((c, 16, v)).astype(F32)
        w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
        a = rng.standard_normal((n, c * v)).astype(F32)
        layer = L.LutLayer(cfg=L.PqConfig(v=v, k=16), books=books, weight=w, qat=True, bias=rng.standard_normal(m)
                           .astype(F32))
        s, e = shard_range(n, rank, world)
        a_dev = torch.from_numpy(a[s:e]).cuda()
        out = {}
        for integer in (True, False):
            full = sharded_forward(a_dev, layer, integer, n_total=n, gather=True)
            out[integer] = full.cpu().numpy()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_forward_two_ranks_bitwise(L):
    """Two ranks (processes) on cuda:0 each run their row shard through the real
    kernels (dist.sharded_forward); the gathered result equals one process
    running all rows, bitwise (rows are independent, kernels.py:78-86)."""
    import multiprocessing as mp
    import socket

    import torch

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
    rng = O.make_rng(77)
    n, c, v, m = 3001, 16, 32, 512
    books = rng.standard_normal((c, 16, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.02).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=16), books=books, weight=w, qat=True,
                       bias=rng.standard_normal(m).astype(F32))
    for integer in (True, False):
        single = layer.forward_device(torch.from_numpy(a).cuda(), integer).cpu().numpy()
        for r in (0, 1):
            assert res[r][integer].tobytes() == single.tobytes(), (r, integer)


@pytest.mark.parametrize("n,d,m", [(1, 1, 1), (70, 33, 65), (300, 256, 130), (64, 0, 8)])
def test_matmul_ref_bitwise(L, n, d, m):
    """The dense baseline (tensor.py:110-125) on the GPU: bitwise equal to the
    ascending-k f32 loop."""
    rng = O.make_rng(n + d + m)
    a = rng.standard_normal((n, d)).astype(F32)
    b = rng.standard_normal((d, m)).astype(F32)
    got = L.matmul_ref(a, b)
    assert got.dtype == np.float32 and got.tobytes() == O.matmul_ref(a, b).tobytes()


def test_bench_kernel_report(L):
    """bench_kernel / BenchReport (kernels.py:249-349): GPU-timed LUT path vs
    the dense matmul_ref, CSV row in the reference's column order."""
    rep = L.bench_kernel((512, 256, 128, 16, 16), repetitions=5)
    assert rep.lut_min_ns > 0 and rep.dense_median_ns > 0 and rep.gflops_equiv > 0
    assert rep.csv_row().count(",") == L.BenchReport.CSV_HEADER.count(",")
    with pytest.raises(L.ConfigError):
        L.bench_kernel((8, 10, 4, 4, 3))
    with pytest.raises(L.ConfigError):
        L.bench_kernel((8, 8, 4, 4, 2), repetitions=3)


@pytest.mark.parametrize("n,c,k,v,m", [(1024, 48, 16, 16, 768), (300, 7, 8, 4, 33), (5000, 24, 16, 32, 130),
                                       (1, 3, 16, 9, 5), (16384, 16, 16, 8, 64)])
def test_small_layer_bitwise(L, n, c, k, v, m):
    """Few-row fp32 layers (configs[0] and smaller / ragged shapes) through
    lut_layer_forward: bytes equal to the oracle's lut_layer_infer
    (kernels.py:143-178), bias and ReLU epilogue included."""
    import torch

    rng = O.make_rng(n + c)
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) / np.sqrt(c * v)).astype(F32)
    bias = rng.standard_normal(m).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, bias=bias)
    table = O.build_table(w, books)
    want = O.lut_layer_infer(a, books, table=table, bias=bias, integer=False)
    got = layer.forward_device(torch.from_numpy(a).cuda(), False).cpu().numpy()
    assert got.tobytes() == want.tobytes()
    relu = layer.with_act("relu").forward_device(torch.from_numpy(a).cuda(), False).cpu().numpy()
    assert relu.tobytes() == np.maximum(want, 0).astype(F32).tobytes()
