"""GPU: guard bands around every output buffer of the C ABI's kernels.

compute-sanitizer is closed on this pool (profiles/r02/compute_sanitizer_closed.log), so
out-of-bounds WRITES are checked here instead: codes, float and int32 outputs live in the
middle of larger allocations filled with a sentinel, ragged shapes drive every engine
through its partial tiles (rows not a multiple of 128 / 256 / 512, M not a multiple of the
column tile, C not a multiple of 16), and the bands must come back untouched while the
payload equals the oracle's bytes (kernels.py:62-178)."""

import ctypes as C

import numpy as np
import pytest

from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32
PAD = 64  # guard rows on each side
SENT_F = 12345.5
SENT_B = 0xA5


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


def _banded(torch, rows, cols, dtype, fill):
    big = torch.full((rows + 2 * PAD, cols), fill, dtype=dtype, device="cuda")
    return big, big[PAD:PAD + rows]


def _bands_intact(torch, big, rows, fill):
    return bool((big[:PAD] == fill).all()) and bool((big[PAD + rows:] == fill).all())


SHAPES = [  # n, c, k, v, m: every encode / gather engine, ragged everywhere
    (1000, 128, 16, 32, 4096),   # screening encode + resident pair gather (plain epilogue)
    (777, 128, 64, 32, 516),     # K = 64 screen + streamed gather, M % 128 != 0
    (513, 24, 16, 32, 3072),     # small C*K pair gather
    (300, 7, 16, 16, 100),       # TMA FFMA2 encode, C % 16 != 0
    (129, 5, 8, 9, 34),          # generic row encode, tiny M
    (2050, 96, 16, 32, 770),     # M % 4 != 0: direct-store epilogues
]


@pytest.mark.parametrize("n,c,k,v,m", SHAPES)
@pytest.mark.parametrize("gather", ["tensor", "cuda"])
def test_layer_outputs_stay_in_bounds(L, n, c, k, v, m, gather):
    import torch

    rng = O.make_rng(n + 7 * c + m)
    books = rng.standard_normal((c, k, v)).astype(F32)
    w = (rng.standard_normal((c * v, m)) * 0.05).astype(F32)
    a = rng.standard_normal((n, c * v)).astype(F32)
    layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=books, weight=w, qat=True, gather=gather)
    a_dev = torch.from_numpy(a).cuda()
    table = O.build_table(w, books)
    q, s = O.quantize_table(table)
    idx = np.r_[0:min(n, 40), max(0, n - 40):n]
    for integer in (True, False):
        big_o, out = _banded(torch, n, m, torch.float32, SENT_F)
        big_c, codes = _banded(torch, n, layer.code_stride, torch.uint8, SENT_B)
        layer.forward_device(a_dev, integer, out=out, codes=codes)
        torch.cuda.synchronize()
        assert _bands_intact(torch, big_o, n, SENT_F), "output guard band overwritten"
        assert _bands_intact(torch, big_c, n, SENT_B), "code guard band overwritten"
        # row padding bytes of the code rows (stride > C) may be written; the rows' payload is exact
        np.testing.assert_array_equal(codes[:, :c].cpu().numpy()[idx], O.encode_hard(a[idx], books))
        got = out.cpu().numpy()[idx]
        if integer:
            assert got.tobytes() == O.lut_layer_infer(a[idx], books, q=q, scale=s).tobytes()
        elif gather == "cuda":
            assert got.tobytes() == O.lut_layer_infer(a[idx], books, table=table, integer=False).tobytes()
        else:
            np.testing.assert_allclose(got, O.lut_layer_infer(a[idx], books, table=table, integer=False),
                                       rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("b,cin,hw,stride,pad", [(5, 16, 32, 1, 1), (7, 13, 6, 1, 1), (3, 16, 16, 2, 1), (9, 40, 8, 1, 0)])
def test_conv_layer_outputs_stay_in_bounds(L, b, cin, hw, stride, pad):
    """lut_conv_layer_forward (fused-im2col encode + NCHW lookup): strip, tensor-core and
    generic conv encodes, f32 and int8 tables."""
    import torch

    lib = L._lib.load()
    rng = O.make_rng(b * 31 + cin + hw)
    x = np.abs(rng.standard_normal((b, cin, hw, hw))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    cout = cin
    w = (rng.standard_normal((cin * 9, cout)) * 0.1).astype(F32)
    ho = (hw + 2 * pad - 3) // stride + 1
    n = b * ho * ho
    lut = L.LutLayer(cfg=L.PqConfig(v=9, k=16), books=books, weight=w, qat=True)
    x_dev = torch.from_numpy(x).cuda()
    cols = O.im2col(x, 3, 3, stride, pad)
    table = O.build_table(w, books)
    q, s = O.quantize_table(table)
    for integer in (False, True):
        big_o, out = _banded(torch, 1, b * cout * ho * ho, torch.float32, SENT_F)
        big_c, codes = _banded(torch, n, lut.code_stride, torch.uint8, SENT_B)
        desc = lut.desc(integer)
        L._lib.check(lib.lut_conv_layer_forward(C.byref(desc), x_dev.data_ptr(), b, cin, hw, hw, 3, 3, stride, pad,
                                                out.data_ptr(), codes.data_ptr(), None,
                                                torch.cuda.current_stream().cuda_stream), "conv layer")
        torch.cuda.synchronize()
        assert _bands_intact(torch, big_o, 1, SENT_F) and _bands_intact(torch, big_c, n, SENT_B)
        np.testing.assert_array_equal(codes[:, :cin].cpu().numpy(), O.encode_hard(cols, books))
        want = (O.lut_layer_infer(cols, books, q=q, scale=s) if integer
                else O.lut_layer_infer(cols, books, table=table, integer=False))
        want = want.reshape(b, ho, ho, cout).transpose(0, 3, 1, 2)
        assert out.cpu().numpy().reshape(b, cout, ho, ho).tobytes() == np.ascontiguousarray(want).tobytes()


def test_int32_gather_stays_in_bounds(L):
    """lut_gather_onehot with an int32 output (lut_gather_i32 on the tensor cores: the
    generic epilogue's scalar stores), M odd."""
    import torch

    rng = O.make_rng(515)
    n, c, k, m = 700, 64, 16, 203
    q = rng.integers(-127, 128, size=(c, k, m)).astype(np.int8)
    enc = rng.integers(0, k, size=(n, c)).astype(np.uint8)
    want = O.lut_gather_i32(enc, q)
    lib = L._lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    stride = int(lib.lut_code_stride(c))
    codes = torch.zeros((n, stride), dtype=torch.uint8, device="cuda")
    codes[:, :c] = torch.from_numpy(enc).cuda()
    q_dev = torch.from_numpy(q).cuda()
    img = torch.empty(lib.lut_onehot_image_bytes(c, k, m, 1), dtype=torch.uint8, device="cuda")
    L._lib.check(lib.lut_onehot_prepare_i8(q_dev.data_ptr(), c, k, m, img.data_ptr(), sp), "prepare")
    big_o, out = _banded(torch, n, m, torch.int32, 0x5A5A5A5A)
    L._lib.check(lib.lut_gather_onehot(codes.data_ptr(), stride, n, c, k, m, 1, img.data_ptr(), None, 0, None, 0, None,
                                       out.data_ptr(), 0, sp), "gather_onehot")
    torch.cuda.synchronize()
    assert _bands_intact(torch, big_o, n, 0x5A5A5A5A)
    assert np.array_equal(out.cpu().numpy(), want)
