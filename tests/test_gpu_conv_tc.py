"""GPU: the 3x3 conv encodes == encode_hard on the im2col patches (pq.py:171-174,
tensor.py:36-79).  Stride-1 shapes with an even output width run the FP32-pipe
strip kernel (csrc/encode_conv_strip.cu); the others the tensor-core screen
(csrc/encode_conv_tc.cu, 3xTF32 + exact refinement) or the plane / generic row
kernels.  configs[2] geometries, partial units and channel groups, strides /
padding, crafted ties (duplicate centroids -> lowest k), exact centroid hits and
large / small magnitudes."""

import numpy as np
import pytest

from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


def _conv_codes(L, x, books, stride, pad):
    import torch

    lib = L._lib.load()
    b, cin, h, w = x.shape
    ho, wo = (h + 2 * pad - 3) // stride + 1, (w + 2 * pad - 3) // stride + 1
    xd = torch.from_numpy(x).cuda()
    bd = torch.from_numpy(books).cuda()
    prep = L.kernels.prepare_books(bd)
    codes = torch.empty((b * ho * wo, cin), dtype=torch.uint8, device="cuda")
    near = torch.zeros(1, dtype=torch.int32, device="cuda")
    L._lib.check(lib.lut_encode_conv_f32(xd.data_ptr(), b, cin, h, w, 3, 3, stride, pad, prep.data_ptr(), cin, 16, 9,
                                         codes.data_ptr(), 8, near.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return codes.cpu().numpy(), int(near.item())


@pytest.mark.parametrize("b,cin,hw,stride,pad", [(4, 16, 32, 1, 1), (6, 32, 16, 1, 1), (20, 64, 8, 1, 1),
                                                 (3, 24, 16, 1, 1), (5, 16, 16, 2, 1), (9, 40, 8, 1, 0),
                                                 # strip kernel: 2-pixel strips (Wo = 6), odd channel / image tails
                                                 (7, 13, 6, 1, 1), (21, 9, 8, 1, 1), (3, 8, 12, 1, 0), (2, 5, 18, 1, 1),
                                                 # odd output width / pad 2: generic kernels
                                                 (3, 8, 7, 1, 1), (2, 8, 8, 1, 2)])
def test_conv_tc_encode_random(L, b, cin, hw, stride, pad):
    rng = O.make_rng(b * cin + hw)
    x = np.abs(rng.standard_normal((b, cin, hw, hw))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    got, _ = _conv_codes(L, x, books, stride, pad)
    np.testing.assert_array_equal(got, O.encode_hard(O.im2col(x, 3, 3, stride, pad), books))


@pytest.mark.parametrize("stride", [1, 2])
def test_conv_tc_encode_crafted(L, stride):
    rng = O.make_rng(4242)
    b, cin, hw = 8, 32, 16
    x = np.abs(rng.standard_normal((b, cin, hw, hw))).astype(F32)
    books = np.abs(rng.standard_normal((cin, 16, 9))).astype(F32)
    books[0, 9] = books[0, 3]                            # duplicate: lowest index wins
    books[1, 15] = books[1, 0]
    books[2, 7] = books[2, 6] * np.float32(1 + 2 ** -20)  # near duplicate
    books[3] *= np.float32(1e3)
    x[:, 3] *= np.float32(1e3)
    books[4] *= np.float32(1e-3)
    x[:, 4] *= np.float32(1e-3)
    # exact hits: interior pixels whose 3x3 patch equals a centroid
    for i in range(40):
        bi, c, k = i % b, i % cin, i % 16
        y, xx = 1 + (i * 3) % (hw - 2), 1 + (i * 5) % (hw - 2)
        if stride == 2:  # patch centres of the stride-2 output grid (pad 1): even coordinates
            y, xx = max(2, y & ~1), max(2, xx & ~1)
        x[bi, c, y - 1:y + 2, xx - 1:xx + 2] = books[c, k].reshape(3, 3)
    # duplicated-centroid hits (exact ties)
    x[0, 0, 3:6, 3:6] = books[0, 3].reshape(3, 3)      # centre (4, 4)
    x[1, 1, 7:10, 7:10] = books[1, 0].reshape(3, 3)    # centre (8, 8)
    got, near = _conv_codes(L, x, books, stride, 1)
    want = O.encode_hard(O.im2col(x, 3, 3, stride, 1), books)
    np.testing.assert_array_equal(got, want)
    assert near >= 2  # the exact ties were re-decided in f64
