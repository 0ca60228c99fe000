"""GPU: hand-worked known answers for the pq layer of the path (the categories of
the reference's tests/test_pq.py:67-141 — exact centroid hits, worked distances,
the tie rule, brute-force optimality, build_table / lut_matmul_ref by hand and
their shape / range errors), with this repo's own numbers, plus empty inputs.
Everything goes through the drop-in names (numpy in -> numpy out)."""

import numpy as np
import pytest

from oracle import lut_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def L():
    import paper_2302_03213_b200 as lg

    return lg


def test_rows_built_from_centroids_encode_to_them(L):
    rng = O.make_rng(77)
    books = rng.standard_normal((3, 6, 4)).astype(F32)
    picks = [(5, 0, 2), (1, 1, 1), (4, 3, 0)]
    a = np.stack([np.concatenate([books[c, k] for c, k in enumerate(p)]) for p in picks])
    for fn in (L.encode_hard, L.centroid_search_fast):
        enc = fn(a, books)
        assert enc.dtype == np.uint8 and enc.shape == (3, 3)
        np.testing.assert_array_equal(enc, picks)


def test_worked_distances(L):
    # one codebook, V = 2: |(3, 1) - (2, 2)|^2 = 2 beats 10 (origin) and 5 ((4, 3))
    books = np.array([[[0.0, 0.0], [2.0, 2.0], [4.0, 3.0]]], F32)
    assert L.encode_hard(np.array([[3.0, 1.0]], F32), books)[0, 0] == 1
    # V = 1, two codebooks: 0.4 -> {-1, 0.5, 3} picks 0.5; -7 -> {-6.5, -8} picks -6.5 (0.25 < 1)
    books = np.array([[[-1.0], [0.5], [3.0]], [[-6.5], [-8.0], [100.0]]], F32)
    np.testing.assert_array_equal(L.centroid_search_fast(np.array([[0.4, -7.0]], F32), books), [[1, 0]])


def test_ties_go_to_the_lowest_index(L):
    # 5 is equidistant from 3 and 7; the duplicate 7s tie exactly on an exact hit
    books = np.array([[[9.0], [3.0], [7.0], [7.0]]], F32)
    for fn in (L.encode_hard, L.centroid_search_fast):
        assert fn(np.array([[5.0]], F32), books)[0, 0] == 1
        assert fn(np.array([[7.0]], F32), books)[0, 0] == 2


@pytest.mark.parametrize("seed", range(6))
def test_index_is_a_brute_force_minimum(L, seed):
    rng = O.make_rng(900 + seed)
    n, c, k, v = 11, 4, 9, 3
    a = rng.standard_normal((n, c * v)).astype(F32)
    books = rng.standard_normal((c, k, v)).astype(F32)
    enc = L.centroid_search_fast(a, books)
    for i in range(n):
        for j in range(c):
            sub = a[i, j * v:(j + 1) * v].astype(np.float64)
            d = [float(((sub - p.astype(np.float64)) ** 2).sum()) for p in books[j]]
            assert enc[i, j] == int(np.argmin(d))  # literal f64 distances, first minimum


def test_encode_shape_errors(L):
    books = np.zeros((3, 4, 5), F32)
    with pytest.raises(L.ShapeError):
        L.encode_hard(np.zeros((2, 14), F32), books)
    with pytest.raises(L.ShapeError):
        L.centroid_search_fast(np.zeros((2, 16), F32), books)


def test_build_table_by_hand(L):
    # V = 1: the table is the outer product of centroid scalars and the weight row
    books = np.array([[[1.5], [-2.0]]], F32)
    w = np.array([[4.0, -0.5, 8.0]], F32)
    np.testing.assert_array_equal(L.build_table(w, books)[0], [[6.0, -0.75, 12.0], [-8.0, 1.0, -16.0]])
    # unit centroids select weight rows: codebook 1 owns rows 2..3 of W
    books = np.array([[[1.0, 0.0], [0.0, 1.0]], [[0.0, 1.0], [1.0, 1.0]]], F32)
    w = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0], [7.0, 8.0]], F32)
    t = L.build_table(w, books)
    np.testing.assert_array_equal(t[0], [[1.0, 2.0], [3.0, 4.0]])
    np.testing.assert_array_equal(t[1], [[7.0, 8.0], [12.0, 14.0]])
    # zero weights -> zero table of the right shape
    rng = O.make_rng(2)
    t0 = L.build_table(np.zeros((8, 5), F32), rng.standard_normal((2, 3, 4)).astype(F32))
    assert t0.shape == (2, 3, 5) and not t0.any()


def test_lut_matmul_ref_by_hand(L):
    rng = O.make_rng(31)
    table = rng.standard_normal((1, 5, 6)).astype(F32)
    np.testing.assert_array_equal(L.lut_matmul_ref(np.array([[3]], np.uint8), table), table[0, 3][None, :])
    # two codebooks: the row is an f32 sum of the two selected table rows, c ascending from +0
    table = np.array([[[1.0, 10.0], [2.0, 20.0]], [[0.25, -10.0], [0.5, 5.0]]], F32)
    out = L.lut_matmul_ref(np.array([[1, 0], [0, 1]], np.uint8), table)
    np.testing.assert_array_equal(out, [[2.25, 10.0], [1.5, 15.0]])
    assert not L.lut_matmul_ref(np.zeros((4, 3), np.uint8), np.zeros((3, 2, 7), F32)).any()
    with pytest.raises(L.CorruptionError):
        L.lut_matmul_ref(np.array([[5]], np.uint8), np.zeros((1, 5, 2), F32))


def test_empty_inputs(L):
    rng = O.make_rng(8)
    books = rng.standard_normal((4, 16, 8)).astype(F32)
    w = rng.standard_normal((32, 12)).astype(F32)
    table = L.build_table(w, books)
    qt = L.quantize_table(table)
    a0 = np.zeros((0, 32), F32)
    enc0 = L.centroid_search_fast(a0, books)
    assert enc0.shape == (0, 4) and enc0.dtype == np.uint8
    assert L.encode_hard(a0, books).shape == (0, 4)
    assert L.lut_gather_f32(enc0, table).shape == (0, 12)
    out_i = L.lut_gather_i32(enc0, qt.q)
    assert out_i.shape == (0, 12) and out_i.dtype == np.int32
    assert L.lut_gather_accumulate(enc0, qt).shape == (0, 12)
    layer = L.LutLayer(cfg=L.PqConfig(v=8, k=16), books=books, weight=w, qat=True)
    for integer in (False, True):
        out = L.lut_layer_infer(a0, layer, integer=integer)
        assert out.shape == (0, 12) and out.dtype == F32
