"""`.lutn` parsing / writing on the host (no GPU): the reference's own
container tests (tests/test_container.py:29-116) replayed against bytes the
reference wrote (tests/golden/make_golden.py `lutn_*`)."""

import struct

import numpy as np
import pytest

from paper_2302_03213_b200.container import DenseRecord, LutRecord, parse_records, records_bytes
from paper_2302_03213_b200.errors import ContainerError


@pytest.fixture(params=["a", "b"])
def raw(request, golden):
    return golden.arrays[f"lutn_{request.param}_bytes"].tobytes()


def test_round_trip_byte_identical(raw):
    assert records_bytes(parse_records(raw)) == raw


def test_header(raw):
    assert raw[:4] == b"LUTN" and int.from_bytes(raw[4:8], "little") == 1


def test_model_a_structure(golden):
    recs = parse_records(golden.arrays["lutn_a_bytes"].tobytes())
    kinds = [(type(r).__name__, act) for r, act in recs]
    assert kinds == [("LutRecord", 1), ("LutRecord", 1), ("DenseRecord", 0)]
    l1, l2 = recs[0][0], recs[1][0]
    assert l1.books.shape == (4, 8, 4) and l1.table.shape == (4, 8, 12) and l1.q is None
    assert l2.q.shape == (3, 16, 7) and l2.q.dtype == np.int8 and l2.scale > 0 and l2.table is None
    assert [len(t[0]) for t in l1.trees] == [3] * 4 and [len(t[0]) for t in l2.trees] == [4] * 3
    assert all(t[2].shape == (16,) for t in l2.trees)


def test_model_b_conv_geometry(golden):
    recs = parse_records(golden.arrays["lutn_b_bytes"].tobytes())
    assert [r.conv for r, _ in recs] == [(3, 1, 1), (3, 2, 1), None]
    assert isinstance(recs[0][0], LutRecord) and isinstance(recs[1][0], DenseRecord)
    assert recs[1][0].weight.shape == (8 * 9, 4)


def test_bad_magic():
    with pytest.raises(ContainerError):
        parse_records(b"XXXX" + b"\x00" * 16)


def test_bad_version(raw):
    bad = bytearray(raw)
    bad[4] = 99
    with pytest.raises(ContainerError):
        parse_records(bytes(bad))


def test_unknown_record_kind(raw):
    bad = bytearray(raw)
    bad[12] = 77
    with pytest.raises(ContainerError):
        parse_records(bytes(bad))


def test_unknown_geometry_and_activation(raw):
    for off, val in ((14, 5), (13, 3)):
        bad = bytearray(raw)
        bad[off] = val
        with pytest.raises(ContainerError):
            parse_records(bytes(bad))


def test_truncation(raw):
    for cut in (3, 1, len(raw) // 2, len(raw) - 9):
        with pytest.raises(ContainerError):
            parse_records(raw[: len(raw) - cut])


def test_trailing_garbage(raw):
    with pytest.raises(ContainerError):
        parse_records(raw + b"\x00")


def test_unknown_table_tag(golden):
    raw = golden.arrays["lutn_a_bytes"].tobytes()
    # first record: 3 head bytes, then u32 D,M,K,V + f32 t, centroids (4*8*4 f32), then the tag
    off = 12 + 3 + 20 + 4 * 8 * 4 * 4
    assert raw[off] == 1
    bad = bytearray(raw)
    bad[off] = 9
    with pytest.raises(ContainerError):
        parse_records(bytes(bad))


def test_corrupt_dv():
    rec = struct.pack("<BBB", 2, 0, 0) + struct.pack("<IIIIf", 10, 4, 8, 3, 1.0)
    with pytest.raises(ContainerError):
        parse_records(b"LUTN" + struct.pack("<II", 1, 1) + rec)


def test_empty_model():
    raw = b"LUTN" + struct.pack("<II", 1, 0)
    assert parse_records(raw) == [] and records_bytes([]) == raw
