"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side validation raises the reference's exception
classes before any device work; row-sharding host logic (gloo, 2 ranks)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F32 = np.float32


def header_symbols():
    with open(os.path.join(ROOT, "include", "lutgpu.h")) as f:
        return sorted(set(re.findall(r"LUT_API\s+[\w\s\*]+?\b(lut_\w+)\s*\(", f.read())))


def test_library_exports_every_header_symbol():
    from paper_2302_03213_b200 import _lib

    declared = header_symbols()
    assert len(declared) >= 17
    import ctypes

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"
    h = _lib.load()
    assert h.lut_version() == 100
    # record: centroids, norms, max norm (padded to 4 floats); V=32, K=16 adds the
    # swizzled tf32 operand tile and the rounded-up |p_k| of the screening encode
    assert h.lut_books_prep_bytes(128, 16, 32) == 128 * ((16 * 32 + 16 + 1 + 3) // 4 * 4 + 16 * 32 + 16) * 4
    assert h.lut_books_prep_bytes(48, 16, 16) == 48 * ((16 * 16 + 16 + 1 + 3) // 4 * 4) * 4


def test_abi_rejects_bad_geometry_without_gpu():
    """Shape/option errors are host-side: no device is touched."""
    from paper_2302_03213_b200 import _lib

    h = _lib.load()
    assert h.lut_encode_f32(None, 10, 7, None, 2, 16, 4, None, 8, 0, None, None) == 2  # d != C*V
    assert h.lut_encode_f32(None, 10, 8, None, 2, 300, 4, None, 8, 0, None, None) == 2  # K > 256
    assert h.lut_encode_f32(None, 10, 8, None, 2, 32, 4, None, 4, 0, None, None) == 2  # u4 with K > 16
    assert b"4-bit" in h.lut_last_error()
    assert h.lut_gather_f32(None, 8, 5, 2, 16, 4, None, None, 9, None, 0, None, None) == 2  # bad act
    assert h.lut_gather_i8(None, 8, 5, 2, 16, 4, None, None, -1, None, 0, None, None, 0, None, None) == 2
    assert h.lut_im2col_f32(None, 1, 1, 2, 2, 3, 3, 1, 0, None, None) == 2  # kernel does not fit
    assert h.lut_pipeline_create(0, 0, 4, 4, 1, None) == 2


def test_python_validation_matches_reference_exceptions():
    import paper_2302_03213_b200 as L

    with pytest.raises(L.ConfigError):
        L.KernelPlan(group_size=259)
    with pytest.raises(L.ConfigError):
        L.KernelPlan(group_size=0)
    L.KernelPlan(group_size=258)
    assert L.MAX_GROUP == 258
    with pytest.raises(L.ShapeError):
        L.centroid_search_fast(np.zeros((1, 5), F32), np.zeros((2, 4, 3), F32))
    with pytest.raises(L.ShapeError):
        L.centroid_search_fast(np.zeros((5,), F32), np.zeros((2, 4, 3), F32))
    with pytest.raises(L.ConfigError):
        L.centroid_search_fast(np.zeros((1, 6), F32), np.zeros((2, 300, 3), F32))
    with pytest.raises(L.ShapeError):
        L.lut_gather_i32(np.zeros((2, 3), np.uint8), np.zeros((3, 4, 2), np.int16))
    with pytest.raises(L.ShapeError):
        L.lut_gather_i32(np.zeros((2, 2), np.uint8), np.zeros((3, 4, 2), np.int8))
    with pytest.raises(L.ShapeError):
        L.lut_gather_f32(np.zeros((2,), np.uint8), np.zeros((3, 4, 2), F32))
    with pytest.raises(L.ConfigError):
        L.PqConfig(v=0, k=4)
    with pytest.raises(L.ConfigError):
        L.PqConfig(v=2, k=257)
    with pytest.raises(L.ShapeError):
        L.build_table(np.zeros((5, 2), F32), np.zeros((2, 4, 3), F32))
    with pytest.raises(L.ShapeError):
        L.im2col(np.zeros((1, 1, 2, 2), F32), 3, 3)
    with pytest.raises(L.ConfigError):
        L.im2col(np.zeros((1, 1, 4, 4), F32), 2, 2, stride=0)
    with pytest.raises(L.ShapeError):
        L.LookupTableI8(q=np.zeros((2, 2), np.int8), scale=np.float32(1.0))
    with pytest.raises(L.DataError):
        L.LookupTableI8(q=np.zeros((1, 2, 2), np.int8), scale=np.float32(0.0))
    with pytest.raises(L.DataError):
        L.LookupTableI8(q=np.full((1, 2, 2), -128, np.int8), scale=np.float32(1.0))


def test_compute_without_gpu_fails_loudly():
    import torch

    import paper_2302_03213_b200 as L

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.DeviceError):
        L.centroid_search_fast(np.zeros((2, 6), F32), np.zeros((2, 4, 3), F32))


def test_flop_counter():
    import paper_2302_03213_b200 as L

    c = L.flop_counter(100, 64, 128, 16, 8)
    assert (c["encode"], c["lookup_aggregate"], c["dense"]) == (102400, 102400, 819200)
    assert L.flop_counter(10**4, 768, 96, 16, 32)["encode"] == 122_880_000
    with pytest.raises(L.ConfigError):
        L.flop_counter(1, 10, 4, 4, 3)


def test_shard_range_partitions_rows():
    from paper_2302_03213_b200.dist import shard_range, shard_sizes

    for n in (0, 1, 7, 1024, 2**20 + 3):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(shard_sizes(n, world)) - min(shard_sizes(n, world)) <= 1


def _gloo_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    from paper_2302_03213_b200.dist import gather_rows, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        full = torch.arange(n * 3, dtype=torch.float32).reshape(n, 3)
        s, e = shard_range(n, rank, world)
        # each rank "computes" its rows (an elementwise stand-in for the layer)
        local = full[s:e] * 2 + 1
        got = gather_rows(local, n)
        q.put((rank, bool(torch.equal(got, full * 2 + 1))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 7, 1])
def test_gather_rows_gloo_world2(n):
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


class _HostLayer:
    """Stand-in with LutLayer.forward_device's contract for the CPU test: a
    row-wise map (out row i depends only on input row i), as the LUT layer is."""

    def forward_device(self, a, integer):
        import torch

        w = torch.arange(a.shape[1] * 5, dtype=torch.float32).reshape(a.shape[1], 5) / 7.0
        return a @ w + (1.0 if integer else 0.0)


def _sharded_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    from paper_2302_03213_b200.dist import shard_range, sharded_forward

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        full = torch.linspace(-3, 3, n * 4, dtype=torch.float32).reshape(n, 4)
        s, e = shard_range(n, rank, world)
        layer = _HostLayer()
        got = sharded_forward(full[s:e], layer, True, n_total=None, gather=True)  # n_total via all_reduce
        local = sharded_forward(full[s:e], layer, False)
        q.put((rank, bool(torch.equal(got, layer.forward_device(full, True))) and local.shape[0] == e - s))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [9, 2])
def test_sharded_forward_gloo_world2(n):
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


def test_bench_reference_arm_small():
    """bench.py --impl reference on a small layer: one JSON line with the
    reference-arm keys (all-core value, one-core figure, linearity check)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--dim", "256",
                        "--v", "16", "--cpu-rows", "64", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2 and line["warmup"] == 1
    assert line["one_core"]["cores"] == 1 and "linear" in line["linearity"]
    assert line["rows_sampled_per_step"] == line["cpu_baseline"]["cores"] * 64
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_rng_and_split_dropins():
    """make_rng / child_rng are the reference's Philox streams (rng.py:15-28);
    split_subvectors returns D/v views (tensor.py:128-135)."""
    import paper_2302_03213_b200 as L
    from oracle import lut_oracle as O

    assert np.array_equal(L.make_rng(42).integers(0, 2**63, 16), O.make_rng(42).integers(0, 2**63, 16))
    assert np.array_equal(L.child_rng(7, 3).standard_normal(5), O.child_rng(7, 3).standard_normal(5))
    assert not np.array_equal(L.child_rng(7, 0).standard_normal(5), L.make_rng(7).standard_normal(5))
    with pytest.raises(ValueError):
        L.child_rng(1, -1)
    a = np.arange(24, dtype=F32).reshape(2, 12)
    parts = L.split_subvectors(a, 4)
    assert len(parts) == 3 and all(p.shape == (2, 4) for p in parts)
    assert np.array_equal(np.concatenate(parts, axis=1), a)
    with pytest.raises(L.ConfigError):
        L.split_subvectors(a, 5)
    with pytest.raises(L.ConfigError):
        L.split_subvectors(a, 0)
