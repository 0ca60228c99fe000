"""Inference kernels — drop-in mirror of lutkit/kernels.py on the B200.

Same names, arguments, return dtypes and exceptions as the reference
(lutkit/kernels.py:39-193); every computation runs in the sm_100a kernels of
`csrc/` through the C ABI (include/lutgpu.h).  numpy in -> numpy out (the
reference contract); torch CUDA tensors in -> torch CUDA tensors out with no
host round trip.  There is no CPU fallback.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import LayerDesc, check, load
from .errors import ConfigError, CorruptionError, ShapeError
from .quant import QMAX, LookupTableI8

INT16_MAX = 32767
MAX_GROUP = INT16_MAX // QMAX  # 258 (kernels.py:34-36)
MAX_CENTROIDS = 256
F32 = np.float32
ACTS = {None: 0, "none": 0, "relu": 1, "gelu": 2}


@dataclass(frozen=True)
class KernelPlan:
    """Reference blocking parameters (kernels.py:39-59), validated identically.

    The GPU kernels choose their own tiles; `n_block`/`k_block` are accepted
    for API compatibility and `group_size` keeps its 1..258 contract (the GPU
    integer sum is exact for any grouping).  `code_bits` (extension) selects
    the device code format: 8 (u8, reference) or 4 (packed nibbles, K <= 16).
    """

    n_block: int = 64
    k_block: int = 8
    group_size: int = 128
    lane_hint: int = 16
    code_bits: int = 8

    def __post_init__(self) -> None:
        if self.n_block < 1 or self.k_block < 1:
            raise ConfigError("block sizes must be >= 1")
        if not 1 <= self.group_size <= MAX_GROUP:
            raise ConfigError(f"group_size must be in [1, {MAX_GROUP}] to keep INT16 partials exact")
        if self.code_bits not in (4, 8):
            raise ConfigError("code_bits must be 8 or 4")


class EncodeStats:
    """Near-tie count of the last encode on this thread."""

    last_near_ties = 0


# ------------------------------------------------------------- validation


def _matrix_shape(a, name="a"):
    shp = D.shape_of(a)
    if len(shp) != 2:
        raise ShapeError(f"{name} must be 2-D, got shape {shp}")
    return shp


def _books_shape(books):
    shp = D.shape_of(books)
    if len(shp) != 3:
        raise ShapeError(f"codebooks must have shape (C, K, V), got {shp}")
    if shp[1] > MAX_CENTROIDS:
        raise ConfigError(f"K={shp[1]} exceeds the u8 encoding limit {MAX_CENTROIDS}")
    if shp[1] < 1 or shp[2] < 1:
        raise ConfigError(f"codebooks need K >= 1 and V >= 1, got {shp}")
    return shp


def prepare_books(books_dev: torch.Tensor) -> torch.Tensor:
    """Device record of centroids + ||p||^2 + max ||p||^2 (lut_prepare_books)."""
    lib = load()
    c, k, v = books_dev.shape
    prep = torch.empty(max(1, lib.lut_books_prep_bytes(c, k, v)), dtype=torch.uint8, device=books_dev.device)
    check(lib.lut_prepare_books(D.ptr(books_dev), c, k, v, prep.data_ptr(), D.stream_ptr()), "prepare_books")
    return prep


def _check_enc_shape(enc, c_expected: int):
    shp = D.shape_of(enc)
    if len(shp) != 2:
        raise ShapeError(f"encoding must be (N, C), got {shp}")
    if shp[1] != c_expected:
        raise ShapeError(f"encoding C={shp[1]} != table C={c_expected}")


def _codes_device(enc, c_expected: int, k: int, dev):
    """Validate an encoding like kernels.py:109-118 and return device u8 codes."""
    _check_enc_shape(enc, c_expected)
    if isinstance(enc, torch.Tensor):
        t = enc.to(dev)
        if t.dtype != torch.uint8:
            if t.numel() and (int(t.min()) < 0 or int(t.max()) >= k):
                raise CorruptionError(f"encoding index {int(t.max())} >= K={k}")
            t = t.to(torch.uint8)
        return t.contiguous()
    arr = np.ascontiguousarray(enc)
    if arr.dtype != np.uint8:
        if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= k):
            raise CorruptionError(f"encoding index {int(arr.max())} >= K={k}")
        arr = arr.astype(np.uint8)
    return D.to_device(arr, np.uint8, dev)


# ------------------------------------------------------------------ encode


def encode_device(a_dev: torch.Tensor, prep: torch.Tensor, c: int, k: int, v: int, code_bits: int = 8,
                  near: torch.Tensor | None = None) -> torch.Tensor:
    """Device-to-device encode (lut_encode_f32)."""
    lib = load()
    n = a_dev.shape[0]
    width = c if code_bits == 8 else (c + 1) // 2
    codes = torch.empty((n, width), dtype=torch.uint8, device=a_dev.device)
    check(lib.lut_encode_f32(D.ptr(a_dev), n, c * v, D.ptr(prep), c, k, v, D.ptr(codes), code_bits, 0,
                             D.ptr(near), D.stream_ptr()), "centroid_search_fast")
    return codes


def centroid_search_fast(a, books, plan: KernelPlan = KernelPlan(), return_near_ties: bool = False):
    """Nearest-centroid indices, (N, C) uint8, identical to encode_hard
    (kernels.py:62-87; pq.py:171-174).  Near ties (fp32 gap inside the error
    bound) are re-decided in fp64; their count is returned on request."""
    n, d = _matrix_shape(a, "a")
    c, k, v = _books_shape(books)
    if d != c * v:
        raise ShapeError(f"input cols {d} != C*V = {c}*{v}")
    kind = D.kind_of(a)
    dev = D.require_cuda()
    a_dev = D.to_device(a, np.float32, dev)
    books_dev = D.to_device(books, np.float32, dev)
    prep = prepare_books(books_dev)
    near = torch.zeros(1, dtype=torch.int32, device=dev)
    codes = encode_device(a_dev, prep, c, k, v, 8, near)
    out = D.from_device(codes, kind)
    ties = int(near.item())
    EncodeStats.last_near_ties = ties
    return (out, ties) if return_near_ties else out


def _tree_parts(t):
    if isinstance(t, (tuple, list)):
        return t[0], t[1], t[2]
    return t.dims, t.thresholds, t.leaves


def hash_trees_device(trees, dev):
    """Stack per-codebook trees (hashing.HashTree or (dims, thr, leaves)) into
    device arrays; every tree must have the same depth."""
    if not trees:
        raise ShapeError("need at least one tree")
    parts = [_tree_parts(t) for t in trees]
    levels = {len(np.asarray(d)) for d, _, _ in parts}
    if len(levels) != 1:
        raise ConfigError("all hash trees of a layer must have the same depth")
    L = levels.pop()
    if not 1 <= L <= 16:
        raise ConfigError(f"tree depth {L} outside [1, 16]")
    dims = np.stack([np.asarray(d, np.int64) for d, _, _ in parts]).astype(np.int32)
    thr = np.stack([np.asarray(t, np.float32) for _, t, _ in parts])
    leaves = np.stack([np.asarray(lv, np.uint8) for _, _, lv in parts])
    if thr.shape[1] != (1 << L) - 1 or leaves.shape[1] != (1 << L):
        raise ShapeError("tree arrays inconsistent with their depth")
    return (D.to_device(dims, np.int32, dev), D.to_device(thr, np.float32, dev), D.to_device(leaves, np.uint8, dev), L)


def encode_hash(a, trees, code_stride: int = 0):
    """Tree-traversal encoding, (N, C) u8 (hashing.py:171-196) on the GPU."""
    n, d = _matrix_shape(a, "a")
    if not trees:
        raise ShapeError("need at least one tree")
    c = len(trees)
    if d % c != 0:
        raise ShapeError(f"input cols {d} not divisible by {c} trees")
    v = d // c
    kind = D.kind_of(a)
    dev = D.require_cuda()
    dims, thr, leaves, L = hash_trees_device(trees, dev)
    if int(dims.max()) >= v or int(dims.min()) < 0:
        raise ShapeError("tree split dimension outside the sub-vector")
    a_dev = D.to_device(a, np.float32, dev)
    width = code_stride or c
    codes = torch.empty((n, width), dtype=torch.uint8, device=dev)
    check(load().lut_encode_hash(D.ptr(a_dev), n, d, D.ptr(dims), D.ptr(thr), D.ptr(leaves), c, L, v, D.ptr(codes),
                                 width, D.stream_ptr()), "encode_hash")
    return D.from_device(codes if width == c else codes[:, :c], kind)


# ------------------------------------------------------------------ gather


def lut_gather_i32(enc, q, plan: KernelPlan = KernelPlan()):
    """Exact INT32 sums of INT8 entries (kernels.py:105-127)."""
    qshape = D.shape_of(q)
    qdt = q.dtype if isinstance(q, torch.Tensor) else np.asarray(q).dtype
    if len(qshape) != 3 or qdt not in (np.int8, torch.int8):
        raise ShapeError(f"table must be int8 (C, K, M), got {qdt} {qshape}")
    c, k, m = qshape
    _check_enc_shape(enc, c)
    kind = D.kind_of(enc)
    dev = D.require_cuda()
    codes = _codes_device(enc, c, k, dev)
    q_dev = D.to_device(q, np.int8, dev)
    n = codes.shape[0]
    out = torch.empty((n, m), dtype=torch.int32, device=dev)
    err = D.ErrFlag(dev)
    lib = load()
    check(lib.lut_gather_i8(D.ptr(codes), 8, n, c, k, m, D.ptr(q_dev), None, 0, None, 0, None, D.ptr(out), 0,
                            err.p, D.stream_ptr()), "lut_gather_i32")
    check(lib.lut_read_status(err.p, D.stream_ptr()), "lut_gather_i32")
    return D.from_device(out, kind)


def _gather_i8_f32(codes, q_dev, scales_dev, scale_mtile, bias_dev, act, c, k, m, err_p=None, out_hw=0, out=None):
    lib = load()
    n = codes.shape[0] if out_hw == 0 else codes.shape[0]
    if out is None:
        out = torch.empty((n, m), dtype=torch.float32, device=codes.device)
    check(lib.lut_gather_i8(D.ptr(codes), 8, n, c, k, m, D.ptr(q_dev), D.ptr(scales_dev), scale_mtile,
                            D.ptr(bias_dev), act, D.ptr(out), None, out_hw, err_p, D.stream_ptr()), "lut_gather_i8")
    return out


def _gather_f32(codes, table_dev, bias_dev, act, c, k, m, err_p=None, out_hw=0, out=None):
    lib = load()
    n = codes.shape[0]
    if out is None:
        out = torch.empty((n, m), dtype=torch.float32, device=codes.device)
    check(lib.lut_gather_f32(D.ptr(codes), 8, n, c, k, m, D.ptr(table_dev), D.ptr(bias_dev), act, D.ptr(out),
                             out_hw, err_p, D.stream_ptr()), "lut_gather_f32")
    return out


def lut_gather_accumulate(enc, table: LookupTableI8, plan: KernelPlan = KernelPlan()):
    """f32 output = f32(exact INT32 sum) * f32(scale) (kernels.py:130-135)."""
    c, k, m = D.shape_of(table.q)
    _check_enc_shape(enc, c)
    kind = D.kind_of(enc)
    dev = D.require_cuda()
    codes = _codes_device(enc, c, k, dev)
    err = D.ErrFlag(dev)
    if getattr(table, "per_codebook", False):  # extension: f32 sum of the dequantized entries
        from .quant import dequantized_table

        out = _gather_f32(codes, dequantized_table(table, dev), None, 0, c, k, m, err.p)
    else:
        q_dev = D.to_device(table.q, np.int8, dev)
        out = _gather_i8_f32(codes, q_dev, table.scales_tensor(dev), table.scale_mtile, None, 0, c, k, m, err.p)
    check(load().lut_read_status(err.p, D.stream_ptr()), "lut_gather_accumulate")
    return D.from_device(out, kind)


def lut_gather_f32(enc, table):
    """Float lookup; ascending-c f32 accumulation, bitwise equal to
    lut_matmul_ref (kernels.py:138-140, pq.py:196-214)."""
    tshape = D.shape_of(table)
    if len(tshape) != 3:
        raise ShapeError(f"table must be (C, K, M), got {tshape}")
    c, k, m = tshape
    _check_enc_shape(enc, c)
    kind = D.kind_of(enc)
    dev = D.require_cuda()
    codes = _codes_device(enc, c, k, dev)
    t_dev = D.to_device(table, np.float32, dev)
    err = D.ErrFlag(dev)
    out = _gather_f32(codes, t_dev, None, 0, c, k, m, err.p)
    check(load().lut_read_status(err.p, D.stream_ptr()), "lut_gather_f32")
    return D.from_device(out, kind)


def lut_gather_i32_tc(enc, q):
    """lut_gather_i32 on the tensor cores (one-hot kind::i8 GEMM, exact int32).
    Power-of-two K <= 128; codes are range-checked on the host/device first."""
    qshape = D.shape_of(q)
    if len(qshape) != 3:
        raise ShapeError(f"table must be int8 (C, K, M), got {qshape}")
    c, k, m = qshape
    _check_enc_shape(enc, c)
    kind = D.kind_of(enc)
    dev = D.require_cuda()
    codes = _codes_device(enc, c, k, dev)
    n = codes.shape[0]
    if codes.numel() and int(codes.max()) >= k:
        raise CorruptionError(f"encoding index {int(codes.max())} >= K={k}")
    lib = load()
    if lib.lut_onehot_image_bytes(c, k, m, 1) == 0:
        raise ConfigError("shape not supported by the tensor-core gather")
    stride = int(lib.lut_code_stride(c))
    padded = torch.zeros((n, stride), dtype=torch.uint8, device=dev)
    padded[:, :c] = codes
    q_dev = D.to_device(q, np.int8, dev)
    img = torch.empty(lib.lut_onehot_image_bytes(c, k, m, 1), dtype=torch.uint8, device=dev)
    check(lib.lut_onehot_prepare_i8(D.ptr(q_dev), c, k, m, img.data_ptr(), D.stream_ptr()), "onehot_prepare_i8")
    out = torch.empty((n, m), dtype=torch.int32, device=dev)
    check(lib.lut_gather_onehot(D.ptr(padded), stride, n, c, k, m, 1, img.data_ptr(), None, 0, None, 0, None,
                                D.ptr(out), 0, D.stream_ptr()), "lut_gather_i32_tc")
    return D.from_device(out, kind)


# ------------------------------------------------------------------- layer


def lut_layer_infer(a, layer, plan: KernelPlan = KernelPlan(), integer: bool | None = None,
                    encoder: str = "dist", out=None):
    """Full layer inference (kernels.py:143-178): encode -> lookup -> + bias.

    `layer` is this package's LutLayer, or any object with the reference
    LutLayer's attributes (books, table, qtable, bias, trees).  numpy input is
    streamed through the native host executor (copies overlapped with
    compute); `out` optionally names a preallocated (pinned) host array."""
    from .layer import as_device_layer

    if encoder not in ("dist", "hash"):
        raise ConfigError(f"unknown encoder {encoder!r}")
    dl = as_device_layer(layer)
    if encoder == "hash":
        if not dl.trees:
            raise ConfigError("layer has no hash trees; train with hashing enabled")
    if integer is None:
        integer = dl.has_qtable
    if integer and not dl.has_qtable:
        raise ConfigError("integer path requested but the layer has no quantized table")
    n, d = _matrix_shape(a, "a")
    if d != dl.d:
        raise ShapeError(f"input cols {d} != C*V = {dl.c}*{dl.v}")
    if encoder == "hash":
        return dl.infer_hash(a, integer)
    return dl.infer(a, bool(integer), out=out)


# ------------------------------------------------------------------- costs


def flop_counter(n: int, d: int, m: int, k: int, v: int) -> dict:
    """encode N*D*K, lookup_aggregate N*M*D/V, dense N*D*M (kernels.py:181-193)."""
    if v < 1 or d % v != 0:
        raise ConfigError(f"D={d} not divisible by V={v}")
    return {"encode": n * d * k, "lookup_aggregate": n * m * (d // v), "dense": n * d * m}


# ------------------------------------------------------------------- bench


@dataclass
class BenchReport:
    """Timing of the LUT pipeline against the dense matmul_ref
    (kernels.py:249-285).  Here both paths run on the GPU and are timed with
    CUDA events on the launching stream (operands resident in HBM)."""

    n: int
    d: int
    m: int
    k: int
    v: int
    plan: KernelPlan
    repetitions: int
    lut_min_ns: int
    lut_median_ns: int
    dense_min_ns: int
    dense_median_ns: int

    @property
    def gflops_equiv(self) -> float:
        """Dense-equivalent MAC throughput of the LUT path, in G MAC/s."""
        return (self.n * self.d * self.m) / self.lut_median_ns

    @property
    def speedup_vs_dense(self) -> float:
        return self.dense_median_ns / self.lut_median_ns

    CSV_HEADER = ("n,d,m,k,v,n_block,k_block,group_size,"
                  "min_ns,median_ns,gflops_equiv,speedup_vs_dense")

    def csv_row(self) -> str:
        return (f"{self.n},{self.d},{self.m},{self.k},{self.v},"
                f"{self.plan.n_block},{self.plan.k_block},{self.plan.group_size},"
                f"{self.lut_min_ns},{self.lut_median_ns},"
                f"{self.gflops_equiv:.6f},{self.speedup_vs_dense:.4f}")


def _time_device(fn, repetitions: int, warmup: int) -> list[int]:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    stream = torch.cuda.current_stream()
    for _ in range(repetitions):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        times.append(int(e0.elapsed_time(e1) * 1e6))
    return times


def bench_kernel(shape, plan: KernelPlan = KernelPlan(), repetitions: int = 9, rng=None,
                 warmup: int = 2) -> BenchReport:
    """Time the quantized LUT pipeline (encode + int8 lookup-accumulate) and
    the dense reference product on one (N, D, M, K, V) shape with random
    operands (kernels.py:288-349); min and median over `repetitions`."""
    n, d, m, k, v = shape
    if repetitions < 5:
        raise ConfigError(f"need at least 5 repetitions, got {repetitions}")
    if d % v != 0:
        raise ConfigError(f"D={d} not divisible by V={v}")
    if rng is None:
        rng = np.random.default_rng(0)
    from .layer import LutLayer
    from .pq import PqConfig

    c_books = d // v
    a = rng.standard_normal((n, d)).astype(F32)
    books = rng.standard_normal((c_books, k, v)).astype(F32)
    b = rng.standard_normal((d, m)).astype(F32)
    dev = D.require_cuda()
    a_dev, b_dev = D.to_device(a, F32, dev), D.to_device(b, F32, dev)
    layer = LutLayer(cfg=PqConfig(v=v, k=k), books=books, weight=b_dev, qat=True, device=dev)
    lib = load()
    out = torch.empty((n, m), dtype=torch.float32, device=dev)
    codes = torch.empty((n, layer.code_stride), dtype=torch.uint8, device=dev)

    def lut_path():
        layer.forward_device(a_dev, True, out=out, codes=codes)

    def dense_path():
        check(lib.lut_matmul_ref_f32(D.ptr(a_dev), D.ptr(b_dev), n, d, m, D.ptr(out), D.stream_ptr()),
              "matmul_ref")

    lut_t = _time_device(lut_path, repetitions, warmup)
    dense_t = _time_device(dense_path, repetitions, warmup)
    return BenchReport(n=n, d=d, m=m, k=k, v=v, plan=plan, repetitions=repetitions,
                       lut_min_ns=int(np.min(lut_t)), lut_median_ns=int(np.median(lut_t)),
                       dense_min_ns=int(np.min(dense_t)), dense_median_ns=int(np.median(dense_t)))
