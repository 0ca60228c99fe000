"""`.lutn` model container, read straight into device tables.

Same format and error behaviour as the reference (lutkit/container.py:1-23):

    magic 'LUTN' | u32 version=1 | u32 record_count | records...
    record: u8 kind (1 dense, 2 lut) | u8 activation (0 none, 1 relu) |
            u8 geometry (0 flat, 1 conv + u32 kernel, stride, pad) | payload
    dense:  u32 D, M | f32 W[D*M] | f32 b[M]
    lut:    u32 D, M, K, V | f32 temperature | f32 centroids[C*K*V] |
            u8 tag (1 f32 table[C*K*M] | 2 i8 q[C*K*M] + f32 scale) |
            u8 tree_count, per tree: u32 L | u32 dims[L] | f32 thr[2^L-1] | u8 leaves[2^L]

Parsing is split from placement: `parse_records` turns the bytes into host
records (zero-copy numpy views where the layout allows) and is what the CPU
tests exercise; `model_from_bytes` then uploads every table once into HBM,
builds the encode record of each codebook and, for int8 tables, the tcgen05
one-hot image, so the first inference call launches kernels only.  A LUT
layer followed by Relu keeps both layers in `Model.layers` (round trips stay
byte-identical) and runs as one fused epilogue in `predict_fast`.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import ContainerError

MAGIC = b"LUTN"
VERSION = 1
KIND_DENSE, KIND_LUT = 1, 2
TABLE_F32, TABLE_I8 = 1, 2
F32 = np.float32


@dataclass
class DenseRecord:
    """container.py:143-150 / :184-197."""

    weight: np.ndarray                      # (D, M) f32
    bias: np.ndarray                        # (M,) f32
    conv: tuple[int, int, int] | None = None  # kernel, stride, pad


@dataclass
class LutRecord:
    """container.py:95-124 / :197-242.  Exactly one of table / q is set."""

    books: np.ndarray                       # (C, K, V) f32
    m: int
    temperature: float
    table: np.ndarray | None = None         # (C, K, M) f32
    q: np.ndarray | None = None             # (C, K, M) i8
    scale: float = 0.0
    trees: list = field(default_factory=list)  # (dims int64 (L,), thr f32, leaves u8)
    conv: tuple[int, int, int] | None = None


class _Reader:
    def __init__(self, raw):
        self.raw = memoryview(raw)
        self.pos = 0

    def take(self, n: int) -> memoryview:
        if n < 0 or self.pos + n > len(self.raw):
            raise ContainerError("container truncated")
        chunk = self.raw[self.pos:self.pos + n]
        self.pos += n
        return chunk

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))

    def array(self, dtype: str, count: int, shape) -> np.ndarray:
        dt = np.dtype(dtype)
        return np.frombuffer(self.take(dt.itemsize * count), dtype=dt).reshape(shape)


def parse_records(raw) -> list[tuple[object, int]]:
    """Bytes -> [(DenseRecord | LutRecord, activation)] with the reference's
    validation (container.py:159-182): magic, version, kind / geometry /
    table / activation tags, truncation and trailing bytes."""
    r = _Reader(raw)
    if bytes(r.take(4)) != MAGIC:
        raise ContainerError("bad magic: not a LUTN model container")
    version, count = r.unpack("<II")
    if version != VERSION:
        raise ContainerError(f"unsupported container version {version}")
    out = []
    for _ in range(count):
        kind, activation, geom = r.unpack("<BBB")
        if kind not in (KIND_DENSE, KIND_LUT):
            raise ContainerError(f"unknown record kind {kind} (version error)")
        if geom not in (0, 1):
            raise ContainerError(f"unknown geometry tag {geom} (version error)")
        conv = tuple(r.unpack("<III")) if geom == 1 else None
        if kind == KIND_DENSE:
            d, m = r.unpack("<II")
            rec = DenseRecord(weight=r.array("<f4", d * m, (d, m)), bias=r.array("<f4", m, (m,)), conv=conv)
        else:
            rec = _parse_lut(r, conv)
        if activation not in (0, 1):
            raise ContainerError(f"unknown activation tag {activation} (version error)")
        out.append((rec, activation))
    if r.pos != len(r.raw):
        raise ContainerError(f"{len(r.raw) - r.pos} trailing bytes after last record")
    return out


def _parse_lut(r: _Reader, conv) -> LutRecord:
    d, m, k, v, temperature = r.unpack("<IIIIf")
    if v == 0 or d % v:
        raise ContainerError(f"corrupt LUT record: D={d} not divisible by V={v}")
    c = d // v
    rec = LutRecord(books=r.array("<f4", c * k * v, (c, k, v)), m=m, temperature=temperature, conv=conv)
    (tag,) = r.unpack("<B")
    if tag == TABLE_F32:
        rec.table = r.array("<f4", c * k * m, (c, k, m))
    elif tag == TABLE_I8:
        rec.q = r.array("|i1", c * k * m, (c, k, m))
        (rec.scale,) = r.unpack("<f")
    else:
        raise ContainerError(f"unknown table tag {tag} (version error)")
    (ntrees,) = r.unpack("<B")
    for _ in range(ntrees):
        (levels,) = r.unpack("<I")
        if levels > 30:
            raise ContainerError(f"corrupt hash tree depth {levels}")
        dims = r.array("<u4", levels, (levels,)).astype(np.int64)
        thr = r.array("<f4", 2 ** levels - 1, (2 ** levels - 1,))
        leaves = r.array("|u1", 2 ** levels, (2 ** levels,))
        rec.trees.append((dims, thr, leaves))
    return rec


def records_bytes(records: list[tuple[object, int]]) -> bytes:
    """[(record, activation)] -> bytes (container.py:50-124 layout)."""
    parts = [MAGIC, struct.pack("<II", VERSION, len(records))]
    for rec, activation in records:
        is_lut = isinstance(rec, LutRecord)
        parts.append(struct.pack("<BBB", KIND_LUT if is_lut else KIND_DENSE, activation, 0 if rec.conv is None else 1))
        if rec.conv is not None:
            parts.append(struct.pack("<III", *rec.conv))
        if not is_lut:
            w = np.ascontiguousarray(rec.weight, dtype="<f4")
            parts += [struct.pack("<II", *w.shape), w.tobytes(), np.ascontiguousarray(rec.bias, dtype="<f4").tobytes()]
            continue
        c, k, v = rec.books.shape
        parts.append(struct.pack("<IIIIf", c * v, rec.m, k, v, rec.temperature))
        parts.append(np.ascontiguousarray(rec.books, dtype="<f4").tobytes())
        if rec.q is not None:
            parts += [struct.pack("<B", TABLE_I8), np.ascontiguousarray(rec.q, dtype="|i1").tobytes(),
                      struct.pack("<f", rec.scale)]
        else:
            parts += [struct.pack("<B", TABLE_F32), np.ascontiguousarray(rec.table, dtype="<f4").tobytes()]
        parts.append(struct.pack("<B", len(rec.trees)))
        for dims, thr, leaves in rec.trees:
            parts += [struct.pack("<I", len(dims)), np.ascontiguousarray(dims, dtype="<u4").tobytes(),
                      np.ascontiguousarray(thr, dtype="<f4").tobytes(),
                      np.ascontiguousarray(leaves, dtype="|u1").tobytes()]
    return b"".join(parts)


# ------------------------------------------------------------ device models


def model_from_bytes(raw, device=None, gather: str = "auto"):
    """Parse and place every layer in HBM (container.py:159-182)."""
    import torch

    from . import _device as D
    from .layer import LutLayer
    from .nn import Conv, Dense, LutConv, LutDense, Model, Relu
    from .pq import PqConfig
    from .quant import LookupTableI8

    dev = torch.device(device) if device is not None else D.require_cuda()
    if isinstance(raw, bytes):
        raw = bytearray(raw)  # writable views -> torch.from_numpy without copies per array
    layers = []
    for rec, activation in parse_records(raw):
        if isinstance(rec, DenseRecord):
            if rec.conv is None:
                layer = Dense(rec.weight, rec.bias, dev)
            else:
                kernel, stride, pad = rec.conv
                layer = Conv(rec.weight.shape[0] // (kernel * kernel), kernel, stride, pad, rec.weight, rec.bias, dev)
        else:
            c, k, v = rec.books.shape
            qtable = None
            if rec.q is not None:
                q = D.to_device(rec.q, np.int8, dev)
                qtable = LookupTableI8(q=q, scale=F32(rec.scale))
                table = q.to(torch.float32) * torch.tensor(F32(rec.scale), device=dev)  # q * scale, container.py:214
            else:
                table = D.to_device(rec.table, F32, dev)
            lut = LutLayer(cfg=PqConfig(v=v, k=k), books=rec.books, weight=None, bias=np.zeros(rec.m, F32),
                           qat=qtable is not None, table=table, qtable=qtable, trees=rec.trees or None, device=dev,
                           gather=gather)
            lut.temperature = rec.temperature
            if qtable is not None and lut.uses_tensor_cores(True):
                lut.onehot_image(True)
            if rec.conv is None:
                layer = LutDense(lut)
            else:
                kernel, stride, pad = rec.conv
                layer = LutConv(c * v // (kernel * kernel), kernel, stride, pad, lut)
        layers.append(layer)
        if activation == 1:
            layers.append(Relu())
    return Model(layers)


def load_model(path, device=None, gather: str = "auto"):
    path = Path(path)
    raw = bytearray(path.stat().st_size)
    with open(path, "rb") as f:
        if f.readinto(raw) != len(raw):
            raise ContainerError("container truncated")
    return model_from_bytes(raw, device, gather)


def _host(x, dtype):
    import torch

    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=dtype)


def model_records(model) -> list[tuple[object, int]]:
    """Layers -> records (container.py:58-124): Relu folds into the previous
    record's activation; a LUT layer's bias is folded into its table as
    bias/C and an int8 table with bias is re-quantized, like the reference."""
    from .nn import Conv, LutConv, LutDense, _is_lut, _is_relu
    from .quant import quantize_table

    layers = model.layers if hasattr(model, "layers") else list(model)
    out = []
    i = 0
    while i < len(layers):
        layer = layers[i]
        if _is_relu(layer):
            raise ContainerError("model starts with or has consecutive activations")
        activation = 1 if i + 1 < len(layers) and _is_relu(layers[i + 1]) else 0
        conv = None
        if _is_lut(layer, LutConv) or isinstance(layer, Conv) or type(layer).__name__ == "Conv":
            conv = (int(layer.kernel), int(layer.stride), int(layer.pad))
        if _is_lut(layer, LutDense) or _is_lut(layer, LutConv):
            out.append((_lut_record(layer.lut, conv, quantize_table), activation))
        else:
            out.append((DenseRecord(_host(layer.weight, F32), _host(layer.bias, F32), conv), activation))
        i += 2 if activation else 1
    return out


def _lut_record(lut, conv, quantize_table) -> LutRecord:
    books = _host(lut.books, F32)
    c = books.shape[0]
    table = getattr(lut, "table", None)
    table = None if table is None else _host(table, F32)
    bias = _host(lut.bias, F32) if lut.bias is not None else np.zeros(0, F32)
    has_bias = bool(bias.size) and bool(np.any(bias))
    if has_bias:
        table = table + (bias / F32(c)).astype(F32)[None, None, :]
    qt = getattr(lut, "qtable", None)
    temperature = getattr(lut, "temperature", None)
    if temperature is None:
        temp = getattr(lut, "temp", None)
        temperature = float(temp.t) if temp is not None else 1.0
    rec = LutRecord(books=books, m=0, temperature=temperature, conv=conv)
    if getattr(lut, "qat", False) or qt is not None:
        if qt is None or has_bias:
            qt = quantize_table(table)
        if getattr(qt, "scale_mtile", 0) or getattr(qt, "per_codebook", False):
            raise ContainerError("per-m-tile int8 scales cannot be stored in a version-1 container")
        rec.q = _host(qt.q, np.int8)
        rec.scale = float(_host(qt.scale, F32).reshape(-1)[0])
        rec.m = rec.q.shape[2]
    else:
        rec.table = table
        rec.m = table.shape[2]
    for t in getattr(lut, "trees", None) or []:
        dims, thr, leaves = (t[0], t[1], t[2]) if isinstance(t, (tuple, list)) else (t.dims, t.thresholds, t.leaves)
        rec.trees.append((_host(dims, np.int64), _host(thr, F32), _host(leaves, np.uint8)))
    return rec


def model_bytes(model) -> bytes:
    return records_bytes(model_records(model))


def save_model(path, model) -> None:
    Path(path).write_bytes(model_bytes(model))
