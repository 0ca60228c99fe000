"""INT8 table quantization — mirror of lutkit/quant.py:19-62, computed on the GPU.

One scale per table (scale = max|T|/127, clamp +-127, round-half-even), plus
the BASELINE config-2 extension `quantize_table(table, scale_mtile=t)`: one
scale per m-tile of `t` output columns, shared by every codebook so the
lookup still accumulates a plain integer sum (parity UNPINNED: the
reference rejects per-codebook scales)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from ._lib import check, load
from .errors import DataError, ShapeError

QMAX = 127
F32 = np.float32


@dataclass(frozen=True)
class LookupTableI8:
    """(C, K, M) int8 entries and one f32 scale (or per-m-tile scales)."""

    q: object             # np.ndarray int8 or torch int8 tensor
    scale: object         # np.float32, or 1-D array of per-m-tile scales
    scale_mtile: int = 0  # 0 = one scale per table (reference)
    # set by quantize_table: entries and scales were produced by the device
    # quantizer (never -128, scales > 0), so construction skips the value
    # checks and their device->host sync
    validated: bool = field(default=False, compare=False, repr=False)
    # extension (configs[1]): scale shape (C, ceil(M / scale_mtile)) — one scale
    # per (codebook, m-tile); the lookup then sums f32(q) * scale per codebook
    per_codebook: bool = False

    def __post_init__(self) -> None:
        q = self.q
        if isinstance(q, torch.Tensor):
            ok = q.dim() == 3 and q.dtype == torch.int8
        else:
            ok = np.asarray(q).ndim == 3 and np.asarray(q).dtype == np.int8
        if not ok:
            raise ShapeError(f"quantized table must be int8 (C, K, M), got {getattr(q, 'dtype', None)} "
                             f"{tuple(q.shape)}")
        if self.validated:
            return
        s = self.scale
        svals = s.detach().cpu().numpy() if isinstance(s, torch.Tensor) else np.asarray(s, F32)
        if not np.all(svals > 0):
            raise DataError(f"scale must be positive, got {s}")
        if q.numel() if isinstance(q, torch.Tensor) else np.asarray(q).size:
            qmin = int(q.min()) if isinstance(q, torch.Tensor) else int(np.asarray(q).min())
            if qmin < -QMAX:
                raise DataError("quantized entries must lie in [-127, 127]")

    def scales_tensor(self, device) -> torch.Tensor:
        s = self.scale
        if isinstance(s, torch.Tensor):
            return s.to(device=device, dtype=torch.float32).reshape(-1)
        return torch.as_tensor(np.asarray(s, F32).reshape(-1), device=device)


def quantize_table(table, scale_mtile: int = 0, per_codebook: bool = False) -> LookupTableI8:
    """GPU restatement of quant.quantize_table (quant.py:40-57); `scale_mtile`
    (one scale per m-tile) and `per_codebook` (one scale per (codebook, m-tile))
    are the BASELINE configs[1] extensions."""
    kind = D.kind_of(table)
    shp = D.shape_of(table)
    if len(shp) != 3:
        raise ShapeError(f"table must be (C, K, M), got {shp}")
    if scale_mtile < 0:
        raise ShapeError("scale_mtile must be >= 0")
    if per_codebook:
        return _quantize_per_codebook(table, scale_mtile or shp[2], kind)
    lib = load()
    dev = D.require_cuda()
    t = D.to_device(table, np.float32, dev)
    c, k, m = shp
    ntiles = (m + scale_mtile - 1) // scale_mtile if scale_mtile > 0 else 1
    q = torch.empty((c, k, m), dtype=torch.int8, device=dev)
    scales = torch.empty(max(ntiles, 1), dtype=torch.float32, device=dev)
    scratch = torch.empty(max(1, lib.lut_quantize_scratch_bytes(c, k, m, scale_mtile)), dtype=torch.uint8,
                          device=dev)
    err = D.ErrFlag(dev)
    check(lib.lut_quantize_table(D.ptr(t), c, k, m, scale_mtile, D.ptr(q), scales.data_ptr(), scratch.data_ptr(),
                                 err.p, D.stream_ptr()), "quantize_table")
    check(lib.lut_read_status(err.p, D.stream_ptr()), "quantize_table")
    if kind == D.TORCH_CUDA:
        return LookupTableI8(q=q, scale=scales if scale_mtile else scales[0], scale_mtile=scale_mtile, validated=True)
    qh = D.from_device(q, kind)
    sh = scales.cpu().numpy()
    return LookupTableI8(q=qh, scale=sh if scale_mtile else F32(sh[0]), scale_mtile=scale_mtile, validated=True)


def _quantize_per_codebook(table, mtile: int, kind) -> LookupTableI8:
    """The per-m-tile quantizer applied to each codebook's (1, K, M) slice."""
    lib = load()
    dev = D.require_cuda()
    t = D.to_device(table, np.float32, dev)
    c, k, m = t.shape
    ntiles = (m + mtile - 1) // mtile
    q = torch.empty((c, k, m), dtype=torch.int8, device=dev)
    scales = torch.empty((max(c, 1), ntiles), dtype=torch.float32, device=dev)
    scratch = torch.empty(max(1, lib.lut_quantize_scratch_bytes(1, k, m, mtile)), dtype=torch.uint8, device=dev)
    err = D.ErrFlag(dev)
    for ci in range(c):
        check(lib.lut_quantize_table(D.ptr(t[ci]), 1, k, m, mtile, D.ptr(q[ci]), scales[ci].data_ptr(),
                                     scratch.data_ptr(), err.p, D.stream_ptr()), "quantize_table")
    check(lib.lut_read_status(err.p, D.stream_ptr()), "quantize_table")
    if kind != D.TORCH_CUDA:
        q, scales = D.from_device(q, kind), scales.cpu().numpy()
    return LookupTableI8(q=q, scale=scales, scale_mtile=mtile, validated=True, per_codebook=True)


def dequantized_table(qt: LookupTableI8, device) -> torch.Tensor:
    """(C, K, M) f32 device table fl(q * scale) for the table's scale layout."""
    q = D.to_device(qt.q, np.int8, device)
    c, k, m = q.shape
    s = qt.scales_tensor(device)
    if qt.per_codebook:
        col = torch.arange(m, device=device) // qt.scale_mtile
        return q.float() * s.reshape(c, -1)[:, col][:, None, :]
    if qt.scale_mtile:
        col = torch.arange(m, device=device) // qt.scale_mtile
        return q.float() * s[col]
    return q.float() * s[0]


def dequantize(qt: LookupTableI8):
    """entry * scale in f32 (quant.py:60-62)."""
    if qt.per_codebook:
        out = dequantized_table(qt, D.require_cuda())
        return out if isinstance(qt.q, torch.Tensor) else out.cpu().numpy()
    q = qt.q
    if isinstance(q, torch.Tensor):
        s = qt.scales_tensor(q.device)
        if qt.scale_mtile:
            col = torch.arange(q.shape[2], device=q.device) // qt.scale_mtile
            return q.float() * s[col]
        return q.float() * s[0]
    q = np.asarray(q)
    if qt.scale_mtile:
        col = np.arange(q.shape[2]) // qt.scale_mtile
        return q.astype(F32) * np.asarray(qt.scale, F32)[col]
    return q.astype(F32) * F32(qt.scale)
