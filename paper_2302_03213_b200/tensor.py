"""Input contract and conv lowering — mirror of lutkit/tensor.py:28-79."""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from ._lib import check, load
from .errors import ConfigError, ShapeError

F32 = np.float32


def as_matrix(a, name: str = "matrix"):
    """Contiguous 2-D f32 (tensor.py:28-33); keeps the caller's array kind."""
    shp = D.shape_of(a)
    if len(shp) != 2:
        raise ShapeError(f"{name} must be 2-D, got shape {shp}")
    if isinstance(a, torch.Tensor):
        return a.to(torch.float32).contiguous()
    return np.ascontiguousarray(a, dtype=F32)


def conv_out_hw(h: int, w: int, kh: int, kw: int, stride: int, pad: int) -> tuple[int, int]:
    if stride < 1:
        raise ConfigError(f"stride must be >= 1, got {stride}")
    if pad < 0:
        raise ConfigError(f"pad must be >= 0, got {pad}")
    hp, wp = h + 2 * pad, w + 2 * pad
    if kh < 1 or kw < 1 or kh > hp or kw > wp:
        raise ShapeError(f"kernel {kh}x{kw} does not fit padded input {hp}x{wp}")
    return (hp - kh) // stride + 1, (wp - kw) // stride + 1


def im2col(x, kernel_h: int, kernel_w: int, stride: int = 1, pad: int = 0):
    """Patch rows (n*ho*wo) x cols (c*kh*kw), channel-major (tensor.py:36-79),
    built by the lut_im2col_f32 kernel."""
    shp = D.shape_of(x)
    if len(shp) != 4:
        raise ShapeError(f"im2col input must be 4-D NCHW, got shape {shp}")
    n, ch, h, w = shp
    ho, wo = conv_out_hw(h, w, kernel_h, kernel_w, stride, pad)
    kind = D.kind_of(x)
    dev = D.require_cuda()
    x_dev = D.to_device(x, F32, dev)
    cols = torch.empty((n * ho * wo, ch * kernel_h * kernel_w), dtype=torch.float32, device=dev)
    if cols.numel():
        check(load().lut_im2col_f32(D.ptr(x_dev), n, ch, h, w, kernel_h, kernel_w, stride, pad, D.ptr(cols),
                                    D.stream_ptr()), "im2col")
    return D.from_device(cols, kind)
