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


def matmul_ref(a, b):
    """Dense product, f32 products added in ascending k from +0.0 (no FMA):
    bitwise equal to tensor.py:110-125, on the GPU (lut_matmul_ref_f32)."""
    ash, bsh = D.shape_of(a), D.shape_of(b)
    if len(ash) != 2 or len(bsh) != 2:
        raise ShapeError(f"matmul_ref needs 2-D operands, got {ash} x {bsh}")
    if ash[1] != bsh[0]:
        raise ShapeError(f"inner dims differ: {ash} x {bsh}")
    kind = D.kind_of(a)
    dev = D.require_cuda()
    a_dev, b_dev = D.to_device(a, F32, dev), D.to_device(b, F32, dev)
    out = torch.empty((ash[0], bsh[1]), dtype=torch.float32, device=dev)
    check(load().lut_matmul_ref_f32(D.ptr(a_dev), D.ptr(b_dev), ash[0], ash[1], bsh[1], D.ptr(out),
                                    D.stream_ptr()), "matmul_ref")
    if ash[1] == 0:
        out.zero_()
    return D.from_device(out, kind)


def split_subvectors(a, v: int) -> list:
    """D/v column blocks of width v, as views (tensor.py:128-135)."""
    a = as_matrix(a, "a")
    if v < 1:
        raise ConfigError(f"sub-vector length must be >= 1, got {v}")
    if a.shape[1] % v != 0:
        raise ConfigError(f"cols {a.shape[1]} not divisible by sub-vector length {v}")
    return [a[:, c * v:(c + 1) * v] for c in range(a.shape[1] // v)]
