"""LUT-replaced Linear / Conv modules and the inference driver.

`LutDense` / `LutConv` keep the reference's shape contract (lutkit/model.py:
136-218): dense flattens inputs with more than two dims to (N, -1); conv
lowers NCHW through im2col (channel-major patches), runs the LUT core and
returns NCHW.  Here the conv lowering is fused into the encode kernel (no
im2col matrix in HBM) and the NCHW raise is fused into the gather's store.
`LutLinear` / `LutConv2d` are torch.nn.Module forms of the same layers for
device-resident pipelines (LutLinear applies over the last dim).
`predict_fast` mirrors lutkit/pipeline.py:206-225."""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from ._lib import check, load
from .errors import ShapeError
from .kernels import ACTS, EncodeStats, KernelPlan, _gather_f32, _gather_i8_f32, lut_layer_infer
from .layer import LutLayer, as_device_layer
from .tensor import conv_out_hw

F32 = np.float32


class LutDense:
    """Dense layer replaced by encode + lookup (model.py:136-176)."""

    def __init__(self, lut):
        self.lut = as_device_layer(lut)

    def core_shape(self):
        return self.lut.d, self.lut.m

    def forward(self, x, train: bool = False, integer=None, encoder="dist"):
        shp = D.shape_of(x)
        if len(shp) > 2:
            x = x.reshape(shp[0], -1)
        return lut_layer_infer(x, self.lut, integer=integer, encoder=encoder), None


class LutConv:
    """Convolution whose im2col'd core runs through the LUT path (model.py:179-218)."""

    def __init__(self, in_channels: int, kernel: int, stride: int, pad: int, lut):
        self.in_channels = in_channels
        self.kernel = kernel
        self.stride = stride
        self.pad = pad
        self.lut = as_device_layer(lut)

    def forward(self, x, train: bool = False, integer=None, encoder="dist"):
        return conv_forward(x, self.lut, self.in_channels, self.kernel, self.stride, self.pad, integer), None


def conv_forward(x, lut: LutLayer, cin: int, kernel: int, stride: int, pad: int, integer=None):
    """Fused conv LUT layer: encode reads NCHW directly (im2col on the fly),
    gather writes NCHW directly (Conv._lower/_raise, model.py:105-114)."""
    shp = D.shape_of(x)
    if len(shp) != 4 or shp[1] != cin:
        raise ShapeError(f"conv expected NCHW with {cin} channels, got {shp}")
    b, _, h, w = shp
    ho, wo = conv_out_hw(h, w, kernel, kernel, stride, pad)
    if cin * kernel * kernel != lut.d:
        raise ShapeError(f"patch cols {cin * kernel * kernel} != C*V = {lut.d}")
    if integer is None:
        integer = lut.has_qtable
    kind = D.kind_of(x)
    dev = lut.device
    x_dev = D.to_device(x, F32, dev)
    n = b * ho * wo
    codes = torch.empty((n, max(lut.c, 1)), dtype=torch.uint8, device=dev)
    near = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = load()
    check(lib.lut_encode_conv_f32(D.ptr(x_dev), b, cin, h, w, kernel, kernel, stride, pad, D.ptr(lut.books_prep),
                                  lut.c, lut.k, lut.v, D.ptr(codes), 8, D.ptr(near), D.stream_ptr()), "LutConv")
    out = torch.empty((b, lut.m, ho, wo), dtype=torch.float32, device=dev)
    act = ACTS[lut.act]
    if integer:
        _gather_i8_f32(codes, lut.qtable.q, lut.qtable.scales_tensor(dev), lut.qtable.scale_mtile, lut.bias, act,
                       lut.c, lut.k, lut.m, None, out_hw=ho * wo, out=out)
    else:
        _gather_f32(codes, lut.table, lut.bias, act, lut.c, lut.k, lut.m, None, out_hw=ho * wo, out=out)
    return D.from_device(out, kind)


class LutLinear(torch.nn.Module):
    """torch module over the last dim: (..., D) -> (..., M) on the GPU."""

    def __init__(self, lut, integer=None):
        super().__init__()
        self.lut = as_device_layer(lut)
        self.integer = self.lut.has_qtable if integer is None else bool(integer)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        lead = x.shape[:-1]
        a = x.reshape(-1, x.shape[-1]).to(torch.float32).contiguous()
        if a.shape[1] != self.lut.d:
            raise ShapeError(f"input cols {a.shape[1]} != C*V = {self.lut.d}")
        return self.lut.forward_device(a, self.integer).reshape(*lead, self.lut.m)


class LutConv2d(torch.nn.Module):
    """torch module: NCHW -> NCHW with fused im2col encode and NCHW store."""

    def __init__(self, in_channels: int, kernel: int, stride: int, pad: int, lut, integer=None):
        super().__init__()
        self.in_channels, self.kernel, self.stride, self.pad = in_channels, kernel, stride, pad
        self.lut = as_device_layer(lut)
        self.integer = integer

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return conv_forward(x, self.lut, self.in_channels, self.kernel, self.stride, self.pad, self.integer)


def predict_fast(model, x, plan: KernelPlan = KernelPlan(), encoder: str = "dist", integer=None):
    """Inference through the GPU kernels; non-LUT layers run their own
    forward (pipeline.py:206-225).  Accepts a reference-style model (object
    with `.layers`) or any iterable of layers; reference LutDense/LutConv
    instances are recognised by their attributes."""
    layers = model.layers if hasattr(model, "layers") else list(model)
    for layer in layers:
        lut = getattr(layer, "lut", None)
        name = type(layer).__name__
        if lut is not None and (isinstance(layer, LutConv) or name == "LutConv"):
            x = conv_forward(x, as_device_layer(lut), layer.in_channels, layer.kernel, layer.stride, layer.pad,
                             integer)
        elif lut is not None and (isinstance(layer, LutDense) or name == "LutDense"):
            shp = D.shape_of(x)
            if len(shp) > 2:
                x = x.reshape(shp[0], -1)
            x = lut_layer_infer(x, lut, plan, integer=integer, encoder=encoder)
        elif isinstance(layer, torch.nn.Module):
            x = layer(x)
        else:
            x, _ = layer.forward(x, train=False)
    return x
