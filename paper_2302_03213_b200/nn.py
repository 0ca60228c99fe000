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

import ctypes as C

import numpy as np
import torch

from . import _device as D
from ._lib import check, load
from .errors import ConfigError, ShapeError
from .kernels import KernelPlan, lut_layer_infer
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
    if integer and not lut.has_qtable:  # kernels.py:166-170
        raise ConfigError("integer path requested but the layer has no quantized table")
    kind = D.kind_of(x)
    dev = lut.device
    x_dev = D.to_device(x, F32, dev)
    n = b * ho * wo
    codes = torch.empty((n, lut.code_stride), dtype=torch.uint8, device=dev)
    out = torch.empty((b, lut.m, ho, wo), dtype=torch.float32, device=dev)
    # one ABI call: fused-im2col encode, then the lookup (launched as a programmatic
    # dependent of the encode) storing NCHW; codes come from the distance encoder,
    # so they are < K by construction and no error flag / stream sync is needed
    check(load().lut_conv_layer_forward(C.byref(lut.desc(bool(integer))), D.ptr(x_dev), b, cin, h, w, kernel, kernel,
                                        stride, pad, D.ptr(out), D.ptr(codes), None, D.stream_ptr()), "LutConv")
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


class Relu:
    """max(x, 0) (model.py:27-35); after a LUT layer it is fused into that
    layer's gather epilogue by predict_fast."""

    def forward(self, x, train: bool = False):
        if isinstance(x, torch.Tensor):
            return torch.clamp_min(x, 0.0), None
        return np.maximum(x, 0.0), None


class Dense:
    """y = x @ W + b on the GPU (model.py:38-72).  Not the LUT path: a plain
    cuBLAS fp32 GEMM (TF32 off) for the layers a LUT model keeps dense."""

    def __init__(self, weight, bias, device=None):
        dev = torch.device(device) if device is not None else D.require_cuda()
        self.weight = D.to_device(weight, F32, dev)
        self.bias = D.to_device(bias, F32, dev)
        if self.weight.dim() != 2 or self.bias.shape != (self.weight.shape[1],):
            raise ShapeError(f"dense weight {tuple(self.weight.shape)} / bias {tuple(self.bias.shape)} mismatch")

    def core_shape(self):
        return tuple(self.weight.shape)

    def forward(self, x, train: bool = False):
        kind = D.kind_of(x)
        t = D.to_device(x, F32, self.weight.device)
        if t.dim() > 2:
            t = t.reshape(t.shape[0], -1)
        if t.shape[1] != self.weight.shape[0]:
            raise ShapeError(f"dense layer got {t.shape[1]} features, expected {self.weight.shape[0]}")
        return D.from_device(_matmul_f32(t, self.weight) + self.bias, kind), None


class Conv(Dense):
    """im2col (lut_im2col_f32) + fp32 GEMM + NCHW raise (model.py:75-133)."""

    def __init__(self, in_channels: int, kernel: int, stride: int, pad: int, weight, bias, device=None):
        super().__init__(weight, bias, device)
        self.in_channels, self.kernel, self.stride, self.pad = in_channels, kernel, stride, pad
        if self.weight.shape[0] != in_channels * kernel * kernel:
            raise ShapeError(f"conv weight rows {self.weight.shape[0]} != {in_channels}*{kernel}*{kernel}")

    def forward(self, x, train: bool = False):
        from .tensor import im2col

        shp = D.shape_of(x)
        if len(shp) != 4 or shp[1] != self.in_channels:
            raise ShapeError(f"conv expected NCHW with {self.in_channels} channels, got {shp}")
        kind = D.kind_of(x)
        ho, wo = conv_out_hw(shp[2], shp[3], self.kernel, self.kernel, self.stride, self.pad)
        cols = im2col(D.to_device(x, F32, self.weight.device), self.kernel, self.kernel, self.stride, self.pad)
        y = _matmul_f32(cols, self.weight) + self.bias
        out = y.reshape(shp[0], ho, wo, -1).permute(0, 3, 1, 2).contiguous()
        return D.from_device(out, kind), None


def _matmul_f32(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return a @ b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


class Model:
    """Ordered layer stack (model.py:224-244); `predict_logits` runs the
    fast path."""

    def __init__(self, layers: list):
        self.layers = layers

    def predict_logits(self, x, encoder: str = "dist", integer=None):
        return predict_fast(self, x, encoder=encoder, integer=integer)


def _is_lut(layer, cls) -> bool:
    return getattr(layer, "lut", None) is not None and (isinstance(layer, cls) or type(layer).__name__ == cls.__name__)


def _is_relu(layer) -> bool:
    return isinstance(layer, Relu) or type(layer).__name__ == "Relu"


def predict_fast(model, x, plan: KernelPlan = KernelPlan(), encoder: str = "dist", integer=None):
    """Inference through the GPU kernels; non-LUT layers run their own
    forward (pipeline.py:206-225).  Accepts a reference-style model (object
    with `.layers`) or any iterable of layers; reference LutDense/LutConv
    instances are recognised by their attributes.  A Relu right after a LUT
    layer is fused into that layer's gather epilogue (same values: the
    reference applies max(y, 0) to the layer's f32 output)."""
    layers = model.layers if hasattr(model, "layers") else list(model)
    kind = D.kind_of(x)
    i = 0
    while i < len(layers):
        layer = layers[i]
        conv, dense = _is_lut(layer, LutConv), _is_lut(layer, LutDense)
        if conv or dense:
            lut = as_device_layer(layer.lut)
            if i + 1 < len(layers) and _is_relu(layers[i + 1]) and lut.act in (None, "none"):
                lut = lut.with_act("relu")
                i += 1
            if conv:
                if encoder != "dist":
                    from .tensor import im2col

                    shp = D.shape_of(x)
                    ho, wo = conv_out_hw(shp[2], shp[3], layer.kernel, layer.kernel, layer.stride, layer.pad)
                    cols = im2col(D.to_device(x, F32, lut.device), layer.kernel, layer.kernel, layer.stride,
                                  layer.pad)
                    y = lut_layer_infer(cols, lut, plan, integer=integer, encoder=encoder)
                    x = y.reshape(shp[0], ho, wo, -1).permute(0, 3, 1, 2).contiguous()
                else:
                    x = conv_forward(D.to_device(x, F32, lut.device), lut, layer.in_channels, layer.kernel,
                                     layer.stride, layer.pad, integer)
            else:
                x = D.to_device(x, F32, lut.device)
                if x.dim() > 2:
                    x = x.reshape(x.shape[0], -1)
                x = lut_layer_infer(x, lut, plan, integer=integer, encoder=encoder)
        elif isinstance(layer, torch.nn.Module):
            x = layer(x)
        elif isinstance(layer, (Dense, Relu)):
            x, _ = layer.forward(x, train=False)
        else:  # a foreign (reference numpy) layer: hand it host data
            x, _ = layer.forward(x.cpu().numpy() if isinstance(x, torch.Tensor) else x, train=False)
        i += 1
    return D.from_device(x, kind) if isinstance(x, torch.Tensor) else x
