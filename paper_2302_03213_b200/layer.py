"""Device-resident LUT layer — mirror of lutkit.softpq.LutLayer (softpq.py:82-172).

Holds the codebooks (plus the prepared encode record), the f32 table and/or
its int8 twin, the bias and an optional fused activation, all in HBM.  The
layer is what `lut_layer_infer` consumes; a reference `LutLayer` (or any
object with the same attributes) is converted once and cached."""

from __future__ import annotations

import ctypes as C
import os
import weakref
import zlib

import numpy as np
import torch

from . import _device as D
from ._lib import LayerDesc, check, load
from .errors import ConfigError, ShapeError
from .kernels import ACTS, EncodeStats, prepare_books
from .pq import PqConfig, build_table_device, validate_codebooks
from .quant import LookupTableI8, dequantize, quantize_table

F32 = np.float32
PIPELINE_MIN_BYTES = 32 << 20   # numpy inputs above this stream through the native executor
PIPELINE_CHUNK_BYTES = int(os.environ.get("LUTGPU_PIPELINE_CHUNK_MB", "256")) << 20  # per input chunk


class LutLayer:
    """One PQ-replaced linear layer on the GPU.

    Arguments mirror the reference dataclass: cfg, books (C,K,V), weight (D,M)
    or None, bias (M,) (empty = no bias add), qat (also build the int8 twin),
    table / qtable (precomputed), trees (hash encoder).  Extensions: `act`
    ("relu" / "gelu" fused into the epilogue) and `scale_mtile` (per-m-tile
    int8 scales)."""

    GATHERS = ("auto", "cuda", "tensor")

    def __init__(self, cfg: PqConfig, books, weight=None, bias=None, qat: bool = False, table=None,
                 qtable: LookupTableI8 | None = None, trees=None, act=None, scale_mtile: int = 0,
                 device=None, gather: str = "auto", f32_digits: int = 4, scale_per_codebook: bool = False):
        """`gather` picks the lookup engine: "cuda" = CUDA-core kernels (f32
        bitwise ascending-c, int8 exact); "tensor" = tcgen05 one-hot GEMM (int8
        exact; f32 as `f32_digits` int8 digit planes, within the fp32
        contract); "auto" = tensor for int8 (bit-identical either way), cuda
        for f32 (bitwise drop-in)."""
        if gather not in self.GATHERS:
            raise ConfigError(f"gather must be one of {self.GATHERS}, got {gather!r}")
        if f32_digits not in (2, 4):
            raise ConfigError("f32_digits must be 2 or 4")
        self.gather = gather
        self.f32_digits = f32_digits
        self._images = {}
        self.device = torch.device(device) if device is not None else D.require_cuda()
        books = validate_codebooks(books)
        c, k, v = D.shape_of(books)
        if (k, v) != (cfg.k, cfg.v):
            raise ShapeError(f"codebooks {(c, k, v)} inconsistent with config {cfg}")
        if act not in ACTS:
            raise ConfigError(f"unknown activation {act!r}")
        self.cfg = cfg
        self.qat = qat
        self.trees = trees
        self.act = act
        self.scale_mtile = scale_mtile
        self.scale_per_codebook = scale_per_codebook
        self._deq = None
        self.books = D.to_device(books, F32, self.device)
        self.books_prep = prepare_books(self.books)
        self.weight = None
        if weight is not None:
            ws = D.shape_of(weight)
            if len(ws) != 2:
                raise ShapeError(f"weight must be 2-D, got shape {ws}")
            if ws[0] != c * v:
                raise ShapeError(f"weight rows {ws[0]} != C*V = {c * v}")
            self.weight = D.to_device(weight, F32, self.device)
        self.table = None if table is None else D.to_device(table, F32, self.device)
        self.qtable = None
        if qtable is not None:
            self.qtable = LookupTableI8(q=D.to_device(qtable.q, np.int8, self.device),
                                        scale=qtable.scales_tensor(self.device) if isinstance(qtable, LookupTableI8)
                                        else torch.as_tensor(np.asarray(qtable.scale, F32).reshape(-1),
                                                             device=self.device),
                                        scale_mtile=getattr(qtable, "scale_mtile", 0),
                                        validated=isinstance(qtable, LookupTableI8),
                                        per_codebook=getattr(qtable, "per_codebook", False))
        if self.table is None and self.qtable is None:
            self.rebuild()
        m = self.m
        if bias is None:
            self.bias = torch.empty(0, dtype=torch.float32, device=self.device)
        else:
            self.bias = D.to_device(bias, F32, self.device).reshape(-1)
            if self.bias.numel() not in (0, m):
                raise ShapeError(f"bias has {self.bias.numel()} entries, expected {m}")
        self._desc_cache = {}
        self._pipelines = {}

    # ------------------------------------------------------------ properties
    @property
    def c(self) -> int:
        return self.books.shape[0]

    @property
    def k(self) -> int:
        return self.cfg.k

    @property
    def v(self) -> int:
        return self.cfg.v

    @property
    def d(self) -> int:
        return self.c * self.cfg.v

    @property
    def m(self) -> int:
        if self.table is not None:
            return self.table.shape[2]
        return self.qtable.q.shape[2]

    @property
    def has_qtable(self) -> bool:
        return self.qtable is not None

    # ----------------------------------------------------------- table build
    def rebuild(self) -> None:
        """Recompute table (and int8 twin under qat) from weight (softpq.py:125-132)."""
        if self.weight is None:
            if self.table is None and self.qtable is None:
                raise ConfigError("layer has neither a weight matrix nor a table")
            return
        self.table = build_table_device(self.weight, self.books)
        self.qtable = quantize_table(self.table, self.scale_mtile, self.scale_per_codebook) if self.qat else None
        self._deq = None
        self._desc_cache = {}
        self._images = {}
        self.__dict__.pop("_act_twins", None)

    def forward_table(self):
        """Table the training forward reads: dequantized under QAT (softpq.py:134-140)."""
        if self.qat:
            if self.qtable is None:
                self.qtable = quantize_table(self.table, self.scale_mtile, self.scale_per_codebook)
            return dequantize(self.qtable)
        return self.table

    def quantize(self, scale_mtile: int | None = None) -> None:
        """Build (or rebuild) the int8 twin from the f32 table."""
        if scale_mtile is not None:
            self.scale_mtile = scale_mtile
        self.qtable = quantize_table(self.table, self.scale_mtile, self.scale_per_codebook)
        self._deq = None
        self._desc_cache = {}
        for key in [k_ for k_ in self._images if k_ == 1 or isinstance(k_, tuple)]:
            self._images.pop(key)  # images built from the int8 table (or its dequantized twin)
        self.__dict__.pop("_act_twins", None)

    def with_act(self, act) -> "LutLayer":
        """The same device tensors with a different fused epilogue activation
        (a LUT layer followed by Relu runs as one epilogue, model.py:27-35)."""
        if act == self.act:
            return self
        cache = self.__dict__.setdefault("_act_twins", {})
        twin = cache.get(act)
        if twin is None:
            if act not in ACTS:
                raise ConfigError(f"unknown activation {act!r}")
            twin = object.__new__(LutLayer)
            twin.__dict__.update({k: v for k, v in self.__dict__.items() if k != "_act_twins"})
            twin.act = act
            twin._desc_cache = {}
            twin._pipelines = {}  # own executor handles: their finalizer is tied to the twin
            cache[act] = twin
        return twin

    # ---------------------------------------------------------------- ABI
    @property
    def per_codebook_scales(self) -> bool:
        return self.qtable is not None and getattr(self.qtable, "per_codebook", False)

    def dequantized(self) -> torch.Tensor:
        """fl(q * scale) as an f32 (C, K, M) table: the lookup table of the
        per-(codebook, m-tile) scale extension (one f32 product per entry)."""
        if self._deq is None:
            from .quant import dequantized_table

            self._deq = dequantized_table(self.qtable, self.device)
        return self._deq

    def _dequantized_path(self, integer: bool) -> bool:
        """Per-(codebook, m-tile) scales: the integer call sums the dequantized entries."""
        return bool(integer) and self.per_codebook_scales

    def uses_tensor_cores(self, integer: bool) -> bool:
        if self.gather == "cuda":
            return False
        if self._dequantized_path(integer) and self.gather != "tensor":
            # scales differ per codebook: no single exact integer sum to put on the MMA; the
            # default is the bitwise f32 sum, gather="tensor" opts into the digit planes (<= 1e-5)
            return False
        if self.gather == "auto" and not integer:
            return False
        digits = 1 if (integer and not self.per_codebook_scales) else self.f32_digits
        return load().lut_onehot_image_bytes(self.c, self.k, self.m, digits) > 0

    def onehot_image(self, integer: bool) -> torch.Tensor:
        """Swizzled tcgen05 B image of the table (built once, lut_onehot_prepare_*): the int8
        table, or int8 digit planes of the f32 table / of the dequantized per-(codebook,
        m-tile) table."""
        deq = self._dequantized_path(integer)
        digits = 1 if (integer and not deq) else self.f32_digits
        key = ("deq", digits) if deq else digits
        img = self._images.get(key)
        if img is None:
            lib = load()
            nbytes = lib.lut_onehot_image_bytes(self.c, self.k, self.m, digits)
            if nbytes == 0:
                raise ConfigError("shape not supported by the tensor-core gather")
            img = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            if integer and not deq:
                check(lib.lut_onehot_prepare_i8(D.ptr(self.qtable.q), self.c, self.k, self.m, img.data_ptr(),
                                                D.stream_ptr()), "onehot_prepare_i8")
            else:
                src = self.dequantized() if deq else self.table
                err = D.ErrFlag(self.device)
                check(lib.lut_onehot_prepare_f32(D.ptr(src), self.c, self.k, self.m, digits, img.data_ptr(),
                                                 err.p, D.stream_ptr()), "onehot_prepare_f32")
                check(lib.lut_read_status(err.p, D.stream_ptr()), "onehot_prepare_f32")
            self._images[key] = img
        return img

    def desc(self, integer: bool) -> LayerDesc:
        key = bool(integer)
        if key in self._desc_cache:
            return self._desc_cache[key]
        d = LayerDesc()
        d.c, d.k, d.v, d.m = self.c, self.k, self.v, self.m
        d.books_prep = D.ptr(self.books_prep)
        d.table = D.ptr(self.table) if self.table is not None else None
        if self.qtable is not None:
            self._scales_dev = self.qtable.scales_tensor(self.device)
            d.q = D.ptr(self.qtable.q)
            d.scales = D.ptr(self._scales_dev)
            d.scale_mtile = self.qtable.scale_mtile
        d.bias = D.ptr(self.bias)
        d.act = ACTS[self.act]
        d.integer = 1 if integer else 0
        if integer and self.per_codebook_scales:
            # per-(codebook, m-tile) scales: sum the dequantized entries in f32,
            # ascending c (oracle lut_gather_accumulate_cmtile)
            d.table = D.ptr(self.dequantized())
            d.integer = 0
        if self.uses_tensor_cores(integer):
            d.onehot_image = D.ptr(self.onehot_image(integer))
            d.onehot_digits = 1 if (integer and not self.per_codebook_scales) else self.f32_digits
        self._desc_cache[key] = d
        return d

    @property
    def code_stride(self) -> int:
        return int(load().lut_code_stride(self.c))

    def forward_device(self, a_dev: torch.Tensor, integer: bool, out: torch.Tensor | None = None,
                       codes: torch.Tensor | None = None, near: torch.Tensor | None = None) -> torch.Tensor:
        """(N, D) f32 CUDA -> (N, M) f32 CUDA through lut_layer_forward."""
        n = a_dev.shape[0]
        if out is None:
            out = torch.empty((n, self.m), dtype=torch.float32, device=a_dev.device)
        if codes is None:
            codes = torch.empty((n, self.code_stride), dtype=torch.uint8, device=a_dev.device)
        check(load().lut_layer_forward(C.byref(self.desc(integer)), D.ptr(a_dev), n, D.ptr(out), D.ptr(codes),
                                       D.ptr(near), D.stream_ptr()), "lut_layer_infer")
        return out

    def _pipeline(self, chunk_rows: int):
        key = (self.device.index, chunk_rows)
        p = self._pipelines.get(key)
        if p is None:
            handle = C.c_void_p()
            check(load().lut_pipeline_create(self.device.index or 0, chunk_rows, self.d, self.m, self.c,
                                             C.byref(handle)), "lut_pipeline_create")
            p = handle
            self._pipelines[key] = p
            weakref.finalize(self, load().lut_pipeline_destroy, p)
        return p

    def infer(self, a, integer: bool, out=None):
        kind = D.kind_of(a)
        n = D.shape_of(a)[0]
        if kind == D.NUMPY and n * self.d * 4 >= PIPELINE_MIN_BYTES:
            a_h = np.ascontiguousarray(a, dtype=F32)
            if out is None:
                out = np.empty((n, self.m), dtype=F32)
            elif out.shape != (n, self.m) or out.dtype != F32 or not out.flags.c_contiguous:
                raise ShapeError(f"out must be a contiguous f32 array of shape {(n, self.m)}")
            chunk = max(1, min(n, PIPELINE_CHUNK_BYTES // max(1, 4 * max(self.d, self.m))))
            # the descriptor may launch one-time prep work (table image) on torch's
            # stream: build it first, then sync, since the executor runs on its own
            # non-blocking streams
            desc = self.desc(integer)
            pipe = self._pipeline(chunk)
            torch.cuda.current_stream().synchronize()
            near = C.c_int32(0)
            check(load().lut_pipeline_run(pipe, C.byref(desc), a_h.ctypes.data, n, out.ctypes.data, C.byref(near)),
                  "lut_layer_infer")
            EncodeStats.last_near_ties = near.value
            return out
        a_dev = D.to_device(a, F32, self.device)
        res = self.forward_device(a_dev, integer)
        if out is not None and kind == D.NUMPY:
            out[...] = res.cpu().numpy()
            return out
        return D.from_device(res, kind)

    def infer_hash(self, a, integer: bool):
        """encoder="hash": tree-traversal codes, then the same lookup machinery
        (kernels.py:159-164 — swapping the encoder only changes the indices)."""
        from .kernels import _gather_f32, _gather_i8_f32, encode_hash

        kind = D.kind_of(a)
        codes = encode_hash(D.to_device(a, F32, self.device), self.trees)
        act = ACTS[self.act]
        # leaves are data: a code >= K raises CorruptionError like lut_gather_i32 /
        # lut_matmul_ref (kernels.py:117-118, pq.py:209-210), never a clamp
        err = D.ErrFlag(self.device)
        if integer and self.per_codebook_scales:
            out = _gather_f32(codes, self.dequantized(), self.bias, act, self.c, self.k, self.m, err.p)
        elif integer:
            out = _gather_i8_f32(codes, self.qtable.q, self.qtable.scales_tensor(self.device), self.qtable.scale_mtile,
                                 self.bias, act, self.c, self.k, self.m, err.p)
        else:
            out = _gather_f32(codes, self.table, self.bias, act, self.c, self.k, self.m, err.p)
        check(load().lut_read_status(err.p, D.stream_ptr()), "lut_layer_infer")
        return D.from_device(out, kind)


_FOREIGN = weakref.WeakKeyDictionary()   # reference layer -> (fingerprint, device layer)
_FOREIGN_BY_ID: dict[int, tuple] = {}     # layers that cannot be weak-referenced (bounded)
_FOREIGN_BY_ID_MAX = 8


def _content_key(x):
    """Cheap identity of a host array's contents: the reference SGD step
    updates books and bias in place (train.py:162), so those are checksummed;
    tables are rebuilt as new objects (softpq.py:125-132), so identity suffices."""
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return ("t", x.data_ptr(), x._version, tuple(x.shape))
    a = np.ascontiguousarray(x)
    return ("a", a.dtype.str, a.shape, zlib.crc32(a.view(np.uint8).reshape(-1)))


def _fingerprint(layer) -> tuple:
    qt = getattr(layer, "qtable", None)
    return (_content_key(layer.books), _content_key(layer.bias), _sample_key(getattr(layer, "table", None)),
            None if qt is None else (_sample_key(qt.q), float(np.asarray(qt.scale).reshape(-1)[0])))


def _sample_key(x):
    """Object identity plus a checksum of ~4096 strided entries (a table that
    was replaced by a new object of the same id still changes the key)."""
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return _content_key(x)
    a = np.asarray(x).reshape(-1)
    step = max(1, a.size // 4096)
    return (id(x), a.dtype.str, a.size, zlib.crc32(np.ascontiguousarray(a[::step]).view(np.uint8)))


def as_device_layer(layer) -> LutLayer:
    """Our LutLayer as is; a reference-style layer is converted once and the
    device copy reused while its books / bias contents and its table objects
    are unchanged (an in-place update of books or bias re-converts).  The cache
    holds the reference layer weakly, so dropping it frees the HBM tables."""
    if isinstance(layer, LutLayer):
        return layer
    fp = _fingerprint(layer)
    try:
        hit = _FOREIGN.get(layer)
        weak = True
    except TypeError:
        hit = _FOREIGN_BY_ID.get(id(layer))
        weak = False
    if hit is not None and hit[0] == fp:
        return hit[1]
    qt = getattr(layer, "qtable", None)
    if qt is not None and not isinstance(qt, LookupTableI8):
        qt = LookupTableI8(q=np.asarray(qt.q), scale=F32(qt.scale))
    cfg = layer.cfg if isinstance(getattr(layer, "cfg", None), PqConfig) else PqConfig(
        v=int(layer.cfg.v), k=int(layer.cfg.k))
    dl = LutLayer(cfg=cfg, books=layer.books, weight=None, bias=layer.bias, table=getattr(layer, "table", None),
                  qtable=qt, trees=getattr(layer, "trees", None))
    if weak:
        _FOREIGN[layer] = (fp, dl)
    else:
        if len(_FOREIGN_BY_ID) >= _FOREIGN_BY_ID_MAX:
            _FOREIGN_BY_ID.pop(next(iter(_FOREIGN_BY_ID)))
        _FOREIGN_BY_ID[id(layer)] = (fp, dl)
    return dl
