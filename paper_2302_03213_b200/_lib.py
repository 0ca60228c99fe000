"""ctypes binding of the native library (include/lutgpu.h).

There is no CPU fallback: if `_lib/liblutgpu.so` is missing or cannot be
loaded, every compute entry point raises.  Loading the library itself does
not need a GPU (the CPU test suite checks the exported symbols)."""

from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS_EXC, DeviceError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "liblutgpu.so")

c_int32_p = C.POINTER(C.c_int32)


class LayerDesc(C.Structure):
    """Mirror of `lut_layer_desc` (include/lutgpu.h)."""

    _fields_ = [
        ("c", C.c_int32), ("k", C.c_int32), ("v", C.c_int32), ("m", C.c_int32),
        ("books_prep", C.c_void_p),
        ("table", C.c_void_p),
        ("q", C.c_void_p),
        ("scales", C.c_void_p),
        ("scale_mtile", C.c_int32),
        ("bias", C.c_void_p),
        ("act", C.c_int32),
        ("integer", C.c_int32),
        ("onehot_image", C.c_void_p),
        ("onehot_digits", C.c_int32),
    ]


# name -> (restype, argtypes); pointers are passed as integers (c_void_p)
P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
SIGNATURES = {
    "lut_version": (C.c_int, []),
    "lut_last_error": (C.c_char_p, []),
    "lut_books_prep_bytes": (C.c_size_t, [I32, I32, I32]),
    "lut_prepare_books": (C.c_int, [P, I32, I32, I32, P, P]),
    "lut_encode_f32": (C.c_int, [P, I64, I32, P, I32, I32, I32, P, I32, I64, P, P]),
    "lut_encode_conv_f32": (C.c_int, [P, I32, I32, I32, I32, I32, I32, I32, I32, P, I32, I32, I32, P, I32, P, P]),
    "lut_im2col_f32": (C.c_int, [P, I32, I32, I32, I32, I32, I32, I32, I32, P, P]),
    "lut_encode_hash": (C.c_int, [P, I64, I32, P, P, P, I32, I32, I32, P, I64, P]),
    "lut_gather_f32": (C.c_int, [P, I32, I64, I32, I32, I32, P, P, I32, P, I64, P, P]),
    "lut_gather_i8": (C.c_int, [P, I32, I64, I32, I32, I32, P, P, I32, P, I32, P, P, I64, P, P]),
    "lut_build_table_f32": (C.c_int, [P, I32, P, I32, I32, I32, P, P]),
    "lut_matmul_ref_f32": (C.c_int, [P, P, I64, I32, I32, P, P]),
    "lut_quantize_scratch_bytes": (C.c_size_t, [I32, I32, I32, I32]),
    "lut_quantize_table": (C.c_int, [P, I32, I32, I32, I32, P, P, P, P, P]),
    "lut_read_status": (C.c_int, [P, P]),
    "lut_onehot_image_bytes": (C.c_size_t, [I32, I32, I32, I32]),
    "lut_onehot_prepare_i8": (C.c_int, [P, I32, I32, I32, P, P]),
    "lut_onehot_prepare_f32": (C.c_int, [P, I32, I32, I32, I32, P, P, P]),
    "lut_gather_onehot": (C.c_int, [P, I64, I64, I32, I32, I32, I32, P, P, I32, P, I32, P, P, I64, P]),
    "lut_code_stride": (I64, [I32]),
    "lut_conv_layer_forward": (C.c_int, [C.POINTER(LayerDesc), P, I32, I32, I32, I32, I32, I32, I32, I32, P, P, P, P]),
    "lut_layer_forward": (C.c_int, [C.POINTER(LayerDesc), P, I64, P, P, P, P]),
    "lut_pipeline_create": (C.c_int, [I32, I64, I32, I32, I32, C.POINTER(C.c_void_p)]),
    "lut_pipeline_run": (C.c_int, [P, C.POINTER(LayerDesc), P, I64, P, c_int32_p]),
    "lut_pipeline_destroy": (C.c_int, [P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("LUTGPU_LIB", path)  # A/B builds (tools/ab_lib.sh): another in-tree .so
    if not os.path.exists(path):
        raise ImportError(
            f"native library missing: {path} — run `python -m paper_2302_03213_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols(path: str = LIB_PATH) -> list[str]:
    lib = C.CDLL(path)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(status: int, what: str = "") -> None:
    """Map a lutgpu status to the reference's exception classes."""
    if status == 0:
        return
    msg = load().lut_last_error().decode(errors="replace")
    exc = STATUS_EXC.get(status, DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)
