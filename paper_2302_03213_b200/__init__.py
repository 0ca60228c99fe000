"""B200-native LUT-layer inference (LUT-NN, arXiv 2302.03213).

Drop-in for the hot path of the reference package `lutkit`: the same public
names (lutkit/__init__.py:17-57 and lutkit.kernels.*) backed by hand-written
sm_100a kernels behind the C ABI in include/lutgpu.h.  Encode (nearest
centroid, exact indices), lookup-aggregate (f32 bitwise / int8 exact), table
build and int8 quantization, im2col-fused conv layers, a host-memory
executor and row-sharded multi-GPU helpers.  No CPU fallback."""

from .errors import (
    ConfigError,
    ContainerError,
    CorruptionError,
    DataError,
    DeviceError,
    DivergenceError,
    LutKitError,
    ShapeError,
)
from .kernels import (
    MAX_GROUP,
    BenchReport,
    EncodeStats,
    KernelPlan,
    bench_kernel,
    centroid_search_fast,
    encode_hash,
    flop_counter,
    lut_gather_accumulate,
    lut_gather_f32,
    lut_gather_i32,
    lut_layer_infer,
)
from .quant import QMAX, LookupTableI8, dequantize, quantize_table
from .pq import PqConfig, build_table, encode_hard, lut_matmul_ref, pq_amm, validate_codebooks
from .tensor import as_matrix, im2col, matmul_ref, split_subvectors
from .rng import child_rng, make_rng
from .layer import LutLayer, as_device_layer
from .nn import Conv, Dense, LutConv, LutConv2d, LutDense, LutLinear, Model, Relu, predict_fast
from .container import load_model, model_bytes, model_from_bytes, save_model

__version__ = "0.1.0"
