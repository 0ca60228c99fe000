"""Device plumbing: move operands to the GPU, hand raw pointers and the
current torch stream to the C ABI, and return results in the caller's kind
(numpy in -> numpy out, the reference's contract; torch CUDA in -> torch
CUDA out, no copies)."""

from __future__ import annotations

import numpy as np
import torch

from .errors import DeviceError

NUMPY, TORCH_CPU, TORCH_CUDA = "numpy", "torch_cpu", "torch_cuda"


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the LUT path runs only on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def kind_of(x) -> str:
    if isinstance(x, torch.Tensor):
        return TORCH_CUDA if x.is_cuda else TORCH_CPU
    return NUMPY


def shape_of(x) -> tuple:
    return tuple(x.shape) if hasattr(x, "shape") else tuple(np.asarray(x).shape)


_NP2T = {np.float32: torch.float32, np.uint8: torch.uint8, np.int8: torch.int8, np.int32: torch.int32,
         np.int64: torch.int64, np.float64: torch.float64}


def to_device(x, np_dtype, device: torch.device | None = None) -> torch.Tensor:
    """Contiguous CUDA tensor of dtype `np_dtype` (cast like np.ascontiguousarray)."""
    device = device or require_cuda()
    tdt = _NP2T[np.dtype(np_dtype).type]
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=tdt, non_blocking=True)
        return t.contiguous()
    arr = np.ascontiguousarray(x, dtype=np_dtype)
    # a plain pageable copy: pinning a fresh host buffer per call (cudaHostAlloc +
    # a host memcpy) costs more than it saves for a one-shot transfer; large
    # numpy layer inputs stream through the native executor's pinned chunks
    return torch.from_numpy(arr).to(device, non_blocking=False)


def from_device(t: torch.Tensor, kind: str):
    if kind == TORCH_CUDA:
        return t
    if kind == TORCH_CPU:
        return t.cpu()
    return t.cpu().numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None or t.numel() == 0:
        return None
    return t.data_ptr()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class ErrFlag:
    """A device int32 the kernels raise data errors into (lut_read_status)."""

    def __init__(self, device):
        self.t = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def p(self) -> int:
        return self.t.data_ptr()
