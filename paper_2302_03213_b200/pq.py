"""PQ semantics on the GPU — mirror of the hot-path half of lutkit/pq.py.

encode_hard / lut_matmul_ref / build_table / pq_amm keep the reference
names and contracts (pq.py:25-231); k-means centroid learning is out of scope
(offline training)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import check, load
from .errors import ConfigError, ShapeError
from .kernels import MAX_CENTROIDS, centroid_search_fast, lut_gather_f32

F32 = np.float32


@dataclass(frozen=True)
class PqConfig:
    """Quantization geometry (pq.py:25-41): sub-vector length v, centroids k."""

    v: int
    k: int

    def __post_init__(self) -> None:
        if self.v < 1:
            raise ConfigError(f"sub-vector length must be >= 1, got {self.v}")
        if not 1 <= self.k <= MAX_CENTROIDS:
            raise ConfigError(f"centroid count must be in [1, {MAX_CENTROIDS}], got {self.k}")

    def codebook_count(self, d: int) -> int:
        if d % self.v != 0:
            raise ConfigError(f"dimension {d} not divisible by sub-vector length {self.v}")
        return d // self.v


def validate_codebooks(books):
    shp = D.shape_of(books)
    if len(shp) != 3:
        raise ShapeError(f"codebooks must have shape (C, K, V), got {shp}")
    if shp[1] > MAX_CENTROIDS:
        raise ConfigError(f"K={shp[1]} exceeds the u8 encoding limit {MAX_CENTROIDS}")
    if isinstance(books, torch.Tensor):
        return books.float().contiguous()
    return np.ascontiguousarray(books, dtype=F32)


def encode_hard(a, books):
    """Nearest-centroid indices, ties to the lowest k (pq.py:171-174).  The GPU
    encode is exact (fp64 near-tie re-decision), so this is the same kernel."""
    return centroid_search_fast(a, books)


def build_table_device(b_dev: torch.Tensor, books_dev: torch.Tensor) -> torch.Tensor:
    c, k, v = books_dev.shape
    m = b_dev.shape[1]
    table = torch.empty((c, k, m), dtype=torch.float32, device=b_dev.device)
    check(load().lut_build_table_f32(D.ptr(b_dev), m, D.ptr(books_dev), c, k, v, D.ptr(table), D.stream_ptr()),
          "build_table")
    return table


def build_table(b, books):
    """(C, K, M) table, T[c,k,m] = sum_j P[c,k,j] B[cV+j,m], f32 multiply then
    f32 add, j ascending — bitwise equal to pq.py:177-193."""
    bshape = D.shape_of(b)
    if len(bshape) != 2:
        raise ShapeError(f"b must be 2-D, got shape {bshape}")
    books = validate_codebooks(books)
    c, k, v = D.shape_of(books)
    if bshape[0] != c * v:
        raise ShapeError(f"weight rows {bshape[0]} != C*V = {c}*{v}")
    kind = D.kind_of(b)
    dev = D.require_cuda()
    table = build_table_device(D.to_device(b, F32, dev), D.to_device(books, F32, dev))
    return D.from_device(table, kind)


def lut_matmul_ref(enc, table):
    """out[n] = sum_c T[c, enc[n,c]] in ascending-c f32 (pq.py:196-214)."""
    return lut_gather_f32(enc, table)


def pq_amm(a, b, cfg: PqConfig, books):
    """Encode A, build the table for B, aggregate (pq.py:217-231)."""
    ashape, bshape = D.shape_of(a), D.shape_of(b)
    if len(ashape) != 2 or len(bshape) != 2:
        raise ShapeError("a and b must be 2-D")
    books = validate_codebooks(books)
    c_books = cfg.codebook_count(ashape[1])
    if ashape[1] != bshape[0]:
        raise ShapeError(f"inner dims differ: {ashape} x {bshape}")
    bs = D.shape_of(books)
    if bs[0] != c_books or bs[1] != cfg.k or bs[2] != cfg.v:
        raise ShapeError(f"codebooks {bs} inconsistent with config (C={c_books}, K={cfg.k}, V={cfg.v})")
    return lut_matmul_ref(encode_hard(a, books), build_table(b, books))
