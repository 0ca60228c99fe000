"""Row sharding across the GPUs of one box.

Rows (tokens / output pixels) are independent: each output row depends only
on its input row, the codebooks and the table (lutkit/kernels.py:78-86,
pq.py:212-213).  So the multi-GPU path is data parallel over rows with the
layer replicated on every rank and NO collective on the compute path.  The
only exchange is optional: `gather_rows` all-gathers the row-sharded
outputs (NCCL over NVLink on GPUs; gloo on CPU for the host-logic tests)
when the caller asks for the full tensor on every rank."""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [start, stop) of n rows for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(n: int, world: int) -> list[int]:
    return [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]


def gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather row shards (uneven allowed) into the full (n_total, ...) tensor."""
    if local.is_cuda and dist.get_backend(group) == "gloo":  # gloo moves host tensors only
        return gather_rows(local.cpu(), n_total, group).to(local.device)
    world = dist.get_world_size(group)
    sizes = shard_sizes(n_total, world)
    rank = dist.get_rank(group)
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, expected {sizes[rank]}")
    maxr = max(sizes) if sizes else 0
    tail = tuple(local.shape[1:])
    padded = local.new_zeros((maxr,) + tail)
    padded[: local.shape[0]] = local
    full = local.new_empty((world * maxr,) + tail)
    dist.all_gather_into_tensor(full, padded, group=group)
    parts = [full[r * maxr: r * maxr + sizes[r]] for r in range(world)]
    return torch.cat(parts, dim=0)


def sharded_forward(a_local: torch.Tensor, layer, integer: bool, n_total: int | None = None,
                    gather: bool = False, group=None) -> torch.Tensor:
    """Run this rank's rows through the layer; optionally all-gather outputs."""
    out = layer.forward_device(a_local, integer)
    if not gather:
        return out
    if n_total is None:
        t = torch.tensor([a_local.shape[0]], device=a_local.device)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())
    return gather_rows(out, n_total, group)
