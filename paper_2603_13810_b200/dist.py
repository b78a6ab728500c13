"""Data-parallel plumbing: contiguous batch shards per rank and the one collective
of the path (gather of final-layer packed spikes and spike counts after the
forward, north_star "NCCL used only to gather outputs and spike
counts").  Compute never crosses ranks: samples are independent.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(B: int, world: int, rank: int):
    """[b0, b0 + n) of rank `rank` for a global batch B split contiguously."""
    if B % world:
        raise ValueError(f"global batch {B} not divisible by world size {world}")
    n = B // world
    return rank * n, n


def gather_batch(x: torch.Tensor, dim: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather shards along `dim` (the batch axis) into the full tensor.
    Uses all_gather_into_tensor (one NCCL call) on contiguous buffers; the shard axis
    is moved to the front so the gathered buffer is rank-major and contiguous."""
    world = dist.get_world_size()
    xs = x.movedim(dim, 0).contiguous()
    if out is None:
        out = torch.empty((world * xs.shape[0],) + tuple(xs.shape[1:]), dtype=xs.dtype,
                          device=xs.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, xs)
    else:  # gloo (CPU tests)
        parts = list(out.chunk(world, 0))
        dist.all_gather(parts, xs)
    return out.movedim(0, dim)
