"""Head sharding across the GPUs of one node.

Every (b, h) head is independent (reference tiled.cpp:146-147), so rank r of N
owns heads [h0, h1) of every batch as its own contiguous [B, h1-h0, S, D]
buffers and calls the same C-ABI entry with H := h1 - h0.  No collective runs
on the data path; `gather_heads` (an all-gather over NCCL/NVLink, or gloo in
CPU tests) is the optional post-hoc step for consumers that want the whole O
on every rank, and `max_over_ranks` is the timing reduction the bench uses.
"""
from __future__ import annotations


def head_range(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal split of H heads over `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if H < 1:
        raise ValueError("H must be >= 1")
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def shard_heads(x, world: int, rank: int):
    """Rank-local contiguous copy of x[:, h0:h1] for x of shape [B, H, S, D]."""
    h0, h1 = head_range(x.shape[1], world, rank)
    return x[:, h0:h1].contiguous()


def gather_heads(local, world: int, group=None):
    """All-gather rank-local [B, h, S, D] shards back into [B, H, S, D]
    (shards must be equal-sized, i.e. H % world == 0)."""
    import torch
    import torch.distributed as dist
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=1)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device time) over the group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
