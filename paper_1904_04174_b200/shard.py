"""Batch-shard host logic for N ranks.

Images are independent, so rank r of `world` owns the contiguous global images
[r*B/world, (r+1)*B/world).  Nothing is exchanged on the data path; the collectives below are
off the timed path: a broadcast of rank 0's per-layer algorithm choices (so every rank runs
the same kernels) and a MAX reduction of per-rank device times (value = total work / max time).
Backend-agnostic: used with NCCL by bench.py and with gloo by tests/test_shard_gloo.py.
"""
from __future__ import annotations


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) images of `rank`; requires global_batch % world == 0 (uniform per-GPU work)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by {world} ranks")
    per = global_batch // world
    return rank * per, (rank + 1) * per


def broadcast_choices(choices: dict, dist, device) -> dict:
    """Rank 0's {layer name: algo id} wins on every rank (sorted-key order is the wire format)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(choices)
    names = sorted(choices)
    t = torch.tensor([int(choices[k]) for k in names], dtype=torch.int32, device=device)
    dist.broadcast(t, 0)
    return dict(zip(names, (int(v) for v in t.tolist())))


def max_over_ranks(value: float, dist, device) -> float:
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_shards(local, dist):
    """Concatenate every rank's output slice along the batch dim (verification only)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.contiguous())
    return torch.cat(parts, dim=0)
