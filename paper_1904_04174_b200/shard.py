"""Batch-shard host logic for N ranks.

Images are independent, so rank r of `world` owns the contiguous global images
[r*B/world, (r+1)*B/world).  Nothing is exchanged on the data path; the collectives below are
off the timed path: a broadcast of rank 0's per-layer algorithm choices and tuned variants (so every
rank runs the same kernels) and a MAX reduction of per-rank device times (value = total work / max time).
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
    """Rank 0's {layer name: choice} wins on every rank; a choice is an int (algorithm id) or a tuple
    of ints (algorithm id, tuned parameter variant).  Wire format: one int32 row per sorted key."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(choices)
    names = sorted(choices)
    rows = [tuple(v) if isinstance(v, (tuple, list)) else (int(v),) for v in (choices[k] for k in names)]
    width = len(rows[0]) if rows else 1
    if any(len(r) != width for r in rows):
        raise ValueError("choices must all have the same arity")
    t = torch.tensor(rows, dtype=torch.int32, device=device).reshape(len(names), width)
    dist.broadcast(t, 0)
    vals = [tuple(int(x) for x in r) for r in t.tolist()]
    return dict(zip(names, (v if width > 1 else v[0] for v in vals)))


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
