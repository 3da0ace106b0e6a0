"""Query sharding across ranks: the index is replicated per
GPU, a batch is split into contiguous shards with the same bounds the C ABI
uses across the GPUs of one handle (pag_host.cpp, pag_gpu_search), results
come back by plain copy — no collective on the data path. The only
collectives are control-plane: the operating point broadcast from rank 0 and
the max-over-ranks step time."""
from __future__ import annotations

from typing import Tuple


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[q0, q1) of rank `rank` out of `world` for an n-query batch."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def broadcast_int(x: int, dist=None, device=None) -> int:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return int(x)
    import torch
    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.broadcast(t, 0)
    return int(t.item())


def max_over_ranks(x: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
