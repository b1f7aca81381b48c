"""Replica-level multi-GPU plumbing.

The hot path has no data exchange: batched evaluation rows and independent runs share nothing, so
``north_star``'s single-GPU path scales out as replicas (weak scaling).  One process per GPU;
torch.distributed (NCCL on GPUs, gloo on CPU for the tests) carries only the barrier, the
max-over-ranks step time and — for the batched-runs layer — the ordered gather of per-run results.
No collective touches the data path.
"""
from __future__ import annotations

import os


def env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced partition [start, stop) of n_items over `world` ranks (the first
    n_items % world ranks take one extra).  Every item is owned by exactly one rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard: bad rank / world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def init(backend: str | None = None, device=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns the dist module or None."""
    rank, world, _ = env()
    if world <= 1:
        return None
    import torch.distributed as dist

    if not dist.is_initialized():
        if backend is None:
            import torch

            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return dist


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """The step time the driver reports: the slowest rank's."""
    if dist is None:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_ordered(local: list, n_items: int, dist=None) -> list:
    """Concatenate each rank's shard results in global item order (rank r holds shard(r))."""
    if dist is None:
        return list(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(local))
    out = [x for p in parts for x in p]
    if len(out) != n_items:
        raise RuntimeError("gather_ordered: shard sizes do not cover the items")
    return out
