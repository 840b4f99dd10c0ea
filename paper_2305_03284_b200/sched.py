"""Stream scheduler: shards independent sensor streams over the GPUs of one
box (north_star "(4) a stream scheduler that shards independent
sensor streams across the 8 GPUs of one box while each stream's timesteps stay
sequential on one device, so no per-step collective is needed").

One process per GPU (torchrun); rank g owns the contiguous stream block
[first, first + count) and one ddh_ctx.  The only cross-rank traffic is
host-side bookkeeping outside the hot loop: barriers around timed regions,
the max over ranks of a device time, and gathers of per-stream scalars
(e.g. Strehl series).  There is no data-path collective: streams never
exchange data (Fig. 1's recurrence is per stream).
"""
from __future__ import annotations

import os
from typing import List, Tuple


def shard(total_streams: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of streams for `rank`: stream s goes to rank
    floor(s * world / total).  Returns (first, count)."""
    if world < 1 or not (0 <= rank < world) or total_streams < 0:
        raise ValueError("bad shard arguments")
    first = -(-rank * total_streams // world)
    last = -(-(rank + 1) * total_streams // world)
    return first, last - first


def env_rank() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str):
    """Initialise torch.distributed when WORLD_SIZE > 1 (rendezvous from env)."""
    import torch.distributed as dist
    world, rank, local = env_rank()
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Maximum of a scalar over ranks (timings: the job is as slow as its
    slowest GPU)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_per_stream(values: List[float], first: int, total: int) -> List[float]:
    """Gather per-stream scalars of every rank's block into one list indexed
    by global stream id (all ranks receive it)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return list(values)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (first, list(values)))
    out = [float("nan")] * total
    for f, vals in parts:
        for k, v in enumerate(vals):
            out[f + k] = v
    return out
