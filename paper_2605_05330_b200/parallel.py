"""Multi-GPU plumbing: one process per GPU, torch.distributed.

* Batches (C4): independent graphs, rank r takes its own contiguous slice of
  the family -- no collective touches the data path; results are gathered on
  request only.
* One graph too large for one GPU (C5): vertex-range partitions with a halo
  exchange of the published values every iteration (partition.py).
* Everything else: replicas.
"""

from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of `total` independent units."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)
