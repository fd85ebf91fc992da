"""Host-side plumbing of the data-parallel path.

Images are independent: rank r of P owns the contiguous shard
``[r*N/P, (r+1)*N/P)``; weights and shared operator data are replicated. The only
exchange is the GLOBAL_MAX stop rule (BASELINE C5): every ``check_every`` iterations the
max residual over the active images of all ranks is all-reduced (NCCL MAX inside the
library's iteration graph) and every rank takes the same stop decision. torch.distributed
is used only to bootstrap: rank 0 draws the ncclUniqueId and broadcasts it.
"""
from __future__ import annotations

import os


def shard(n_images: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of image indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_images, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId through the C ABI (ideq_get_nccl_id) and broadcasts it over
    the initialised torch.distributed process group; returns the 128 bytes on every rank."""
    import torch.distributed as dist
    obj = [None]
    if dist.get_rank() == 0:
        from . import ideq
        obj[0] = ideq.nccl_unique_id()
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def global_stop(local_rmax: float, tol: float, all_reduce_max) -> bool:
    """The GLOBAL_MAX decision given this rank's max residual over its active images (-1 if none):
    stop iff the max over all ranks is a real residual (>= 0) and <= tol. `all_reduce_max` is the
    collective (NCCL on the GPU path, gloo in the CPU tests)."""
    m = all_reduce_max(local_rmax)
    return 0.0 <= m <= tol
