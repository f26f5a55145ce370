"""View-sharded data parallelism.

Every rank holds the full plane set; slot k of a step's view list goes to rank
k mod N (the epoch-shuffled order of optimizer.cpp:49-59 is identical on all
ranks); each rank runs the fused step on its views with view_scale = 1/V_step
and the plane gradients (+ loss) are summed with one NCCL all-reduce over
NVLink (psg_allreduce_grads). Sum-then-project equals project-then-sum because
the tangent projection (renderer.cpp:518-520) is linear, so every rank then
applies psg_finalize_grads and holds the reference's Optimizer::step gradient.

torch.distributed is plumbing only: it carries the 128-byte NCCL unique id.
"""
from __future__ import annotations

import numpy as np


def shard_views(view_ids, world: int, rank: int) -> np.ndarray:
    """Slot k -> rank k mod world (cost-balanced enough for uniform views)."""
    ids = np.asarray(view_ids, dtype=np.int32)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_views: bad rank/world")
    return ids[rank::world]


def nccl_bootstrap(batch, rank: int, world: int) -> None:
    """Create the NCCL communicator of `batch` (a ViewBatch) for this rank."""
    import torch.distributed as dist

    from .renderer import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    batch.comm_init(obj[0], world, rank)
