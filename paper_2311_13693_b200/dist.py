"""Mode-3 slab sharding across ranks (SURVEY §8 e).

Eq. 3 is linear in X, so rank g compresses only k in [k0, k1) of the tensor
into partial replicas (every rank regenerates the same ensemble from the seed
— the RNG is counter based, no communication) and one reduction (sum) over
the ranks yields the replicas. On GPUs the reduction is NCCL over NVLink
(torch.distributed backend "nccl"); the same code runs on "gloo" for tests.
"""
from __future__ import annotations


def slab_range(K: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous mode-3 slab [k0, k1) of rank `rank` out of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("slab_range: bad rank/world")
    base, extra = divmod(K, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def compress_sharded(local_compress, K: int, y, dst: int = 0, group=None):
    """Run ``local_compress(k0, k1, y)`` on this rank's slab, then sum-reduce y to ``dst``.

    ``local_compress`` writes (not accumulates) the rank's partial replicas into
    ``y`` (a torch tensor on the backend's device). Returns y (complete on dst).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = slab_range(K, rank, world)
    if k1 > k0:
        local_compress(k0, k1, y)
    else:
        y.zero_()
    if world > 1:
        dist.reduce(y, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return y
