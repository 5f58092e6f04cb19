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


def decompose_sharded(compress_slab, K: int, y, decompose_replicas, dst: int = 0, group=None):
    """The multi-GPU pipeline (SURVEY §8 e): every rank compresses its mode-3
    slab into partial replicas (``compress_slab(k0, k1, y)``), one sum-reduce
    lands the P replicas on ``dst``, and ``dst`` runs the decomposition,
    alignment and recovery stages on them (``decompose_replicas(y) ->
    (factors, metrics)``; the ALS batch fills one GPU: one CTA per replica).
    The recovered factor triple (three small fp64 matrices) is broadcast back,
    so every rank returns the same factors; metrics only on ``dst``.
    """
    import torch
    import torch.distributed as dist

    compress_sharded(compress_slab, K, y, dst=dst, group=group)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    factors, metrics = (None, None)
    if rank == dst:
        factors, metrics = decompose_replicas(y)
    if world > 1:
        shapes = [list(f.shape) for f in factors] if rank == dst else None
        box = [shapes]
        dist.broadcast_object_list(box, src=dst, group=group)
        out = []
        for m, shp in enumerate(box[0]):
            t = (torch.from_numpy(factors[m].ravel(order="F")).to(y.device) if rank == dst
                 else torch.zeros(shp[0] * shp[1], dtype=torch.float64, device=y.device))
            dist.broadcast(t, src=dst, group=group)
            out.append(t.cpu().numpy().reshape(shp, order="F"))
        factors = tuple(out)
    return factors, metrics


def replica_range(P: int, rank: int, world: int) -> tuple[int, int]:
    """Replicas [p0, p1) that rank `rank` decomposes after the reduce-scatter
    (contiguous blocks of ceil(P / world))."""
    per = -(-P // world)
    p0 = min(P, rank * per)
    return p0, min(P, p0 + per)


def decompose_distributed(compress_slab, K: int, P: int, lmn: int, y, stage1, finish, dst: int = 0, group=None):
    """The multi-GPU pipeline with the per-replica CP-ALS spread over ranks
    (SURVEY §8 e): every rank compresses its mode-3 slab into partial
    replicas (``compress_slab(k0, k1, y)``, y holding ceil(P/G)*G replicas of
    ``lmn`` values); one reduce-scatter (NCCL; all-reduce + slice on gloo)
    leaves rank g the complete replicas [g*ceil(P/G), ...); each rank runs
    stage 1 on them (``stage1(local_replicas, ids) -> Stage1Result``); the
    small per-replica results (factors, fit error, convergence, sweeps) are
    gathered on ``dst``, which runs the survivor rule, alignment and recovery
    (``finish(merged) -> (factors, metrics)``); the recovered factors are
    broadcast. Returns (factors, metrics or None, local stage-1 seconds)."""
    import time

    import numpy as np
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    per = -(-P // world)
    k0, k1 = slab_range(K, rank, world)
    if k1 > k0:
        compress_slab(k0, k1, y)
    else:
        y.zero_()
    mine = y.narrow(0, rank * per * lmn, per * lmn)
    if world > 1:
        if dist.get_backend(group) == "nccl":
            out = torch.empty_like(mine)
            dist.reduce_scatter_tensor(out, y.narrow(0, 0, per * world * lmn), op=dist.ReduceOp.SUM, group=group)
            mine = out
        else:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
            mine = y.narrow(0, rank * per * lmn, per * lmn)
    p0, p1 = replica_range(P, rank, world)
    t0 = time.perf_counter()
    res = stage1(mine.narrow(0, 0, (p1 - p0) * lmn), np.arange(p0, p1, dtype=np.int64)) if p1 > p0 else None
    t_s1 = time.perf_counter() - t0
    if world > 1:
        parts = [None] * world if rank == dst else None
        dist.gather_object(res, parts, dst=dst, group=group)
    else:
        parts = [res]
    factors, metrics = (None, None)
    if rank == dst:
        from .api import Stage1Result
        parts = [r for r in parts if r is not None]
        merged = Stage1Result(*(np.concatenate([getattr(r, f) for r in parts])
                                for f in ("ids", "factors", "fit_err", "converged", "sweeps")))
        factors, metrics = finish(merged)
    if world > 1:
        box = [[list(f.shape) for f in factors] if rank == dst else None]
        dist.broadcast_object_list(box, src=dst, group=group)
        dev = y.device
        out = []
        for m, shp in enumerate(box[0]):
            t = (torch.from_numpy(np.asfortranarray(factors[m]).ravel(order="F")).to(dev) if rank == dst
                 else torch.zeros(shp[0] * shp[1], dtype=torch.float64, device=dev))
            dist.broadcast(t, src=dst, group=group)
            out.append(t.cpu().numpy().reshape(shp, order="F"))
        factors = tuple(out)
    return factors, metrics, t_s1
