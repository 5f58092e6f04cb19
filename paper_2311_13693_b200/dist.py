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


class RemoteStageError(RuntimeError):
    """A stage failed on another rank; every rank raises this (or the
    original exception on the failing rank) instead of blocking in the next
    collective."""


def _broadcast_outcome(rank, dst, group, shapes=None, error=None):
    """dst tells every rank whether its stage succeeded (and the factor
    shapes) before any tensor collective; returns the shapes or raises."""
    import torch.distributed as dist

    box = [(shapes, error)] if rank == dst else [None]
    dist.broadcast_object_list(box, src=dst, group=group)
    shapes, error = box[0]
    if error is not None:
        raise RemoteStageError(error)
    return shapes


def _broadcast_factors(factors, shapes, rank, dst, group, device):
    import numpy as np
    import torch
    import torch.distributed as dist

    out = []
    for m, shp in enumerate(shapes):
        t = (torch.from_numpy(np.asfortranarray(factors[m]).ravel(order="F")).to(device) if rank == dst
             else torch.zeros(shp[0] * shp[1], dtype=torch.float64, device=device))
        dist.broadcast(t, src=dst, group=group)
        out.append(t.cpu().numpy().reshape(shp, order="F"))
    return tuple(out)


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


def coo_share(nnz: int, rank: int, world: int) -> tuple[int, int]:
    """Nonzeros [e0, e1) of rank `rank` for COO input: contiguous ranges, as
    xtsg_multi_compress_coo splits them across the GPUs of one process (a
    k-range when the stream is k-sorted). Eq. 3 is linear in the nonzeros,
    so the partials of any partition sum to the whole."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("coo_share: bad rank/world")
    return nnz * rank // world, nnz * (rank + 1) // world


def csf_shares(slice_ptr, fiber_ptr, world: int) -> list[int]:
    """Slice boundaries q_0 = 0 <= ... <= q_world = n_slices: rank g takes the
    slices [q_g, q_g+1) holding ~1/world of the nonzeros (a k-range for
    k-sorted slices) — the split xtsg_multi_compress_csf makes
    (csrc/multi.cu, CsfIndex::lower)."""
    import numpy as np

    slice_ptr, fiber_ptr = np.asarray(slice_ptr, np.int64), np.asarray(fiber_ptr, np.int64)
    n_slices, n_fibers, nnz = len(slice_ptr) - 1, len(fiber_ptr) - 1, int(fiber_ptr[-1]) if len(fiber_ptr) else 0
    start = fiber_ptr[np.clip(slice_ptr, 0, n_fibers)].clip(0, max(nnz, 0))
    qs = [0] * (world + 1)
    qs[world] = n_slices
    if n_slices > 0:
        e0, e1 = int(start[0]), max(int(start[0]), int(start[-1]))
        for g in range(1, world):
            target = e0 + (e1 - e0) * g // world
            qs[g] = max(qs[g - 1], min(n_slices, int(np.searchsorted(start, target, side="left"))))
    return qs


def csf_part(csf, q0: int, q1: int):
    """Slices [q0, q1) of a CSF tuple (slice_k, slice_ptr, fiber_j, fiber_ptr,
    nz_i, val) as a CSF of their own, pointers rebased to 0."""
    slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val = csf
    f0, f1 = int(slice_ptr[q0]), int(slice_ptr[q1])
    e0, e1 = int(fiber_ptr[f0]), int(fiber_ptr[f1])
    return (slice_k[q0:q1], slice_ptr[q0:q1 + 1] - f0, fiber_j[f0:f1], fiber_ptr[f0:f1 + 1] - e0,
            nz_i[e0:e1], val[e0:e1])


def compress_sparse_sharded(local_compress, y, dst: int = 0, group=None):
    """Sparse input across ranks: ``local_compress(rank, world, y)`` writes this
    rank's partial replicas of its share (``coo_share`` / ``csf_shares``) into
    y, then one sum-reduce to ``dst`` (NCCL on GPUs). Returns y (complete on dst)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local_compress(rank, world, y)
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
    import torch.distributed as dist

    compress_sharded(compress_slab, K, y, dst=dst, group=group)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
        return decompose_replicas(y)
    factors, metrics, err = None, None, None
    if rank == dst:
        try:
            factors, metrics = decompose_replicas(y)
        except Exception as e:  # tell the other ranks before anyone blocks
            err = e
    try:
        shapes = _broadcast_outcome(rank, dst, group, [list(f.shape) for f in factors] if factors else None,
                                    f"rank {dst}: {type(err).__name__}: {err}" if err is not None else None)
    except RemoteStageError:
        if err is not None:
            raise err
        raise
    factors = _broadcast_factors(factors, shapes, rank, dst, group, y.device)
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
    res, s1_err = None, None
    try:
        res = stage1(mine.narrow(0, 0, (p1 - p0) * lmn), np.arange(p0, p1, dtype=np.int64)) if p1 > p0 else None
    except Exception as e:  # reported through the gather, re-raised below
        if world == 1:
            raise
        s1_err = e
    t_s1 = time.perf_counter() - t0
    if world > 1:
        parts = [None] * world if rank == dst else None
        dist.gather_object((res, f"rank {rank}: {type(s1_err).__name__}: {s1_err}" if s1_err else None), parts,
                           dst=dst, group=group)
    else:
        parts = [(res, None)]
    factors, metrics, err = None, None, None
    if rank == dst:
        from .api import Stage1Result
        errs = [e for _, e in parts if e is not None]
        if errs:
            err = "; ".join(errs)
        else:
            try:
                rs = [r for r, _ in parts if r is not None]
                merged = Stage1Result(*(np.concatenate([getattr(r, f) for r in rs])
                                        for f in ("ids", "factors", "fit_err", "converged", "sweeps")))
                factors, metrics = finish(merged)
            except Exception as e:
                if world == 1:
                    raise
                err = f"rank {dst}: {type(e).__name__}: {e}"
    if world > 1:
        try:
            shapes = _broadcast_outcome(rank, dst, group, [list(f.shape) for f in factors] if factors else None, err)
        except RemoteStageError:
            if s1_err is not None:
                raise s1_err
            raise
        factors = _broadcast_factors(factors, shapes, rank, dst, group, y.device)
    return factors, metrics, t_s1
