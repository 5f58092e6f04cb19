"""Multi-rank (gloo, world size 2, CPU) check of the mode-3 slab sharding +
reduction logic used by the multi-GPU path. The per-rank compression is the
CPU oracle here (the CUDA kernels are exercised by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_13693_b200.dist import compress_sharded, slab_range


def test_slab_ranges_partition():
    for K in (1, 7, 2000, 10_000):
        for world in (1, 2, 3, 8):
            spans = [slab_range(K, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restated
    ora = Restated()
    dims, red, P, S, seed = (12, 10, 9), (4, 3, 3), 3, 2, 5
    ens = ora.make_ensemble(dims, red, P, S, seed=seed)
    t = np.asfortranarray(np.random.default_rng(1).standard_normal(dims))

    def local(k0, k1, y):
        parts = [ora.comp(np.asfortranarray(t[:, :, k0:k1]), ens[0][p], ens[1][p], ens[2][p][:, k0:k1])
                 for p in range(P)]
        y.copy_(torch.from_numpy(np.concatenate([x.ravel(order="F") for x in parts])))

    y = torch.zeros(P * int(np.prod(red)), dtype=torch.float64)
    compress_sharded(local, dims[2], y)
    if rank == 0:
        full = np.concatenate([ora.comp(t, ens[0][p], ens[1][p], ens[2][p]).ravel(order="F") for p in range(P)])
        out["err"] = float(np.abs(y.numpy() - full).max())
    dist.destroy_process_group()


def test_gloo_world2_sharded_compression_matches_one_shot():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["err"] <= 1e-12


def _pipeline_worker(rank, world, port, out):
    # host logic of the sharded pipeline: slab compression (oracle stand-in),
    # reduce to rank 0, decomposition there (stand-in: the exact factors are
    # recovered from the replicas by a least-squares fit), broadcast back
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_13693_b200.dist import decompose_sharded
    from oracle.oracle import Restated
    ora = Restated()
    dims, red, P, S, seed = (12, 10, 9), (4, 3, 3), 3, 2, 5
    ens = ora.make_ensemble(dims, red, P, S, seed=seed)
    rng = np.random.default_rng(2)
    f = [np.asfortranarray(rng.standard_normal((n, 2))) for n in dims]
    t = np.asfortranarray(np.einsum("ir,jr,kr->ijk", *f))

    def local(k0, k1, y):
        parts = [ora.comp(np.asfortranarray(t[:, :, k0:k1]), ens[0][p], ens[1][p], ens[2][p][:, k0:k1])
                 for p in range(P)]
        y.copy_(torch.from_numpy(np.concatenate([x.ravel(order="F") for x in parts])))

    def decompose(y):
        full = np.concatenate([ora.comp(t, ens[0][p], ens[1][p], ens[2][p]).ravel(order="F") for p in range(P)])
        assert np.abs(y.numpy() - full).max() <= 1e-12
        return tuple(x * (m + 1) for m, x in enumerate(f)), {"ok": True}

    y = torch.zeros(P * int(np.prod(red)), dtype=torch.float64)
    fac, met = decompose_sharded(local, dims[2], y, decompose)
    out[rank] = (max(float(np.abs(a - b * (m + 1)).max()) for m, (a, b) in enumerate(zip(fac, f))), met is not None)
    dist.destroy_process_group()


def test_gloo_world2_sharded_pipeline():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pipeline_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == (0.0, True) and out[1] == (0.0, False)


def test_replica_ranges_partition():
    from paper_2311_13693_b200.dist import replica_range
    for P in (1, 5, 124, 128):
        for world in (1, 2, 3, 8):
            spans = [replica_range(P, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _distributed_worker(rank, world, port, out):
    # host logic of the ALS-sharded pipeline: slab compression (oracle
    # stand-in), reduce-scatter of the replicas, stage 1 per rank on its own
    # replicas (stand-in: a deterministic function of the replica and its id),
    # gather of the per-replica results on rank 0, finish there, broadcast
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_13693_b200.api import Stage1Result
    from paper_2311_13693_b200.dist import decompose_distributed
    from oracle.oracle import Restated
    ora = Restated()
    dims, red, P, S, seed = (12, 10, 9), (4, 3, 3), 5, 2, 5
    lmn = int(np.prod(red))
    ens = ora.make_ensemble(dims, red, P, S, seed=seed)
    t = np.asfortranarray(np.random.default_rng(3).standard_normal(dims))
    full = [ora.comp(t, ens[0][p], ens[1][p], ens[2][p]).ravel(order="F") for p in range(P)]
    per = -(-P // world)

    def local(k0, k1, y):
        y.zero_()
        for p in range(P):
            part = ora.comp(np.asfortranarray(t[:, :, k0:k1]), ens[0][p], ens[1][p], ens[2][p][:, k0:k1])
            y[p * lmn:(p + 1) * lmn] = torch.from_numpy(part.ravel(order="F"))

    seen = {}

    def stage1(reps, ids):
        reps = reps.numpy().reshape(len(ids), lmn)
        for q, p in enumerate(ids):
            seen[int(p)] = float(np.abs(reps[q] - full[p]).max())
        return Stage1Result(ids, reps * 2.0, ids * 0.5, np.ones(len(ids), np.int32), ids + 100)

    def finish(merged):
        assert list(merged.ids) == list(range(P))
        want = np.stack([2.0 * full[p] for p in range(P)])
        assert np.abs(merged.factors - want).max() <= 1e-12
        assert list(merged.sweeps) == [p + 100 for p in range(P)]
        return (merged.factors[:, :3].copy(order="F"), merged.factors[:, 3:5].copy(order="F"),
                merged.factors[:, 5:6].copy(order="F")), {"ok": True}

    y = torch.zeros(per * world * lmn, dtype=torch.float64)
    fac, met, _ = decompose_distributed(local, dims[2], P, lmn, y, stage1, finish)
    want = np.stack([2.0 * full[p] for p in range(P)])
    out[rank] = (max(seen.values()) if seen else 0.0, sorted(seen),
                 float(np.abs(fac[0] - want[:, :3]).max()), met is not None)
    dist.destroy_process_group()


def test_gloo_world2_als_sharded_pipeline():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_distributed_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0][0] <= 1e-12 and out[1][0] <= 1e-12
    assert out[0][1] == [0, 1, 2] and out[1][1] == [3, 4]   # ceil(5 / 2) replicas per rank
    assert out[0][2] <= 1e-12 and out[1][2] <= 1e-12   # slab sums vs one-shot: rounding only
    assert out[0][3] and not out[1][3]


def _failing_worker(rank, world, port, out, where):
    # a stage that raises on one rank must surface on every rank instead of
    # leaving the others blocked in the next collective
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=__import__("datetime").timedelta(seconds=60))
    from paper_2311_13693_b200.api import Stage1Result
    from paper_2311_13693_b200.dist import decompose_distributed, decompose_sharded
    P, lmn = 4, 8
    y = torch.zeros(P * lmn, dtype=torch.float64)

    def local(k0, k1, yy):
        yy.fill_(1.0)

    def stage1(reps, ids):
        if where == "stage1" and rank == 1:
            raise ValueError("every replica failed to fit")
        return Stage1Result(ids, np.zeros((len(ids), 3)), ids * 0.0, np.ones(len(ids), np.int32), ids)

    def finish(merged):
        if where == "finish":
            raise ValueError("ill-posed stack")
        return (np.zeros((2, 1)),) * 3, {}

    def decompose(yy):
        raise ValueError("no survivors")

    try:
        if where == "sharded":
            decompose_sharded(local, 10, y, decompose)
        else:
            decompose_distributed(local, 10, P, lmn, y, stage1, finish)
        out[rank] = "returned"
    except Exception as e:  # noqa: BLE001
        out[rank] = f"{type(e).__name__}: {e}"
    dist.destroy_process_group()


@pytest.mark.parametrize("where", ["sharded", "stage1", "finish"])
def test_gloo_world2_stage_failure_raises_everywhere(where):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_failing_worker, args=(2, _free_port(), out, where), nprocs=2, join=True)
    assert "returned" not in (out[0], out[1])
    msg = {"sharded": "no survivors", "stage1": "every replica failed", "finish": "ill-posed"}[where]
    assert msg in out[0] and msg in out[1]


def _sparse_csf(dims, nnz, seed):
    from paper_2311_13693_b200.api import Plan
    rng = np.random.default_rng(seed)
    i, j = rng.integers(0, dims[0], nnz), rng.integers(0, dims[1], nnz)
    k = rng.integers(0, dims[2] // 2, nnz) * 2          # odd k empty
    k[: nnz // 3] = 4                                   # one heavy slice
    v = rng.standard_normal(nnz).astype(np.float32)
    return (i, j, k, v), Plan.coo_to_csf(i, j, k, v)


def _dense(dims, i, j, k, v):
    t = np.zeros(dims, order="F")
    np.add.at(t, (np.asarray(i), np.asarray(j), np.asarray(k)), np.asarray(v, np.float64))
    return t


def test_sparse_shares_partition():
    from paper_2311_13693_b200.dist import coo_share, csf_part, csf_shares
    for nnz in (0, 1, 5, 1000):
        for world in (1, 2, 3, 8):
            spans = [coo_share(nnz, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nnz
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    (_, _, _, v), csf = _sparse_csf((20, 15, 40), 3000, 1)
    for world in (1, 2, 3, 8):
        qs = csf_shares(csf[1], csf[3], world)
        assert qs[0] == 0 and qs[-1] == len(csf[0]) and all(a <= b for a, b in zip(qs, qs[1:]))
        parts = [csf_part(csf, a, b) for a, b in zip(qs, qs[1:])]
        assert sum(len(p[5]) for p in parts) == len(v)
        for p in parts:
            assert p[1][0] == 0 and p[1][-1] == len(p[2]) and p[3][0] == 0 and p[3][-1] == len(p[5])
        # balance: no share beyond 1/world of the nonzeros plus the heaviest slice
        heavy = int(np.diff(csf[3][csf[1]]).max())
        assert max(len(p[5]) for p in parts) <= len(v) / world + heavy
    assert csf_shares(np.zeros(1, np.int64), np.zeros(1, np.int64), 4) == [0, 0, 0, 0, 0]


def _sparse_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restated
    from paper_2311_13693_b200.dist import compress_sparse_sharded, coo_share, csf_part, csf_shares
    ora = Restated()
    dims, red, P, S, seed = (20, 15, 40), (4, 3, 5), 3, 2, 7
    u, vv, w = ora.make_ensemble(dims, red, P, S, seed=seed)
    (i, j, k, v), csf = _sparse_csf(dims, 3000, 1)

    def comp(t):
        return torch.from_numpy(np.concatenate([ora.comp(t, u[p], vv[p], w[p]).ravel(order="F")
                                                for p in range(P)]))

    def local_csf(r, g, y):
        qs = csf_shares(csf[1], csf[3], g)
        sk, sp, fj, fp, ni, val = csf_part(csf, qs[r], qs[r + 1])
        kk = np.repeat(np.repeat(sk, np.diff(sp)), np.diff(fp))
        jj = np.repeat(fj, np.diff(fp))
        y.copy_(comp(_dense(dims, ni, jj, kk, val)))

    def local_coo(r, g, y):
        e0, e1 = coo_share(len(v), r, g)
        y.copy_(comp(_dense(dims, i[e0:e1], j[e0:e1], k[e0:e1], v[e0:e1])))

    full = comp(_dense(dims, i, j, k, v)).numpy()
    for name, fn in (("csf", local_csf), ("coo", local_coo)):
        y = torch.zeros(P * int(np.prod(red)), dtype=torch.float64)
        compress_sparse_sharded(fn, y)
        if rank == 0:
            out[name] = float(np.abs(y.numpy() - full).max() / np.abs(full).max())
    dist.destroy_process_group()


def test_gloo_world2_sparse_shares_match_one_shot():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sparse_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["csf"] <= 1e-12 and out["coo"] <= 1e-12
