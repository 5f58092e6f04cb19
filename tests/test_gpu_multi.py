"""The multi-GPU C ABI (xtsg_multi_*): mode-3 slabs per GPU + one NCCL reduce
(SURVEY §8 e). The round's GPU box has one B200, so the clique here is one
GPU (the reduce still runs through NCCL: a 1-rank ncclReduce); the slab split
and reduction arithmetic for G > 1 is the same code path with a longer device
list. Checked against the oracle and the single-plan path."""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu


def test_nccl_resolved(gpu):
    assert gpu.nccl_version() >= 21800


def test_multi_factors_and_dense_vs_oracle(gpu, restated):
    dims, red, P, S, R = (400, 300, 160), (64, 64, 32), 6, 8, 7
    seed = 123
    f = restated.generate_dense(dims, R, 3)
    ens = restated.make_ensemble(dims, red, P, S, seed)
    want = [restated.comp_from_factors(*f, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    mp = gpu.MultiPlan(dims, red, P, S, seed, gpus=[0], precision=gpu.PREC_BF16)
    y = gpu.Plan.replicas(mp.compress_factors(f), P, red)
    assert max(rel_diff(w, g) for w, g in zip(want, y)) <= 5e-3
    assert mp.last_ms() > 0.0
    # same numbers as one plan over the whole tensor
    plan = gpu.Plan(dims, red, P, S, seed, precision=gpu.PREC_BF16)
    y1 = plan.compress_factors(f)
    assert np.array_equal(np.concatenate([x.ravel(order="F") for x in y]), y1)
    # dense host input, accumulate
    t = np.asfortranarray(np.einsum("ir,jr,kr->ijk", *f))
    y2 = mp.compress(t)
    y2 = mp.compress(t, y=y2, accumulate=True)
    y2 = gpu.Plan.replicas(y2 / 2, P, red)
    assert max(rel_diff(w, g) for w, g in zip(want, y2)) <= 5e-3
    mp.close()
    plan.close()


def test_multi_rejects_bad_device_lists(gpu):
    with pytest.raises(gpu.UsageError):
        gpu.MultiPlan((64, 64, 8), (32, 32, 8), 2, 4, 1, gpus=[0, 0])
    with pytest.raises(gpu.UsageError):
        gpu.MultiPlan((64, 64, 8), (32, 32, 8), 2, 4, 1, gpus=[99])


def _dense(dims, i, j, k, v):
    t = np.zeros(dims, order="F")
    np.add.at(t, (i, j, k), v.astype(np.float64))
    return t


def _sparse_case(dims, nnz, seed):
    """k-sorted COO with duplicates, a few dense (j, k) fibers and empty k."""
    rng = np.random.default_rng(seed)
    i = rng.integers(0, dims[0], nnz)
    j = rng.integers(0, dims[1], nnz)
    k = rng.integers(0, dims[2] // 2, nnz) * 2            # every odd k empty
    j[: nnz // 4], k[: nnz // 4] = 7, 10                   # one long fiber (slice 10)
    i[nnz // 2: nnz // 2 + 50] = 3                         # duplicated coordinates
    j[nnz // 2: nnz // 2 + 50], k[nnz // 2: nnz // 2 + 50] = 5, 0
    v = rng.standard_normal(nnz).astype(np.float32)
    order = np.argsort(k, kind="stable")
    return [a[order].astype(np.int32) for a in (i, j, k)] + [v[order]]


def test_multi_sparse_chunked_vs_oracle(gpu, restated, monkeypatch):
    """xtsg_multi_compress_coo / _csf: the nonzero share of a GPU cut into
    XTSG_SPARSE_CHUNK-sized device calls accumulated in its partial, then the
    NCCL reduce; against the oracle's Eq. 3 over the dense tensor and against
    one plan call over all nonzeros."""
    dims, red, P, S, seed = (300, 200, 60), (32, 32, 16), 5, 8, 11
    tol = 1e-2   # the sparse bf16 bar (test_gpu_sparse_tc.TOL): 24k nonzeros average little rounding
    i, j, k, v = _sparse_case(dims, 24000, 3)
    t = _dense(dims, i, j, k, v)
    u, vv, w = restated.make_ensemble(dims, red, P, S, seed)
    want = [restated.comp(t, u[p], vv[p], w[p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, seed)
    y1 = plan.compress_coo(i, j, k, v)
    mp = gpu.MultiPlan(dims, red, P, S, seed, gpus=[0])
    for chunk in ("3001", "100000"):     # 8 accumulated calls / one call
        monkeypatch.setenv("XTSG_SPARSE_CHUNK", chunk)
        y = mp.compress_coo(i, j, k, v)
        assert max(rel_diff(a, b) for a, b in zip(want, gpu.Plan.replicas(y, P, red))) <= tol
        assert rel_diff(y1, y) <= tol
        csf = gpu.Plan.coo_to_csf(i, j, k, v)
        yc = mp.compress_csf(*csf)
        assert max(rel_diff(a, b) for a, b in zip(want, gpu.Plan.replicas(yc, P, red))) <= tol
    # the long fiber's slice (6000 nonzeros) exceeds the chunk: it runs whole
    monkeypatch.setenv("XTSG_SPARSE_CHUNK", "1000")
    yc2 = mp.compress_csf(*csf, y=yc.copy(), accumulate=True)
    assert max(rel_diff(2 * a, b) for a, b in zip(want, gpu.Plan.replicas(yc2, P, red))) <= tol
    # empty input: zero replicas
    z = mp.compress_coo(i[:0], j[:0], k[:0], v[:0])
    assert not z.any()
    # malformed input is rejected by the GPU holding it
    bad = list(csf)
    bad[4] = bad[4].copy()
    bad[4][-1] = dims[0]
    with pytest.raises(gpu.DataError):
        mp.compress_csf(*bad)
    with pytest.raises(gpu.UsageError):
        mp.compress_csf(csf[0], csf[1][:-1], *csf[2:])
    kb = k.copy()
    kb[0] = -1
    with pytest.raises(gpu.DataError):
        mp.compress_coo(i, j, kb, v)
    mp.close()
    plan.close()
