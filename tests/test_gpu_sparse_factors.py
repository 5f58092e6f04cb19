"""GPU parity of the factored-source path (blocks generated on the device) and
the sparse COO path against the fp64 oracle.

Tolerance: same stated bf16 bar as the dense fast path (relative Frobenius
error per replica <= 1e-2 vs the reference's fp64 comp / comp_from_factors).
"""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu
TOL = 1e-2


def test_compress_factors_vs_comp_from_factors(gpu, restated):
    dims, red, P, R = (320, 260, 90), (64, 64, 32), 6, 7
    plan = gpu.Plan(dims, red, P, 16, 31)
    ens = gpu.make_ensemble(dims, red, P, 16, 31)
    a, b, c = restated.generate_dense(dims, R, 5)
    y = gpu.Plan.replicas(plan.compress_factors((a, b, c)), P, red)
    for p in range(P):
        want = restated.comp_from_factors(a, b, c, ens.u[p], ens.v[p], ens.w[p])
        assert rel_diff(want, y[p]) <= TOL
    # k sub-ranges accumulate to the whole (mode-3 slab sharding)
    acc = plan.compress_factors((a, b, c), 0, 40)
    acc = plan.compress_factors((a, b, c), 40, 90, y=acc, accumulate=True)
    assert rel_diff(_flat(y), acc) <= 1e-4


def _flat(reps):
    return np.concatenate([r.ravel(order="F") for r in reps])


def _random_coo(dims, nnz, seed):
    rng = np.random.default_rng(seed)
    i = rng.integers(0, dims[0], nnz).astype(np.int32)
    j = rng.integers(0, dims[1], nnz).astype(np.int32)
    k = rng.integers(0, dims[2], nnz).astype(np.int32)
    v = rng.standard_normal(nnz).astype(np.float32)
    return i, j, k, v


def _dense(dims, i, j, k, v):
    t = np.zeros(dims, order="F")
    np.add.at(t, (i, j, k), v.astype(np.float64))
    return t


@pytest.mark.parametrize("dims,red,P,nnz", [
    ((97, 88, 71), (32, 32, 16), 8, 20000),      # unsorted, with duplicates
    ((300, 50, 40), (64, 30, 20), 3, 5000),     # padded M, P*L not a multiple of 128
])
def test_coo_vs_dense_oracle(gpu, restated, dims, red, P, nnz):
    plan = gpu.Plan(dims, red, P, 8, 77)
    ens = gpu.make_ensemble(dims, red, P, 8, 77)
    i, j, k, v = _random_coo(dims, nnz, 3)
    y = gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red)
    t = _dense(dims, i, j, k, v)
    for p in range(P):
        assert rel_diff(restated.comp(t, ens.u[p], ens.v[p], ens.w[p]), y[p]) <= TOL
    # pre-sorted input (sort skipped) gives the same result
    order = np.lexsort((j, k))
    y2 = plan.compress_coo(i[order], j[order], k[order], v[order])
    assert rel_diff(_flat(y), y2) <= 1e-5


def test_coo_sparse_factor_structure(gpu, restated):
    # config-C4 structure at small scale: X = sum of R rank-1 blocks built from
    # sparse factors (generate(sparse), pipeline.cpp:164-172); duplicates sum
    dims, red, P, R, nz = (5000, 4000, 3000), (32, 32, 32), 4, 3, 12
    rng = np.random.default_rng(9)
    fac = []
    for n in dims:
        m = np.zeros((n, R))
        for r in range(R):
            m[rng.choice(n, nz, replace=False), r] = rng.standard_normal(nz)
        fac.append(m)
    ii, jj, kk, vv = [], [], [], []
    for r in range(R):
        ia, ja, ka = (np.nonzero(f[:, r])[0] for f in fac)
        I3, J3, K3 = np.meshgrid(ia, ja, ka, indexing="ij")
        ii.append(I3.ravel()); jj.append(J3.ravel()); kk.append(K3.ravel())
        vv.append((fac[0][I3, r] * fac[1][J3, r] * fac[2][K3, r]).ravel())
    i, j, k = (np.concatenate(x).astype(np.int32) for x in (ii, jj, kk))
    v = np.concatenate(vv).astype(np.float32)
    plan = gpu.Plan(dims, red, P, 8, 12)
    ens = gpu.make_ensemble(dims, red, P, 8, 12)
    y = gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red)
    for p in range(P):
        want = restated.comp_from_factors(*fac, ens.u[p], ens.v[p], ens.w[p])
        assert rel_diff(want, y[p]) <= TOL


def test_coo_rejects_out_of_range(gpu):
    plan = gpu.Plan((40, 40, 40), (32, 32, 32), 2, 4, 1)
    with pytest.raises(gpu.DataError):
        plan.compress_coo([0, 40], [0, 0], [0, 0], [1.0, 1.0])


def test_csf_matches_coo_bitwise_and_validates(gpu, restated):
    # CSF input skips the sort; the COO path also regroups each slice's fibers
    # by their smallest i, so the two group fibers into different tiles: the
    # replicas agree to bf16 level (duplicate coordinates are summed in bf16 in
    # tile order), and each matches the fp64 oracle at the stated bar
    dims, red, P = (97, 88, 71), (32, 32, 16), 8
    plan = gpu.Plan(dims, red, P, 8, 77)
    ens = gpu.make_ensemble(dims, red, P, 8, 77)
    i, j, k, v = _random_coo(dims, 20000, 3)
    y_coo = plan.compress_coo(i, j, k, v)
    csf = gpu.Plan.coo_to_csf(i, j, k, v)
    y_csf = plan.compress_csf(*csf)
    assert rel_diff(np.asarray(y_coo, np.float64), np.asarray(y_csf, np.float64)) <= 2e-3
    t = _dense(dims, i, j, k, v)
    got = gpu.Plan.replicas(y_csf, P, red)
    for p in range(P):
        assert rel_diff(restated.comp(t, ens.u[p], ens.v[p], ens.w[p]), got[p]) <= TOL
    # accumulate, and duplicate slices (the same k split in two slice records) sum
    sk, sp, fj, fp, ni, nv = csf
    y2 = plan.compress_csf(sk, sp, fj, fp, ni, nv, y=np.asarray(y_csf).copy(), accumulate=True)
    assert rel_diff(2 * np.asarray(y_csf, np.float64), np.asarray(y2, np.float64)) <= 1e-6
    bad_k = sk.copy()
    bad_k[0] = dims[2]
    with pytest.raises(gpu.DataError):
        plan.compress_csf(bad_k, sp, fj, fp, ni, nv)
    bad_fp = fp.copy()
    bad_fp[1], bad_fp[2] = bad_fp[2], bad_fp[1]
    with pytest.raises(gpu.DataError):
        plan.compress_csf(sk, sp, fj, bad_fp, ni, nv)
