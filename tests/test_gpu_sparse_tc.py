"""The tensor-core sparse path (csrc/sparse_tc.cu: dense tiles of a slice)
against the fp64 oracle and against the SIMT fiber kernel (XTSG_SPARSE_TC=0).

Covers the tile machinery's edge cases: a single fiber with more than 512
distinct i (cut into 512-nonzero pieces), tiles whose i support overflows
(retried with fewer fibers), empty slices and fibers in CSF input, duplicate
coordinates, more than four 128-row blocks of stacked U, L = M = 128 (one
replica per row block), padded reduced dims, and fp16 operands.

Tolerance: the sparse path's stated bf16 bar, relative Frobenius error per
replica <= 1e-2 vs the reference's fp64 comp (measured ~3e-3); fp16 2e-3.
"""
import os

import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _dense(dims, i, j, k, v):
    t = np.zeros(dims, order="F")
    np.add.at(t, (i, j, k), v.astype(np.float64))
    return t


def _check(gpu, restated, plan, dims, red, P, seed, i, j, k, v, tol=TOL):
    ens = gpu.make_ensemble(dims, red, P, 8, seed)
    y = gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red)
    t = _dense(dims, i, j, k, v)
    errs = [rel_diff(restated.comp(t, ens.u[p], ens.v[p], ens.w[p]), y[p]) for p in range(P)]
    assert max(errs) <= tol, errs
    return y


def _fiber_path(fn):
    old = os.environ.get("XTSG_SPARSE_TC")
    os.environ["XTSG_SPARSE_TC"] = "0"
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["XTSG_SPARSE_TC"]
        else:
            os.environ["XTSG_SPARSE_TC"] = old


def _flat(reps):
    return np.concatenate([np.asarray(r).ravel(order="F") for r in reps])


def test_long_fiber_and_overflowing_tiles(gpu, restated):
    # slice 0: one fiber with 1500 distinct i (3 pieces of <= 512 nonzeros);
    # slice 1: 64 fibers x 40 disjoint i each (2560 distinct: the 64-fiber
    # tile overflows and is retried at 32, 16, 8 fibers); slice 2: sparse noise
    dims, red, P = (4000, 70, 20), (32, 32, 16), 8
    rng = np.random.default_rng(4)
    i0 = rng.permutation(dims[0])[:1500]
    parts = [(i0, np.full(1500, 3), np.zeros(1500, int))]
    ii, jj = [], []
    for f in range(64):
        ii.append(np.arange(f * 40, f * 40 + 40) + 500)
        jj.append(np.full(40, f + 2))
    parts.append((np.concatenate(ii), np.concatenate(jj), np.ones(64 * 40, int)))
    n = 3000
    parts.append((rng.integers(0, dims[0], n), rng.integers(0, dims[1], n), np.full(n, 2)))
    i, j, k = (np.concatenate([p[q] for p in parts]).astype(np.int32) for q in range(3))
    v = rng.standard_normal(i.size).astype(np.float32)
    plan = gpu.Plan(dims, red, P, 8, 5)
    y = _check(gpu, restated, plan, dims, red, P, 5, i, j, k, v)
    y_f = _fiber_path(lambda: gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red))
    assert rel_diff(_flat(y_f), _flat(y)) <= 5e-3


def test_dense_subcubes_many_row_blocks(gpu, restated):
    # C4-like structure (rank-1 blocks over sparse supports) with P*L = 1280
    # stacked rows (10 row blocks) and duplicates from overlapping blocks
    dims, red, P, R, nz = (3000, 2500, 2000), (64, 64, 32), 20, 3, 40
    rng = np.random.default_rng(8)
    fac = []
    for dn in dims:
        m = np.zeros((dn, R))
        for r in range(R):
            m[rng.choice(dn, nz, replace=False), r] = rng.standard_normal(nz)
        fac.append(m)
    fac[2][:, 1] = 0
    fac[2][np.nonzero(fac[2][:, 0])[0][:10], 1] = 1.0  # blocks 0 and 1 share ten slices
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
    errs = [rel_diff(restated.comp_from_factors(*fac, ens.u[p], ens.v[p], ens.w[p]), y[p]) for p in range(P)]
    assert max(errs) <= TOL, errs


def test_csf_empty_slices_and_fibers(gpu, restated):
    dims, red, P = (300, 200, 50), (32, 32, 16), 6
    rng = np.random.default_rng(2)
    # slices: k=3 (2 fibers, one empty), k=7 (no fibers), k=9 (1 fiber, empty), k=20 (3 fibers)
    slice_k = np.array([3, 7, 9, 20], np.int32)
    slice_ptr = np.array([0, 2, 2, 3, 6], np.int64)
    fiber_j = np.array([5, 6, 7, 1, 50, 199], np.int32)
    counts = np.array([30, 0, 0, 600, 1, 90])
    fiber_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    nnz = int(fiber_ptr[-1])
    nz_i = rng.integers(0, dims[0], nnz).astype(np.int32)
    val = rng.standard_normal(nnz).astype(np.float32)
    plan = gpu.Plan(dims, red, P, 8, 3)
    ens = gpu.make_ensemble(dims, red, P, 8, 3)
    y = gpu.Plan.replicas(plan.compress_csf(slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val), P, red)
    kk = np.repeat(np.repeat(slice_k, np.diff(slice_ptr)), counts)
    jj = np.repeat(fiber_j, counts)
    t = _dense(dims, nz_i, jj, kk, val)
    for p in range(P):
        assert rel_diff(restated.comp(t, ens.u[p], ens.v[p], ens.w[p]), y[p]) <= TOL
    # an i outside the tensor is rejected (range check on the device) before any gather
    for bad in (dims[0], -1):
        bi = nz_i.copy()
        bi[nnz // 2] = bad
        with pytest.raises(gpu.DataError):
            plan.compress_csf(slice_k, slice_ptr, fiber_j, fiber_ptr, bi, val)


@pytest.mark.parametrize("red,P,prec,tol", [
    ((128, 128, 32), 3, "bf16", TOL),   # one replica per row block, Mpad = 128
    ((64, 32, 32), 5, "bf16", TOL),     # Lpad 64 > Mpad 32
    ((32, 32, 32), 9, "fp16", 2e-3),
    ((30, 30, 16), 4, "bf16", TOL),     # padded Lpad = Mpad = 32
])
def test_shapes_and_precisions(gpu, restated, red, P, prec, tol):
    dims = (700, 300, 60)
    rng = np.random.default_rng(11)
    nnz = 60000
    i = rng.integers(0, 200, nnz).astype(np.int32)  # narrow i support: dense tiles
    j = rng.integers(0, dims[1], nnz).astype(np.int32)
    k = rng.integers(0, dims[2], nnz).astype(np.int32)
    v = rng.standard_normal(nnz).astype(np.float32)
    pr = gpu.PREC_FP16 if prec == "fp16" else gpu.PREC_BF16
    plan = gpu.Plan(dims, red, P, 8, 21, precision=pr)
    y = _check(gpu, restated, plan, dims, red, P, 21, i, j, k, v, tol)
    y_f = _fiber_path(lambda: gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red))
    assert rel_diff(_flat(y_f), _flat(y)) <= tol
