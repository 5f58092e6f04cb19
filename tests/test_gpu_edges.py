"""Edge cases of the device path that the reference's own tests exercise for
its CPU functions (empty / degenerate shapes, singleton modes, ragged blocks,
zero inputs, maximum-size guards), through the C ABI."""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu


def test_comp_degenerate_shapes(gpu, restated):
    rng = np.random.default_rng(1)
    # singleton modes (test_compression.cpp:132-140 uses 1x1x1 with a scalar chain)
    for dims, red in [((1, 1, 1), (1, 1, 1)), ((1, 7, 5), (1, 3, 2)), ((9, 1, 4), (2, 1, 4)), ((6, 5, 1), (3, 5, 1))]:
        t = np.asfortranarray(rng.standard_normal(dims))
        u, v, w = (rng.standard_normal((red[m], dims[m])) for m in range(3))
        got = gpu.comp(t, u, v, w)
        assert rel_diff(restated.comp(t, u, v, w), got) <= 1e-12
    # an all-zero tensor compresses to exact zeros
    z = gpu.comp(np.zeros((4, 5, 6), order="F"), rng.standard_normal((2, 4)), rng.standard_normal((2, 5)),
                 rng.standard_normal((2, 6)))
    assert not z.any()


def test_plan_single_slices_and_ragged_blocks(gpu, restated):
    dims, red, P, S = (70, 33, 5), (32, 16, 3), 3, 2
    ens = restated.make_ensemble(dims, red, P, S, seed=8)
    t = np.asfortranarray(np.random.default_rng(2).standard_normal(dims))
    plan = gpu.Plan(dims, red, P, S, 8)
    # one slice at a time (extent 1 along mode 3), accumulated
    y = None
    for k in range(dims[2]):
        blk = np.asfortranarray(t[:, :, k:k + 1])
        y = plan.compress(blk, y=y, offset=(0, 0, k), accumulate=k > 0)
    got = gpu.Plan.replicas(y, P, red)
    for p in range(P):
        assert rel_diff(restated.comp(t, ens[0][p], ens[1][p], ens[2][p]), got[p]) <= 1e-2
    # ragged interior block at an unaligned offset (TMA needs an aligned copy)
    blk = np.asfortranarray(t[3:70, 5:33, 1:4])
    sub = gpu.Plan.replicas(plan.compress(blk, offset=(3, 5, 1)), P, red)
    for p in range(P):
        want = restated.comp(blk, ens[0][p][:, 3:70], ens[1][p][:, 5:33], ens[2][p][:, 1:4])
        assert rel_diff(want, sub[p]) <= 1e-2
    # blocks outside the tensor are usage errors
    with pytest.raises(gpu.UsageError):
        plan.compress(np.zeros((8, 8, 2), order="F"), offset=(65, 0, 0))


def test_coo_empty_and_duplicates(gpu, restated):
    dims, red, P = (40, 30, 20), (16, 16, 8), 2
    plan = gpu.Plan(dims, red, P, 4, 3)
    empty = np.zeros(0, np.int32)
    y = plan.compress_coo(empty, empty, empty, np.zeros(0, np.float32))
    assert not np.asarray(y).any()
    # accumulate onto existing replicas with an empty batch keeps them
    y0 = np.arange(P * int(np.prod(red)), dtype=np.float32)
    y1 = plan.compress_coo(empty, empty, empty, np.zeros(0, np.float32), y=y0.copy(), accumulate=True)
    assert np.array_equal(np.asarray(y1), y0)
    # one coordinate repeated: duplicates sum (a16)
    i = np.array([5, 5, 5], np.int32)
    j = np.array([7, 7, 7], np.int32)
    k = np.array([3, 3, 3], np.int32)
    v = np.array([1.0, 2.0, -0.5], np.float32)
    got = gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red)
    t = np.zeros(dims, order="F")
    t[5, 7, 3] = 2.5
    ens = restated.make_ensemble(dims, red, P, 4, seed=3)
    for p in range(P):
        assert rel_diff(restated.comp(t, ens[0][p], ens[1][p], ens[2][p]), got[p]) <= 1e-2


def test_als_rank_guards_and_nan(gpu):
    t = np.asfortranarray(np.random.default_rng(3).standard_normal((3, 3, 3)))
    with pytest.raises(gpu.UsageError):
        gpu.cp_als(t, 10)   # rank above min(JK, IK, IJ) = 9 (cp_als.cpp:51-54)
    with pytest.raises(gpu.UsageError):
        gpu.cp_als(t, 0)
    bad = t.copy()
    bad[1, 1, 1] = np.nan
    with pytest.raises(gpu.DataError):
        gpu.cp_als(bad, 2)


@pytest.mark.parametrize("prec", ["fp64", "fp16x3"])
def test_pageable_host_input_staged_copy(gpu, prec):
    """Pageable host input of >= 8 MB is copied by host threads through pinned
    64 MB chunks (h2d_copy): a tensor of 2 chunks plus a ragged tail must give
    the same replicas as the same tensor resident on the device (bitwise on
    the fp64 path; the compensated mode's fp64 mode-3 sums may reorder)."""
    import torch
    dims, red, P = (257, 251, 161), (16, 16, 8), 2      # 83 MB of fp64
    x = np.asfortranarray(np.random.default_rng(4).standard_normal(dims))
    plan = gpu.Plan(dims, red, P, 8, 5, precision=gpu.PREC_FP64 if prec == "fp64" else gpu.PREC_FP16X3)
    yh = np.asarray(plan.compress(x))
    xd = torch.from_numpy(x).cuda()
    assert xd.stride() == (1, dims[0], dims[0] * dims[1])
    yd = plan.compress(xd)
    yd = yd.cpu().numpy() if hasattr(yd, "cpu") else np.asarray(yd)
    if prec == "fp64":
        assert np.array_equal(yh.ravel(), yd.ravel())
    else:
        assert rel_diff(yh.ravel(), yd.ravel()) <= 1e-12
    plan.close()
