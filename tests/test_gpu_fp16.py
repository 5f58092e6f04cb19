"""GPU parity of the fp16 tensor-core precision (XTSG_PREC_FP16): same
tcgen05 kind::f16 path with fp16 operands (10 mantissa bits instead of
bf16's 7), U scaled by 2^-s and W by 2^s to keep the mode-1 intermediate in
binary16 range, binary16 overflow -> HalfRangeError.

Stated tolerance: per replica relative Frobenius error <= 2e-3 against the
reference's fp64 comp (bf16: 1e-2); measured ~4e-4, i.e. ~8x below bf16.
"""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu
FP16_TOL = 2e-3


def _tensor(shape, seed, rank=4):
    rng = np.random.default_rng(seed)
    a, b, c = (rng.standard_normal((n, rank)) for n in shape)
    return np.asfortranarray(np.einsum("ir,jr,kr->ijk", a, b, c))


@pytest.mark.parametrize("dims,red,P", [
    ((256, 300, 72), (64, 64, 64), 4),
    ((200, 200, 40), (30, 30, 30), 12),
    ((130, 257, 20), (32, 32, 16), 5),
    ((192, 160, 8), (128, 128, 8), 2),
])
def test_fp16_plan_host_and_device_inputs(gpu, restated, dims, red, P):
    import torch
    ens = restated.make_ensemble(dims, red, P, 8, seed=21)
    t = _tensor(dims, 5)
    want = [restated.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, 8, 21, precision=gpu.PREC_FP16)
    errs = {}
    # host f64 (narrowed to fp16 on the host), device fp16 (direct TMA), device f32 (staged)
    y_host = gpu.Plan.replicas(plan.compress(t), P, red)
    xd = torch.from_numpy(t.ravel(order="F")).cuda().reshape(dims[2], dims[1], dims[0]).permute(2, 1, 0)
    y_h16 = gpu.Plan.replicas(plan.compress(xd.to(torch.float16)).cpu().numpy(), P, red)
    y_f32 = gpu.Plan.replicas(plan.compress(xd.to(torch.float32)).cpu().numpy(), P, red)
    for name, got in (("host", y_host), ("fp16", y_h16), ("f32", y_f32)):
        errs[name] = max(rel_diff(w, g) for w, g in zip(want, got))
    assert max(errs.values()) <= FP16_TOL, errs
    # bf16 on the same data for the record: fp16 must be clearly tighter
    bplan = gpu.Plan(dims, red, P, 8, 21, precision=gpu.PREC_BF16)
    yb = gpu.Plan.replicas(bplan.compress(t), P, red)
    eb = max(rel_diff(w, g) for w, g in zip(want, yb))
    assert errs["host"] < eb / 3, (errs, eb)


def test_fp16_factors_coo_and_large_i(gpu, restated):
    # large mode-1 extent exercises the 2^-s scaling of U (sum_i U X ~ sqrt(I))
    dims, red, P, R = (4096, 96, 40), (32, 32, 16), 4, 5
    a, b, c = restated.generate_dense(dims, R, 3)
    plan = gpu.Plan(dims, red, P, 8, 33, precision=gpu.PREC_FP16)
    ens = restated.make_ensemble(dims, red, P, 8, seed=33)
    got = gpu.Plan.replicas(plan.compress_factors((a, b, c)), P, red)
    for p in range(P):
        want = restated.comp_from_factors(a, b, c, ens[0][p], ens[1][p], ens[2][p])
        assert rel_diff(want, got[p]) <= FP16_TOL
    # sparse COO through the fp16 fiber kernel (fma.rn.f32.f16)
    rng = np.random.default_rng(4)
    n = 30000
    i = rng.integers(0, dims[0], n).astype(np.int32)
    j = rng.integers(0, dims[1], n).astype(np.int32)
    k = rng.integers(0, dims[2], n).astype(np.int32)
    v = rng.standard_normal(n).astype(np.float32)
    t = np.zeros(dims, order="F")
    np.add.at(t, (i, j, k), v.astype(np.float64))
    got = gpu.Plan.replicas(plan.compress_coo(i, j, k, v), P, red)
    for p in range(P):
        want = restated.comp(t, ens[0][p], ens[1][p], ens[2][p])
        assert rel_diff(want, got[p]) <= FP16_TOL


def test_fp16_overflow_is_half_range_error(gpu):
    dims, red, P = (64, 64, 16), (32, 32, 16), 2
    plan = gpu.Plan(dims, red, P, 4, 5, precision=gpu.PREC_FP16)
    t = np.ones(dims, order="F")
    t[3, 4, 5] = 1e6   # not representable in binary16
    with pytest.raises(gpu.HalfRangeError):
        plan.compress(t)


def test_fp16_pipeline_end_to_end(gpu):
    # decompose with fp16 compression: recovered factors tighter than bf16's
    dims, R = (120, 110, 100), 4
    f = gpu.generate_factors(dims, R, seed=5)
    errs = {}
    for name, prec in (("fp16", gpu.PREC_FP16), ("bf16", gpu.PREC_BF16)):
        cfg = gpu.PipelineConfig(reduced=(24, 24, 24), rank=R, seed=6, precision=prec, replica_fit_tol=1e-2)
        rec, met = gpu.decompose(cfg, factors=f)
        errs[name] = max(gpu.evaluate(f, rec).mode_rel_err)
    assert errs["fp16"] <= 2e-3 and errs["fp16"] < errs["bf16"], errs


def test_fp16_host_narrowing_matches_device_staging_bitwise(gpu):
    # host f32/f64 -> binary16 on the host (host_narrow.cpp f2h, RNE incl.
    # subnormals) == the device staging kernel's __float2half_rn
    import torch
    dims, red, P = (160, 96, 20), (32, 32, 16), 4
    rng = np.random.default_rng(12)
    t = np.asfortranarray(rng.standard_normal(dims) * 30.0)
    t[0, 0, 0], t[1, 0, 0], t[2, 0, 0], t[3, 0, 0] = 3e-6, -6.1e-5, 65500.0, 2.9802322387695312e-08
    plan = gpu.Plan(dims, red, P, 8, 19, precision=gpu.PREC_FP16)
    for dt in (np.float32, np.float64):
        th = np.asfortranarray(t.astype(dt))
        y_host = plan.compress(th)
        xd = torch.from_numpy(th.ravel(order="F")).cuda().reshape(dims[2], dims[1], dims[0]).permute(2, 1, 0)
        y_dev = plan.compress(xd).cpu().numpy()
        assert np.array_equal(y_host, y_dev), dt
