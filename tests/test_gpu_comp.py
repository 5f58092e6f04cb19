"""Compensated tensor-core compression (XTSG_PREC_FP16X3) against the fp64
oracle: the reference's Eq. 5 operand split (mixed.cpp:18-24: x = hi + lo,
the residual stored in fp16) carried onto tcgen05 — each mode product is
hi*hi + hi*lo + lo*hi over fp16 pairs. Every operand (U, V, each X launch,
the mode-1 result) is pre-scaled by a power of two that puts its largest
value in [2^13, 2^14), so lo stays a normal binary16 number and inputs of any
magnitude compress (the reference's mixed path, half.cpp, raises
HalfRangeError instead; that path is replayed bit-exactly in mixed.cu).

Stated tolerance: per-replica relative Frobenius error <= COMP_TOL vs the
reference's fp64 comp / comp_from_factors. What bounds it is the fp32
accumulation inside the tensor core (measured on B200: ~0.3 ulp of the
accumulator per MMA, growing linearly with the chain length), so the mode-1
sum runs in chunks of 8 i-steps (512 i) and the mode-2 sum in two chains of 24
MMAs per 256-wide j tile: measured 0.75e-6 (shortest chains) to 2.5e-6 (C2).
That is ~1300x below the bf16 path's 3.3e-3, and below the reference
pipeline's default replica fit tolerance (1e-6) in fit error, which the
pipeline test checks.
"""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu
COMP_TOL = 4e-6


def _errs(want, y, P, red):
    import torch
    y = y.cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
    n = int(np.prod(red))
    return [rel_diff(w, y[p * n:(p + 1) * n].reshape(red, order="F")) for p, w in enumerate(want)]


@pytest.mark.parametrize("dims,red,P,S", [
    ((256, 300, 72), (64, 64, 64), 4, 8),
    ((200, 200, 200), (30, 30, 30), 12, 10),     # config-1 shape: L pads to 32, rows pad to pairs
    ((130, 257, 20), (32, 32, 16), 5, 4),        # ragged i / j
    ((192, 160, 8), (128, 128, 8), 2, 4),        # L = 128
    ((1100, 96, 12), (64, 32, 12), 3, 4),        # three i chunks (the last one partial)
])
def test_comp_dense_vs_oracle(gpu, restated, dims, red, P, S):
    import torch
    seed = 41
    t = np.asfortranarray(np.random.default_rng(3).standard_normal(dims))
    ens = restated.make_ensemble(dims, red, P, S, seed)
    want = [restated.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, seed, precision=gpu.PREC_FP16X3)
    errs = _errs(want, plan.compress(t), P, red)          # host fp64 input
    assert max(errs) <= COMP_TOL, errs
    # device fp32 input
    xd = torch.from_numpy(np.asarray(t, np.float32).ravel(order="F")).cuda()
    xd = xd.reshape(dims[2], dims[1], dims[0]).permute(2, 1, 0)
    y = plan.compress(xd)
    torch.cuda.synchronize()
    want32 = [restated.comp(np.asarray(t, np.float32), ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    errs32 = _errs(want32, y, P, red)
    assert max(errs32) <= COMP_TOL, errs32
    plan.close()


def test_comp_blocks_accumulate(gpu, restated):
    """BlockGrid cells (unaligned i/j offsets) accumulate to the one-shot replicas."""
    dims, red, P, S = (200, 180, 30), (32, 32, 16), 4, 4
    t = np.asfortranarray(np.random.default_rng(5).standard_normal(dims))
    ens = restated.make_ensemble(dims, red, P, S, 9)
    want = [restated.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, 9, precision=gpu.PREC_FP16X3)
    y = None
    for i0, i1 in [(0, 77), (77, 200)]:
        for j0, j1 in [(0, 101), (101, 180)]:
            for k0, k1 in [(0, 13), (13, 30)]:
                blk = np.asfortranarray(t[i0:i1, j0:j1, k0:k1])
                y = plan.compress(blk, y=y, offset=(i0, j0, k0), accumulate=y is not None)
    errs = _errs(want, y, P, red)
    assert max(errs) <= COMP_TOL, errs
    plan.close()


def test_comp_factored_vs_comp_from_factors(gpu, restated):
    """Slabs generated on the device as fp16 pairs (600 x 500 x 300, P = 32 x 64^3)."""
    dims, red, P, S, R = (600, 500, 300), (64, 64, 64), 32, 40, 20
    seed = restated.derive(2, 11)
    f = restated.generate_dense(dims, R, 1)
    ens = restated.ensemble_cols(dims, red, P, S, seed)
    want = [restated.comp_from_factors(*f, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, seed, precision=gpu.PREC_FP16X3)
    errs = _errs(want, plan.compress_factors(f), P, red)
    assert max(errs) <= COMP_TOL, errs
    plan.close()


@pytest.mark.parametrize("scale,outlier", [(1.0, 1e6), (1e-9, None), (1e12, None)])
def test_comp_any_magnitude(gpu, restated, scale, outlier):
    """Values outside binary16 (an outlier at 1e6, a tensor at 1e12) and far
    below its normal range (1e-9) compress to the oracle's tolerance: the
    power-of-two pre-scale of each X launch keeps hi and lo in range."""
    dims, red, P, S, seed = (64, 64, 8), (32, 32, 8), 2, 4, 1
    t = np.asfortranarray(np.random.default_rng(0).standard_normal(dims)) * scale
    if outlier is not None:
        t[3, 4, 5] = outlier
    ens = restated.make_ensemble(dims, red, P, S, seed)
    want = [restated.comp(t, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, seed, precision=gpu.PREC_FP16X3)
    errs = _errs(want, plan.compress(t), P, red)
    assert max(errs) <= COMP_TOL, errs
    plan.close()


@pytest.mark.parametrize("scale", [1e-12, 1e9])
def test_comp_factored_any_magnitude(gpu, restated, scale):
    """Factored sources take X's pre-scale from the factor bound
    sum_r max|a_r| max|b_r| max|c_r| (no pass over the slabs); tiny and huge
    factors compress to the same tolerance."""
    dims, red, P, S, R = (300, 260, 90), (32, 32, 32), 6, 8, 5
    seed = restated.derive(2, 11)
    a, b, c = restated.generate_dense(dims, R, 3)
    f = (np.asfortranarray(a * scale), b, c)
    ens = restated.ensemble_cols(dims, red, P, S, seed)
    want = [restated.comp_from_factors(*f, ens[0][p], ens[1][p], ens[2][p]) for p in range(P)]
    plan = gpu.Plan(dims, red, P, S, seed, precision=gpu.PREC_FP16X3)
    errs = _errs(want, plan.compress_factors(f), P, red)
    assert max(errs) <= COMP_TOL, errs
    plan.close()


def test_comp_sparse_input_rejected(gpu):
    plan = gpu.Plan((64, 64, 8), (32, 32, 8), 2, 4, 1, precision=gpu.PREC_FP16X3)
    with pytest.raises(gpu.UsageError):
        plan.compress_coo(np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32), np.ones(1, np.float32))
    plan.close()


def test_comp_pipeline_at_default_fit_tolerance(gpu):
    """decompose with compensated compression keeps every replica at the
    reference's default replica_fit_tol = 1e-6 (pipeline.hpp:41), where the
    bf16 path loses all of them."""
    dims, R, L, S = (1000, 1000, 1000), 10, 64, 20
    f = gpu.generate_factors(dims, R, seed=1)
    cfg = gpu.PipelineConfig(reduced=(L, L, L), rank=R, shared=S, precision=gpu.PREC_FP16X3, seed=2)
    assert cfg.replica_fit_tol == 1e-6
    rec, met = gpu.decompose(cfg, factors=f)
    assert met.replicas_dropped == 0
    assert max(gpu.evaluate(f, rec).mode_rel_err) <= 1e-5
    cfg.precision = gpu.PREC_BF16
    with pytest.raises(gpu.StageError):
        gpu.decompose(cfg, factors=f)
