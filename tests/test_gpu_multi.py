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
