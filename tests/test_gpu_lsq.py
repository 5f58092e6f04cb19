"""Stacked least squares on the device vs /root/reference/proj/tests/test_alignment.cpp:195-231
and acceptance criterion 10 (acceptance.cpp:288-304)."""
import numpy as np
import pytest

from oracle.oracle import rel_diff

pytestmark = pytest.mark.gpu


def rmat(r, c, seed):
    from oracle.oracle import Restated
    return Restated().gen_gaussian(r, c, seed)


def test_scaled_identity_block(gpu):
    g = rmat(4, 2, 700)
    u = 2.0 * np.eye(4)
    sol = gpu.solve_stacked_ls([u @ g], [u])
    assert np.abs(sol - g).max() <= 1e-12


def test_noiseless_forward_model(gpu):
    g = rmat(20, 3, 710)
    us = [rmat(8, 20, 720 + p) for p in range(4)]
    sol = gpu.solve_stacked_ls([u @ g for u in us], us)
    assert rel_diff(g, sol) <= 1e-9


def test_hopeless_systems(gpu):
    g = rmat(20, 2, 730)
    u = rmat(8, 20, 731)
    f = u @ g
    with pytest.raises(gpu.IllPosedError):
        gpu.solve_stacked_ls([f], [u])
    with pytest.raises(gpu.IllPosedError) as e:
        gpu.solve_stacked_ls([f, f, f], [u, u, u])
    assert e.value.effective_rank <= 8
    with pytest.raises(gpu.UsageError):
        gpu.solve_stacked_ls([], [])
    with pytest.raises(gpu.UsageError):
        gpu.solve_stacked_ls([f], [u, u])


def test_acceptance_10(gpu):
    # 20 instances, I=40, L=10, P=6, worst relative error <= 1e-9
    worst = 0.0
    for seed in range(20):
        g = rmat(40, 3, 5000 + seed)
        us = [rmat(10, 40, 6000 + 10 * seed + p) for p in range(6)]
        sol = gpu.solve_stacked_ls([u @ g for u in us], us)
        worst = max(worst, rel_diff(g, sol))
    assert worst <= 1e-9


def test_config1_stack_rank(gpu, restated):
    # config 1 (200^3, P=12, L=30): S=20 anchors leave 140 distinct rows -> rank 140
    # (the reference fails the same way, tests/golden/decompose_c1.npz); S=10 solves
    for S, ok in [(10, True), (20, False)]:
        ens = restated.make_ensemble([200, 200, 200], [30, 30, 30], 12, S, seed=99)
        g = rmat(200, 10, 1)
        fs = [u @ g for u in ens[0]]
        if ok:
            assert rel_diff(g, gpu.solve_stacked_ls(fs, ens[0])) <= 1e-9
        else:
            with pytest.raises(gpu.IllPosedError) as e:
                gpu.solve_stacked_ls(fs, ens[0])
            assert e.value.effective_rank == 140


def test_large_stack_matches_numpy(gpu):
    rng = np.random.default_rng(1)
    us = [rng.standard_normal((64, 700)) for _ in range(12)]
    g = rng.standard_normal((700, 20))
    sol = gpu.solve_stacked_ls([u @ g for u in us], us)
    assert rel_diff(g, sol) <= 1e-9


# ---- large stacks take the normal-equations fast path (blocked Cholesky with
# refinement, lsq.cu lsq_chol_dev); rank-deficient ones fall back to the
# column-pivoted QR and report the reference's rank

def _stack(cols, P, L, S, seed):
    from oracle.oracle import Restated
    ens = Restated().make_ensemble([cols, 16, 16], [L, 8, 8], P, S, seed=seed)
    return ens[0]


def test_large_stack_fast_path_matches_reference(gpu, reference):
    us = _stack(640, 12, 64, 8, 5)            # 768 x 640, well conditioned
    g = rmat(640, 7, 901)
    rng = np.random.default_rng(3)
    fs = [u @ g + 1e-3 * rng.standard_normal((u.shape[0], 7)) for u in us]   # inconsistent system
    sol = gpu.solve_stacked_ls(fs, us)
    rc, _, want = reference.solve_stacked_ls(fs, us)
    assert rc == 0
    assert rel_diff(want, sol) <= 1e-9


def test_large_rank_deficient_falls_back_to_qr(gpu, reference):
    us = _stack(600, 12, 64, 40, 6)           # 12 * 24 + 40 = 328 distinct rows < 600
    g = rmat(600, 3, 902)
    fs = [u @ g for u in us]
    with pytest.raises(gpu.IllPosedError) as e:
        gpu.solve_stacked_ls(fs, us)
    rc, rank, _ = reference.solve_stacked_ls(fs, us)
    assert rc != 0 and e.value.effective_rank == rank == 328
