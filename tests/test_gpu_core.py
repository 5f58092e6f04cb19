"""GPU parity: RNG/ensembles bit-exact, fp64 compression chain vs the oracle.

Mirrors /root/reference/proj/tests/test_compression.cpp; tolerances are the
reference's own (cited per test).
"""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def test_golden_ensembles_bitexact(gpu):
    from tests.golden.make_golden import CONFIGS
    g = np.load(GOLDEN / "ensembles.npz")
    for tag, c in CONFIGS.items():
        ens = gpu.make_ensemble(c["dims"], c["red"], c["P"], c["S"], c["seed"],
                                kind="sparse" if c["kind"] == 1 else "gaussian", s=c.get("s", 1.0))
        for m, mats in enumerate((ens.u, ens.v, ens.w)):
            for p, mat in enumerate(mats):
                ref = g[f"ens_{tag}_{m}_{p}"]
                assert np.array_equal(mat, ref), (tag, m, p, np.abs(mat - ref).max())


def test_gen_gaussian_stream_bitexact(gpu, restated):
    for rows, cols, seed in [(100, 100, 7), (1, 1, 3), (37, 1001, 99), (1000, 20, 2**63 + 5)]:
        assert np.array_equal(gpu.gen_gaussian(rows, cols, seed), restated.gen_gaussian(rows, cols, seed))
    g = np.load(GOLDEN / "ensembles.npz")["normals_seed12345"]
    assert np.array_equal(gpu.gen_gaussian(4096, 1, 12345)[:, 0], g)


def test_gen_sparse_projection_bitexact(gpu, restated):
    for rows, cols, s, seed in [(100, 100, 4.0, 3), (10, 10, 1.0, 4), (20, 30, 4.0, 5)]:
        assert np.array_equal(gpu.gen_sparse_projection(rows, cols, s, seed), restated.gen_sparse(rows, cols, s, seed))


@pytest.mark.parametrize("dims,red,P,S,seed", [
    ([200, 200, 200], [30, 30, 30], 12, 10, 11),
    ([2000, 1999, 1003], [64, 63, 17], 3, 16, 2 ** 40 + 3),
    ([12, 11, 10], [5, 4, 4], 3, 2, 17),
    ([10007, 64, 64], [128, 32, 32], 2, 16, 99),
])
def test_make_ensemble_bitexact_large(gpu, restated, dims, red, P, S, seed):
    ens = gpu.make_ensemble(dims, red, P, S, seed)
    ref = restated.make_ensemble(dims, red, P, S, seed=seed)
    for m, mats in enumerate((ens.u, ens.v, ens.w)):
        for p in range(P):
            assert np.array_equal(mats[p], ref[m][p]), (m, p)


def test_make_ensemble_sparse_and_two_stage(gpu, restated):
    ens = gpu.make_ensemble([100, 90, 80], [10, 9, 8], 3, 2, 5, kind="sparse", s=4.0)
    ref = restated.make_ensemble([100, 90, 80], [10, 9, 8], 3, 2, seed=5, kind=1, s=4.0)
    for m, mats in enumerate((ens.u, ens.v, ens.w)):
        for p in range(3):
            assert np.array_equal(mats[p], ref[m][p])
    # two-stage: test_compression.cpp:103-123 shapes; u[p] == outer[p] * inner to fp64 rounding
    ens = gpu.make_ensemble([100, 100, 100], [50, 50, 50], 2, 2, 23, kind="two_stage", inner_kind="sparse",
                            inner_s=1.25)
    ts = ens.two_stage
    assert ts["inner"][0].shape == (80, 100) and ts["outer"][0][0].shape == (50, 80)
    ref = restated.make_ensemble([100, 100, 100], [50, 50, 50], 2, 2, seed=23, kind=2, inner_kind=1, inner_s=1.25)
    for p in range(2):
        assert np.abs(ens.u[p] - ref[0][p]).max() <= 1e-12 * np.abs(ref[0][p]).max()


def test_identity_singleton_and_oracle(gpu, restated):
    rng = np.random.default_rng(31)
    t = np.asfortranarray(rng.standard_normal((4, 5, 6)))
    assert np.array_equal(gpu.comp(t, np.eye(4), np.eye(5), np.eye(6)), t)   # :125-130
    y = gpu.comp(np.full((1, 1, 1), 2.0), [[3.0]], [[5.0]], [[7.0]])          # :132-140
    assert y[0, 0, 0] == 210.0
    for seed in range(3):                                                     # :142-152, 1e-10
        t = np.asfortranarray(np.random.default_rng(40 + seed).standard_normal((6, 7, 8)))
        u, v, w = gpu.gen_gaussian(3, 6, 50 + seed), gpu.gen_gaussian(3, 7, 60 + seed), gpu.gen_gaussian(3, 8, 70 + seed)
        assert np.abs(gpu.comp(t, u, v, w) - restated.comp_triple_sum(t, u, v, w)).max() <= 1e-10


def test_comp_golden_and_multilinear(gpu):
    g = np.load(GOLDEN / "comp.npz")
    from tests.golden.make_golden import CONFIGS
    c = CONFIGS["rag"]
    ens = gpu.make_ensemble(c["dims"], c["red"], c["P"], c["S"], c["seed"])
    for p in range(c["P"]):
        y = gpu.comp(g["t"], ens.u[p], ens.v[p], ens.w[p])
        assert np.abs(y - g[f"y_{p}"]).max() <= 1e-10
        yf = gpu.comp_from_factors((g["a"], g["b"], g["c"]), ens.u[p], ens.v[p], ens.w[p])
        assert np.abs(yf - g[f"yf_{p}"]).max() <= 1e-10 * max(1.0, np.abs(g[f"yf_{p}"]).max())
    # multilinearity, test_compression.cpp:154-170 (1e-12)
    rng = np.random.default_rng(81)
    x, yv = rng.standard_normal((5, 6, 7)), rng.standard_normal((5, 6, 7))
    u, v, w = rng.standard_normal((3, 5)), rng.standard_normal((3, 6)), rng.standard_normal((2, 7))
    lhs = gpu.comp(1.7 * x - 0.4 * yv, u, v, w)
    assert np.abs(lhs - 1.7 * gpu.comp(x, u, v, w) + 0.4 * gpu.comp(yv, u, v, w)).max() <= 1e-12


def test_kronecker_operator(gpu):
    # test_compression.cpp:172-185
    rng = np.random.default_rng(91)
    t = np.asfortranarray(rng.standard_normal((4, 3, 5)))
    u, v, w = rng.standard_normal((2, 4)), rng.standard_normal((3, 3)), rng.standard_normal((2, 5))
    y = gpu.comp(t, u, v, w)
    op = np.kron(np.kron(w, v), u)
    assert np.abs(op @ t.ravel(order="F") - y.ravel(order="F")).max() <= 1e-10


def test_reconstruct_bitexact(gpu, restated):
    rng = np.random.default_rng(7)
    a, b, c = rng.standard_normal((13, 5)), rng.standard_normal((11, 5)), rng.standard_normal((9, 5))
    assert np.array_equal(gpu.reconstruct(a, b, c), restated.reconstruct(a, b, c))


def _memory_source(t, block):
    # make_memory_block_source (compression.cpp:254-278): cells mode-1 fastest
    n = t.shape
    cells = [-(-n[m] // block[m]) for m in range(3)]
    for c3 in range(cells[2]):
        for c2 in range(cells[1]):
            for c1 in range(cells[0]):
                o = (c1 * block[0], c2 * block[1], c3 * block[2])
                yield (c1, c2, c3), t[o[0]:o[0] + block[0], o[1]:o[1] + block[1], o[2]:o[2] + block[2]]


def test_blocked_deterministic_bitwise_and_fast(gpu):
    # test_compression.cpp:251-287
    for seed in range(4):
        t = np.asfortranarray(np.random.default_rng(400 + seed).standard_normal((8, 8, 8)))
        ens = gpu.make_ensemble([8, 8, 8], [3, 3, 3], 2, 1, 500 + seed)
        direct = [gpu.comp(t, ens.u[p], ens.v[p], ens.w[p]) for p in range(2)]
        for block in ([4, 4, 4], [3, 3, 2], [8, 8, 8]):
            reps = gpu.comp_blocked([8, 8, 8], block, _memory_source(t, block), ens, deterministic=True)
            for p in range(2):
                assert np.array_equal(reps[p], direct[p])
    t = np.asfortranarray(np.random.default_rng(601).standard_normal((9, 8, 7)))
    ens = gpu.make_ensemble([9, 8, 7], [4, 3, 3], 3, 1, 602)
    reps = gpu.comp_blocked([9, 8, 7], [4, 3, 2], _memory_source(t, [4, 3, 2]), ens, deterministic=False)
    from oracle.oracle import rel_diff
    for p in range(3):
        assert rel_diff(reps[p], gpu.comp(t, ens.u[p], ens.v[p], ens.w[p])) <= 1e-12


def test_blocked_regions(gpu):
    # the facade's whole-tensor push of an untouched memory source: bitwise the
    # one-shot comp; regions mix with cell records, and keep the stream checks
    t = np.asfortranarray(np.random.default_rng(611).standard_normal((9, 8, 7)))
    ens = gpu.make_ensemble([9, 8, 7], [4, 3, 3], 3, 1, 612)
    direct = [gpu.comp(t, ens.u[p], ens.v[p], ens.w[p]) for p in range(3)]
    reps = gpu.comp_blocked([9, 8, 7], [4, 3, 2], [], ens, regions=[((0, 0, 0), t)])
    for p in range(3):
        assert np.array_equal(reps[p], direct[p])
    # k cells 0-1 as a region, the rest as records (ragged i/j edges inside the region)
    recs = [r for r in _memory_source(t, [4, 3, 2]) if r[0][2] >= 2]
    reps = gpu.comp_blocked([9, 8, 7], [4, 3, 2], recs, ens, regions=[((0, 0, 0), t[:, :, :4])])
    for p in range(3):
        assert np.array_equal(reps[p], direct[p])
    with pytest.raises(gpu.DataError):  # not on cell boundaries
        gpu.comp_blocked([9, 8, 7], [4, 3, 2], [], ens, regions=[((0, 0, 1), t[:, :, 1:])])
    with pytest.raises(gpu.DataError):  # a cell twice
        gpu.comp_blocked([9, 8, 7], [4, 3, 2], list(_memory_source(t, [4, 3, 2])), ens,
                         regions=[((0, 0, 0), t[:, :, :2])])
    # fast mode: a region is one big block (per-cell sum up to rounding)
    reps = gpu.comp_blocked([9, 8, 7], [4, 3, 2], recs, ens, deterministic=False, regions=[((0, 0, 0), t[:, :, :4])])
    from oracle.oracle import rel_diff
    for p in range(3):
        assert rel_diff(reps[p], direct[p]) <= 1e-12


def test_blocked_stream_faults(gpu):
    # test_compression.cpp:289-337
    t = np.asfortranarray(np.random.default_rng(621).standard_normal((6, 6, 6)))
    ens = gpu.make_ensemble([6, 6, 6], [3, 3, 3], 1, 1, 622)
    recs = list(_memory_source(t, [3, 3, 3]))
    with pytest.raises(gpu.DataError):
        gpu.comp_blocked([6, 6, 6], [3, 3, 3], recs[:2] + recs[3:], ens)
    with pytest.raises(gpu.DataError):
        gpu.comp_blocked([6, 6, 6], [3, 3, 3], recs[:1] + recs, ens)
    with pytest.raises(gpu.DataError):
        gpu.comp_blocked([6, 6, 6], [3, 3, 3], [((0, 0, 0), np.zeros((2, 3, 3)))], ens)
    with pytest.raises(gpu.UsageError):
        gpu.comp_blocked([7, 6, 6], [3, 3, 3], recs, ens)
