"""Pin the CPU oracle before trusting it (CPU-only, no GPU).

Known-answer tests are the reference's own (file:line cited); the restated
oracle is additionally checked bit-for-bit against the reference compiled in
place (oracle/_ref) and against the committed golden vectors.
"""
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_splitmix_canonical_value(restated):
    # canonical splitmix64 first output for seed 0
    assert int(restated.rng_u64(0, 1)[0]) == 0xE220A8397B1DCDAF


def test_replica_count_kats(restated):
    # test_compression.cpp:15-21
    assert restated.replica_count([1000] * 3, [50] * 3, 10) == 31
    assert restated.replica_count([300] * 3, [50] * 3, 0) == 7
    assert restated.replica_count([20] * 3, [20] * 3, 0) == 1
    assert restated.replica_count([10] * 3, [12, 10, 10], 0) == -1
    assert restated.replica_count([10] * 3, [2, 10, 10], 0) == -1


def test_gaussian_statistics(restated):
    # test_compression.cpp:23-38
    a = restated.gen_gaussian(100, 100, 7)
    assert np.array_equal(a, restated.gen_gaussian(100, 100, 7))
    assert not np.array_equal(a, restated.gen_gaussian(100, 100, 8))
    assert abs(a.mean()) <= 0.05 and 0.9 <= a.var() <= 1.1


def test_sparse_law(restated):
    # test_compression.cpp:40-56
    m = restated.gen_sparse(100, 100, 4.0, 3)
    assert set(np.unique(m)) <= {-2.0, 0.0, 2.0}
    assert 0.20 <= np.count_nonzero(m) / 1e4 <= 0.30
    d = restated.gen_sparse(10, 10, 1.0, 4)
    assert set(np.unique(d)) <= {-1.0, 1.0}


def test_anchor_rows_shared_and_stable(restated):
    # test_compression.cpp:69-88
    u, v, w = restated.make_ensemble([12, 11, 10], [5, 4, 4], 3, 2, seed=17)
    for p in range(1, 3):
        assert np.array_equal(u[0][:2], u[p][:2])
        assert np.array_equal(v[0][:2], v[p][:2])
        assert np.array_equal(w[0][:2], w[p][:2])
    assert u[0][3, 0] != u[1][3, 0]
    two = restated.make_ensemble([12, 11, 10], [5, 4, 4], 2, 2, seed=17)
    three = restated.make_ensemble([12, 11, 10], [5, 4, 4], 2, 3, seed=17)
    assert np.array_equal(two[0][0][4], three[0][0][4])
    assert np.array_equal(two[0][0][1], three[0][0][1])


def test_comp_identity_and_singleton(restated):
    # test_compression.cpp:125-140
    t = np.asfortranarray(np.random.default_rng(31).standard_normal((4, 5, 6)))
    y = restated.comp(t, np.eye(4), np.eye(5), np.eye(6))
    assert np.array_equal(y, t)
    y = restated.comp(np.full((1, 1, 1), 2.0), [[3.0]], [[5.0]], [[7.0]])
    assert y[0, 0, 0] == 210.0


def test_comp_matches_triple_sum(restated):
    # test_compression.cpp:142-152 (1e-10 abs)
    for seed in range(3):
        rng = np.random.default_rng(40 + seed)
        t = np.asfortranarray(rng.standard_normal((6, 7, 8)))
        u, v, w = (restated.gen_gaussian(3, n, 50 + 10 * k + seed) for k, n in enumerate((6, 7, 8)))
        assert np.abs(restated.comp(t, u, v, w) - restated.comp_triple_sum(t, u, v, w)).max() <= 1e-10


def test_factored_equals_materialized(restated):
    # test_compression.cpp:202-215
    rng = np.random.default_rng(301)
    a, b, c = rng.standard_normal((9, 2)), rng.standard_normal((8, 2)), rng.standard_normal((7, 2))
    u, v, w = restated.gen_gaussian(4, 9, 304), restated.gen_gaussian(4, 8, 305), restated.gen_gaussian(3, 7, 306)
    direct = restated.comp_from_factors(a, b, c, u, v, w)
    via = restated.comp(restated.reconstruct(a, b, c), u, v, w)
    assert np.abs(direct - via).max() <= 1e-10


@pytest.mark.parametrize("kind,kw", [(0, {}), (1, {"s": 4.0})])
def test_restated_ensemble_bitexact_vs_reference(restated, reference, kind, kw):
    for dims, red, P, S, seed in [([200, 190, 180], [30, 31, 32], 12, 10, 77), ([64, 70, 33], [8, 9, 10], 3, 2, 9)]:
        mine = restated.make_ensemble(dims, red, P, S, seed=seed, kind=kind, **kw)
        ref = reference.make_ensemble(dims, red, P, S, seed=seed, kind=kind, **kw)
        for m in range(3):
            for a, b in zip(mine[m], ref[m]):
                assert np.array_equal(a, b)


def test_restated_two_stage_vs_reference(restated, reference):
    mine = restated.make_ensemble([100, 100, 100], [50, 50, 50], 2, 2, seed=23, kind=2, inner_kind=1, inner_s=1.25)
    ref = reference.make_ensemble([100, 100, 100], [50, 50, 50], 2, 2, seed=23, kind=2, inner_kind=1, inner_s=1.25)
    for m in range(3):
        for a, b in zip(mine[m], ref[m]):
            assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())


def test_restated_rng_and_log_vs_reference(restated, reference):
    assert np.array_equal(restated.rng_normal(12345, 100000), reference.rng_normal(12345, 100000))


def test_restated_comp_vs_reference(restated, reference):
    rng = np.random.default_rng(5)
    t = np.asfortranarray(rng.standard_normal((9, 8, 7)))
    u, v, w = rng.standard_normal((4, 9)), rng.standard_normal((3, 8)), rng.standard_normal((5, 7))
    assert np.abs(restated.comp(t, u, v, w) - reference.comp(t, u, v, w)).max() <= 1e-12


def test_golden_vectors_match_oracle(restated):
    g = np.load(GOLDEN / "ensembles.npz")
    for key in g.files:
        if not key.startswith("ens_"):
            continue
        _, tag, mode, p = key.split("_")
        cfg = _golden_cfgs()[tag]
        ens = restated.make_ensemble(cfg["dims"], cfg["red"], cfg["P"], cfg["S"], seed=cfg["seed"],
                                     kind=cfg["kind"], s=cfg.get("s", 1.0))
        assert np.array_equal(ens[int(mode)][int(p)], g[key]), key


def _golden_cfgs():
    from tests.golden.make_golden import CONFIGS
    return CONFIGS


# ---- precision model (half.cpp / mixed.cpp): restatement pinned bitwise ----

def test_half_bits_restatement_matches_reference(restated, reference):
    from tests.test_gpu_mixed import TABLE
    for v, bits in TABLE:                       # test_mixed_precision.cpp:15-48
        assert restated.half_bits(v) == bits == reference.half_bits(v)
    rng = np.random.default_rng(42)
    xs = np.concatenate([rng.standard_normal(1000) * np.exp2(rng.integers(-30, 18, 1000)),
                         [65519.0, 65520.0, 65536.0, np.nan, np.inf, -1e300, 2.9802322387695312e-08]])
    for x in xs:
        assert restated.half_bits(x) == reference.half_bits(x), x


def test_comp_mixed_restatement_bitexact(restated, reference):
    rng = np.random.default_rng(5)
    t = np.asfortranarray(rng.standard_normal((9, 7, 6)))
    u, v, w = rng.standard_normal((3, 9)), rng.standard_normal((4, 7)), rng.standard_normal((2, 6))
    for stored in (False, True):
        parts = [restated.split(a, 2 if stored else 1) for a in (t, u, v, w)]
        for a, (h, r) in zip((t, u, v, w), parts):
            rh, rr = reference.split(a, 2 if stored else 1)
            assert np.array_equal(h, rh) and np.array_equal(r, rr)
        assert np.array_equal(restated.comp_mixed(*parts), reference.comp_mixed(t, u, v, w, stored))
    rounded = [restated.split(a, 0)[0] for a in (t, u, v, w)]
    assert np.array_equal(restated.comp_half(*rounded), reference.comp_naive_half(t, u, v, w))


def test_ensemble_cols_matches_make_ensemble(restated):
    """or_gen_replica_cols (column subsets, threaded) == or_make_ensemble."""
    for kind, s in ((0, 1.0), (1, 3.0)):
        dims, red, P, S, seed = (50, 40, 30), (6, 5, 4), 3, 2, 7
        full = restated.make_ensemble(dims, red, P, S, seed, kind=kind, s=s)
        sub = restated.ensemble_cols(dims, red, P, S, seed, kind=kind, s=s)
        assert all(np.array_equal(full[m][p], sub[m][p]) for m in range(3) for p in range(P))
        idx = [np.array([0, 3, 17, 49]), None, np.array([29])]
        sub2 = restated.ensemble_cols(dims, red, P, S, seed, cols=idx, kind=kind, s=s)
        assert np.array_equal(sub2[0][1], full[0][1][:, idx[0]])
        assert np.array_equal(sub2[1][2], full[1][2])
        assert np.array_equal(sub2[2][2], full[2][2][:, [29]])
