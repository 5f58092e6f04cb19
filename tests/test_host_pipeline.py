"""Host-side pieces of the pipeline that need no device: synthetic factor
generation (generate, pipeline.cpp:157-207) bit-exact against the reference
build, and evaluate (pipeline.cpp:577-609) against the reference's."""
import numpy as np


def test_generate_factors_bit_exact(xt, reference):
    for law, nnz in [("dense", 0), ("sparse", 7), ("sparse", 0)]:
        got = xt.generate_factors((50, 40, 300), 5, law=law, nnz_per_col=nnz, seed=9)
        want = reference.generate((50, 40, 300), 5, 9, law=0 if law == "dense" else 1, nnz_per_col=nnz)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def test_generate_factors_errors(xt):
    import pytest
    with pytest.raises(xt.UsageError):
        xt.generate_factors((10, 10, 10), 0)
    with pytest.raises(xt.UsageError):
        xt.generate_factors((10, 10, 10), 2, law="sparse", nnz_per_col=11)


def test_evaluate_matches_reference(xt, reference):
    f = xt.generate_factors((30, 40, 50), 4, seed=5)
    rng = np.random.default_rng(0)
    perm = [2, 0, 3, 1]
    rec = tuple(np.asfortranarray(x[:, perm] * np.array([2.0, -1.0, 0.5, 3.0])
                                  + 1e-6 * rng.standard_normal(x.shape)) for x in f)
    rep = xt.evaluate(f, rec)
    errs, mse = reference.evaluate(f, rec)
    assert np.allclose(rep.mode_rel_err, errs, rtol=1e-12, atol=0)
    assert abs(rep.sample_mse - mse) <= 1e-12 * mse + 1e-300
    # the aligned factors undo the permutation and scaling
    for m in range(3):
        assert np.abs(rep.aligned[m] - f[m]).max() < 1e-4
