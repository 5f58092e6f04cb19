"""GPU OMP (omp_recover, alignment.cpp:306-419) on dictionaries large enough
for the GPU-wide atom search (>= 4096 atoms), against a numpy restatement of
the reference's greedy loop (same selection rule, Cholesky growth, stopping)."""
import numpy as np
import pytest

from paper_2311_13693_b200._lib import check, lib, ptr

pytestmark = pytest.mark.gpu


def _omp_ref(Y, D, s, tol):
    # alignment.cpp:306-419 restated (numpy; small sizes only)
    rows, atoms = D.shape
    nrm = np.linalg.norm(D, axis=0)
    out = np.zeros((atoms, Y.shape[1]))
    for c in range(Y.shape[1]):
        y = Y[:, c]
        r = y.copy()
        act = []
        coef = np.zeros(0)
        while len(act) < s:
            if np.linalg.norm(r) <= tol:
                break
            corr = np.abs(D.T @ r) / nrm
            corr[act] = -1.0
            j = int(np.argmax(corr))          # first maximum
            if corr[j] <= 0.0:
                break
            Da = D[:, act + [j]]
            G = Da.T @ Da
            try:
                L = np.linalg.cholesky(G)
            except np.linalg.LinAlgError:
                break
            if L[-1, -1] ** 2 <= 1e-28:
                break
            act.append(j)
            coef = np.linalg.solve(G, Da.T @ y)
            r = y - Da @ coef
        out[act, c] = coef
    return out


# the last two: stacked systems taller than the 16-column residual batch fits
# in shared memory (batch shrinks to 14 / 7 columns)
@pytest.mark.parametrize("rows,atoms,ncols,s", [(128, 6000, 3, 8), (96, 20000, 18, 5),
                                                (2048, 5000, 20, 6), (4096, 4100, 9, 4)])
def test_wide_omp_matches_reference_loop(gpu, rows, atoms, ncols, s):
    rng = np.random.default_rng(atoms)
    D = np.asfortranarray(rng.standard_normal((rows, atoms)))
    X = np.zeros((atoms, ncols))
    for c in range(ncols):
        X[rng.choice(atoms, s, replace=False), c] = rng.choice([-1.0, 1.0], s) * (1 + rng.random(s))
    Y = np.asfortranarray(D @ X)
    out = np.zeros((atoms, ncols), order="F")
    check(lib.xtsg_omp_recover(ptr(Y), rows, ncols, ptr(D), atoms, s, 1e-9, ptr(out)))
    want = _omp_ref(Y, D, s, 1e-9)
    assert np.array_equal(np.nonzero(out)[0], np.nonzero(want)[0])
    assert np.abs(out - want).max() <= 1e-9 * np.abs(want).max()
    assert np.abs(out - X).max() <= 1e-9 * np.abs(X).max()    # exact recovery of s-sparse columns
