"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/xtsg.h declares, maps the reference's error taxonomy, and
refuses compute without a device (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "xtsg.h").read_text()
    return sorted(set(re.findall(r"\b(xtsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(xt):
    syms = declared_symbols()
    assert len(syms) >= 25
    lib = C.CDLL(str(ROOT / "paper_2311_13693_b200" / "libxtsg.so"))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a(xt):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_2311_13693_b200" / "libxtsg.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_replica_count_and_errors(xt):
    # compression.cpp:82-95 and test_compression.cpp:15-21 (host arithmetic)
    assert xt.compute_replica_count([1000] * 3, [50] * 3, 10) == 31
    assert xt.compute_replica_count([300] * 3, [50] * 3, 0) == 7
    assert xt.compute_replica_count([20] * 3, [20] * 3, 0) == 1
    with pytest.raises(xt.UsageError):
        xt.compute_replica_count([10] * 3, [12, 10, 10], 0)
    with pytest.raises(xt.UsageError):
        xt.compute_replica_count([10] * 3, [2, 10, 10], 0)


def test_host_alignment_entry_points(xt):
    # alignment.cpp:87-144 vs exhaustive search (test_support.hpp:67-82)
    import itertools
    rng = np.random.default_rng(100)
    for _ in range(50):
        q = rng.standard_normal((5, 5))
        best = max(itertools.permutations(range(5)), key=lambda p: sum(q[r, p[r]] for r in range(5)))
        assert xt.max_trace_assignment(q) == list(best)
    m = np.array([[1.0], [-2.0], [4.0], [8.0]])
    norm, piv = xt.normalize_shared(m, 3)
    assert piv[0] == 4.0 and np.allclose(norm[:, 0], [0.25, -0.5, 1.0, 2.0])
    with pytest.raises(xt.DegenerateColumnError):
        xt.normalize_shared(np.array([[0.0, 1.0], [0.0, 0.0], [5.0, 0.0]]), 2)
    with pytest.raises(xt.UsageError):
        xt.normalize_shared(m, 0)


def test_no_cpu_fallback_without_device(xt):
    if xt.device_ready():
        pytest.skip("device present")
    with pytest.raises(xt.CudaError):
        xt.gen_gaussian(4, 4, 1)
    with pytest.raises(xt.CudaError):
        xt.comp(np.zeros((2, 2, 2)), np.eye(2), np.eye(2), np.eye(2))
    with pytest.raises(xt.CudaError):
        xt.Plan([64] * 3, [32] * 3, 4, 2, 1)


def test_usage_errors_precede_device_checks(xt):
    with pytest.raises(xt.UsageError):
        xt.gen_sparse_projection(100, 100, 40.0, 6)   # test_compression.cpp:61-63
    with pytest.raises(xt.UsageError):
        xt.gen_sparse_projection(10, 10, 0.5, 6)
    with pytest.raises(xt.UsageError):
        xt.make_ensemble([8, 8, 8], [9, 4, 4], 2, 1, 5)  # :98-100
    with pytest.raises(xt.UsageError):
        xt.make_ensemble([8, 8, 8], [4, 4, 4], 0, 1, 5)
    with pytest.raises(xt.UsageError):
        xt.make_ensemble([8, 8, 8], [4, 4, 4], 2, 5, 5)
    with pytest.raises(xt.UsageError):
        xt.make_ensemble([100] * 3, [50] * 3, 2, 2, 23, kind="two_stage", alpha=1.0)


def test_header_is_plain_c_and_cpp():
    # the drop-in boundary must compile as C (cgo/ctypes-style callers) and C++
    import subprocess
    import tempfile
    src = '#include "xtsg.h"\nint main(void) { xtsg_plan_desc d; (void)d; return xtsg_version() > 0 ? 0 : 1; }\n'
    with tempfile.TemporaryDirectory() as td:
        for cc, ext in (("gcc", "c"), ("g++", "cpp")):
            f = Path(td) / f"t.{ext}"
            f.write_text(src)
            r = subprocess.run([cc, "-std=c11" if ext == "c" else "-std=c++17", "-Wall", "-Werror", "-fsyntax-only",
                                "-I", str(ROOT / "include"), str(f)], capture_output=True, text=True)
            assert r.returncode == 0, (cc, r.stderr)


def test_coo_to_csf_host_helper(xt):
    rng = np.random.default_rng(5)
    n = 500
    i, j, k = (rng.integers(0, 9, n) for _ in range(3))
    v = rng.standard_normal(n).astype(np.float32)
    sk, sp, fj, fp, ni, nv = xt.Plan.coo_to_csf(i, j, k, v)
    assert sp[0] == 0 and sp[-1] == len(fj) and fp[0] == 0 and fp[-1] == n
    assert np.all(np.diff(sk) > 0)                      # one record per distinct k, sorted
    dense = np.zeros((9, 9, 9))
    np.add.at(dense, (i, j, k), v.astype(np.float64))
    back = np.zeros((9, 9, 9))
    for q, kk in enumerate(sk):
        for f in range(sp[q], sp[q + 1]):
            for e in range(fp[f], fp[f + 1]):
                back[ni[e], fj[f], kk] += nv[e]
    assert np.allclose(dense, back)
