"""Out-of-core .xts source: header parsing on the host (no GPU)
and compression straight from disk on the GPU, against files written by the
reference's own writer (io.cpp:55-89, compiled in oracle/_ref)."""
import struct

import numpy as np
import pytest

from oracle.oracle import rel_diff


def _tensor(dims, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal(dims))


def test_header_of_reference_written_files(xt, reference, tmp_path):
    t = _tensor((5, 4, 3), 1)
    reference.write_tensor_file(tmp_path / "t.xts", t)
    assert xt.xts_header(tmp_path / "t.xts") == ("tensor", (5, 4, 3), 0)
    a, b, c = np.ones((6, 2)), np.ones((7, 2)), np.ones((8, 2))
    reference.write_factor_file(tmp_path / "f.xts", a, b, c)
    assert xt.xts_header(tmp_path / "f.xts") == ("factors", (6, 7, 8), 2)
    # the payload is the column-major doubles right after the 32-byte header
    raw = (tmp_path / "t.xts").read_bytes()
    assert len(raw) == 32 + 8 * t.size
    assert np.array_equal(np.frombuffer(raw[32:], np.float64), t.ravel(order="F"))


def test_header_errors_are_data_errors(xt, reference, tmp_path):
    t = _tensor((4, 4, 4), 2)
    reference.write_tensor_file(tmp_path / "t.xts", t)
    raw = (tmp_path / "t.xts").read_bytes()
    cases = {
        "magic": b"XTSX" + raw[4:],
        "version": raw[:4] + struct.pack("<H", 2) + raw[6:],
        "kind": raw[:6] + b"\x07" + raw[7:],
        "width": raw[:31] + b"\x04" + raw[32:],
        "truncated_payload": raw[:-8],
        "truncated_header": raw[:10],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.xts"
        p.write_bytes(data)
        with pytest.raises(xt.DataError):
            xt.xts_header(p)
    with pytest.raises(xt.DataError):
        xt.xts_header(tmp_path / "missing.xts")


@pytest.mark.gpu
def test_compress_file_dense_matches_in_memory(gpu, reference, restated, tmp_path):
    dims, red, P, S = (96, 80, 70), (32, 32, 16), 5, 8
    t = _tensor(dims, 3)
    path = tmp_path / "t.xts"
    reference.write_tensor_file(path, t)
    ens = restated.make_ensemble(dims, red, P, S, seed=11)
    for prec, tol in ((gpu.PREC_BF16, 1e-2), (gpu.PREC_FP64, 1e-10)):
        plan = gpu.Plan(dims, red, P, S, 11, precision=prec)
        # small slabs so the reader ring cycles (70 slices of 60 KB, ~3 per slab)
        y_file = plan.compress_file(path, slab_bytes=3 * 96 * 80 * 8)
        y_mem = plan.compress(t)
        got = gpu.Plan.replicas(y_file, P, red)
        for p in range(P):
            assert rel_diff(restated.comp(t, ens[0][p], ens[1][p], ens[2][p]), got[p]) <= tol
        assert rel_diff(y_mem, y_file) <= (1e-5 if prec == gpu.PREC_BF16 else 1e-13)
        # accumulate adds onto the caller's replicas
        y2 = plan.compress_file(path, y=y_file.copy(), accumulate=True)
        assert rel_diff(2 * y_file, y2) <= 1e-6
        plan.close()


@pytest.mark.gpu
def test_compress_file_factors_and_errors(gpu, reference, restated, tmp_path):
    dims, red, P, S, R = (128, 96, 64), (32, 32, 32), 4, 8, 5
    a, b, c = restated.generate_dense(dims, R, 9)
    reference.write_factor_file(tmp_path / "f.xts", a, b, c)
    plan = gpu.Plan(dims, red, P, S, 13)
    got = gpu.Plan.replicas(plan.compress_file(tmp_path / "f.xts"), P, red)
    ens = restated.make_ensemble(dims, red, P, S, seed=13)
    for p in range(P):
        assert rel_diff(restated.comp_from_factors(a, b, c, ens[0][p], ens[1][p], ens[2][p]), got[p]) <= 1e-2
    reference.write_tensor_file(tmp_path / "wrong.xts", _tensor((10, 10, 10), 1))
    with pytest.raises(gpu.UsageError):
        plan.compress_file(tmp_path / "wrong.xts")
    raw = (tmp_path / "f.xts").read_bytes()
    (tmp_path / "trunc.xts").write_bytes(raw[:-16])
    with pytest.raises(gpu.DataError):
        plan.compress_file(tmp_path / "trunc.xts")
