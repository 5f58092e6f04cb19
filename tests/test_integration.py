"""The reference's OWN unit tests and acceptance runner, compiled unchanged
(integration/Makefile) and linked against the drop-in: reference callers
(pipeline.cpp, mixed.cpp, ...) + the C++ facade over libxtsg.so in place of
compression.cpp / cp_als.cpp / alignment.cpp / linalg.cpp.

The CPU self-check links the same unchanged sources against the reference
itself, pinning the harness shims (doctest / test_support) to the reference's
logged results (proj/test_output.txt).
"""
import os
import re
import subprocess
from pathlib import Path

import pytest

B = Path(__file__).resolve().parents[1] / "integration" / "_build"
ENV = dict(os.environ, OPENBLAS_NUM_THREADS="1")


def _run(binary, timeout):
    if not (B / binary).exists():
        pytest.skip(f"{binary} not built (make -C integration needs /root/reference)")
    return subprocess.run([str(B / binary)], capture_output=True, text=True, timeout=timeout, env=ENV)


def _acceptance(out):
    res = {}
    for line in out.splitlines():
        m = re.match(r"(PASS|FAIL)\s+(\d+)\.", line)
        if m:
            res[int(m.group(2))] = m.group(1) == "PASS"
    return res


def test_harness_selfcheck_reference_unit_tests():
    r = _run("unit_tests_ref", 300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "102 passed | 0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_unit_tests_pass_against_dropin(gpu):
    r = _run("unit_tests", 900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_against_dropin(gpu):
    r = _run("acceptance", 1200)
    res = _acceptance(r.stdout)
    # criterion 7 fails in the reference itself (proj/test_output.txt:13): an
    # unattainable coherence precondition, independent of the compression path
    for crit in (1, 2, 3, 4, 5, 6, 8, 9, 10):
        assert res.get(crit), (crit, r.stdout)
    # criterion 8 runs comp_mixed / comp_naive_half on the device, bit-exact
    # with the reference, so the logged ratio is reproduced (test_output.txt:14)
    m = re.search(r"median error ratio ([0-9.eE+-]+)", r.stdout)
    assert m and abs(float(m.group(1)) - 0.000253996) < 5e-10, r.stdout


@pytest.mark.gpu
def test_facade_concurrent_cp_als_and_memory_source(gpu):
    # integration/facade_concurrency.cpp: 16 threads' cp_als calls batched by
    # the facade equal the same calls made alone (bitwise), a NaN tensor fails
    # only its own call; comp_blocked over an in-memory source == comp
    r = _run("facade_concurrency", 300)
    assert r.returncode == 0 and "facade_concurrency: ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
