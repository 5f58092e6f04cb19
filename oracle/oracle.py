"""TEST INFRASTRUCTURE ONLY — parity oracle for the xtsg compression path.

Two layers, both CPU-only and never used by the product:

* ``Restated``: ctypes binding of ``oracle/xts_oracle.c`` (plain-C restatement
  of the reference RNG / make_ensemble / comp / comp_from_factors /
  reconstruct, each citing the reference file:line) plus numpy restatements of
  the dense linear-algebra steps further down the path (cp_als, stacked least
  squares, alignment) in this module.
* ``Reference``: ctypes binding of ``oracle/_ref/libxts_ref.so`` — the
  reference's own sources compiled in place (oracle/ref_build/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATED_SO = HERE / "_build" / "libxts_oracle.so"
REF_SO = HERE / "_ref" / "libxts_ref.so"

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


class Restated:
    def __init__(self):
        if not RESTATED_SO.exists():
            build()
        L = C.CDLL(str(RESTATED_SO))
        sig = {
            "or_derive": (_U64, [_U64, _U64]),
            "or_rng_u64": (None, [_U64, _I64, _P]),
            "or_rng_normal": (None, [_U64, _I64, _P]),
            "or_replica_count": (_I64, [_P, _P, _I64]),
            "or_gen_gaussian": (None, [_I64, _I64, _U64, _P]),
            "or_gen_sparse": (None, [_I64, _I64, _D, _U64, _P]),
            "or_make_ensemble": (None, [_P, _P, _I64, _I64, C.c_int, _D, C.c_int, _D, _P, _U64, _P, _P, _P]),
            "or_gen_replica_cols": (None, [_I64, _I64, _I64, C.c_int, _D, _U64, _U64, _U64, _I64, _P, _P]),
            "or_comp": (None, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "or_reconstruct": (None, [_P, _P, _P, _I64, _I64, _I64, _I64, _P]),
            "or_comp_from_factors": (None, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "or_comp_triple_sum": (None, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "or_generate_dense": (None, [_P, _I64, _U64, _P, _P, _P]),
            "or_half_bits": (C.c_int32, [_D]),
            "or_split": (C.c_int, [_P, _I64, C.c_int, _P, _P]),
            "or_comp_half": (None, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "or_comp_mixed": (None, [_P, _P, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P]),
        }
        for n, (r, a) in sig.items():
            fn = getattr(L, n)
            fn.restype = r
            fn.argtypes = a
        self.L = L

    def derive(self, seed, tag):
        return int(self.L.or_derive(seed, tag))

    def rng_u64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.L.or_rng_u64(seed, n, _ptr(out))
        return out

    def rng_normal(self, seed, n):
        out = np.zeros(n)
        self.L.or_rng_normal(seed, n, _ptr(out))
        return out

    def replica_count(self, dims, red, slack):
        return int(self.L.or_replica_count(_ptr(np.asarray(dims, np.int64)), _ptr(np.asarray(red, np.int64)), slack))

    def gen_gaussian(self, rows, cols, seed):
        out = np.zeros((rows, cols), order="F")
        self.L.or_gen_gaussian(rows, cols, seed, _ptr(out))
        return out

    def gen_sparse(self, rows, cols, s, seed):
        out = np.zeros((rows, cols), order="F")
        self.L.or_gen_sparse(rows, cols, s, seed, _ptr(out))
        return out

    def make_ensemble(self, dims, red, count, shared, seed, kind=0, s=1.0, inner_kind=1, inner_s=1.0,
                      ratios=(1.6, 1.6, 1.6)):
        dims = np.asarray(dims, np.int64)
        red = np.asarray(red, np.int64)
        inner = np.asarray([int(np.floor(ratios[m] * red[m] + 0.5)) for m in range(3)], np.int64)
        bufs = [np.zeros(count * red[m] * dims[m]) for m in range(3)]
        self.L.or_make_ensemble(_ptr(dims), _ptr(red), count, shared, kind, s, inner_kind, inner_s, _ptr(inner),
                                seed, *[_ptr(b) for b in bufs])
        per = [int(red[m] * dims[m]) for m in range(3)]
        return [[bufs[m][p * per[m]:(p + 1) * per[m]].reshape(int(red[m]), int(dims[m]), order="F")
                 for p in range(count)] for m in range(3)]

    def ensemble_cols(self, dims, red, count, shared, seed, cols=None, kind=0, s=1.0, threads=None):
        """make_ensemble (gaussian/sparse kinds, compression.cpp:115-155)
        restricted to the columns cols[m] (sorted int64 indices; None = all)
        of each mode; the (mode, replica) matrices are generated on a thread
        pool (ctypes releases the GIL). Returns [mode][p] -> red[m] x len(cols[m])."""
        from concurrent.futures import ThreadPoolExecutor
        import os
        cols = [np.arange(int(dims[m]), dtype=np.int64) if cols is None or cols[m] is None
                else np.ascontiguousarray(cols[m], dtype=np.int64) for m in range(3)]
        out = [[np.zeros((int(red[m]), len(cols[m])), order="F") for _ in range(count)] for m in range(3)]

        def one(mp):
            m, p = mp
            self.L.or_gen_replica_cols(int(red[m]), p, shared, kind, s, self.derive(seed, 101 + m), seed, m,
                                       len(cols[m]), _ptr(cols[m]), _ptr(out[m][p]))

        with ThreadPoolExecutor(threads or os.cpu_count() or 4) as ex:
            list(ex.map(one, [(m, p) for m in range(3) for p in range(count)]))
        return out

    def comp(self, t, u, v, w):
        t, u, v, w = _f(t), _f(u), _f(v), _f(w)
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self.L.or_comp(_ptr(t), *t.shape, _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w), w.shape[0], _ptr(y))
        return y

    def comp_triple_sum(self, t, u, v, w):
        t, u, v, w = _f(t), _f(u), _f(v), _f(w)
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self.L.or_comp_triple_sum(_ptr(t), *t.shape, _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w),
                                  w.shape[0], _ptr(y))
        return y

    def reconstruct(self, a, b, c):
        a, b, c = _f(a), _f(b), _f(c)
        out = np.zeros((a.shape[0], b.shape[0], c.shape[0]), order="F")
        self.L.or_reconstruct(_ptr(a), _ptr(b), _ptr(c), a.shape[0], b.shape[0], c.shape[0], a.shape[1], _ptr(out))
        return out

    def comp_from_factors(self, a, b, c, u, v, w):
        a, b, c, u, v, w = map(_f, (a, b, c, u, v, w))
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self.L.or_comp_from_factors(_ptr(a), _ptr(b), _ptr(c), a.shape[0], b.shape[0], c.shape[0], a.shape[1],
                                    _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w), w.shape[0], _ptr(y))
        return y

    def half_bits(self, x):
        """double_to_half_bits (half.cpp:10-47); None for HalfRangeError."""
        b = self.L.or_half_bits(float(x))
        return None if b < 0 else b

    def split(self, x, mode):
        """mode 0 round_to_half, 1 fp16_split, 2 fp16_split_stored (mixed.cpp:11-61)."""
        x = _f(x)
        half = np.zeros(x.shape, order="F")
        res = np.zeros(x.shape, order="F")
        if self.L.or_split(_ptr(x), x.size, mode, _ptr(half), _ptr(res)):
            raise OverflowError("HalfRangeError")
        return half, res

    def comp_half(self, t, u, v, w):
        t, u, v, w = _f(t), _f(u), _f(v), _f(w)
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self.L.or_comp_half(_ptr(t), *t.shape, _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w), w.shape[0],
                            _ptr(y))
        return y

    def comp_mixed(self, t, u, v, w):
        """comp_mixed from (half, residual) pairs."""
        (th, tr), (uh, ur), (vh, vr), (wh, wr) = [(_f(a), _f(b)) for a, b in (t, u, v, w)]
        y = np.zeros((uh.shape[0], vh.shape[0], wh.shape[0]), order="F")
        self.L.or_comp_mixed(_ptr(th), _ptr(tr), *th.shape, _ptr(uh), _ptr(ur), uh.shape[0], _ptr(vh), _ptr(vr),
                             vh.shape[0], _ptr(wh), _ptr(wr), wh.shape[0], _ptr(y))
        return y

    def generate_dense(self, dims, rank, seed):
        a = np.zeros((dims[0], rank), order="F")
        b = np.zeros((dims[1], rank), order="F")
        c = np.zeros((dims[2], rank), order="F")
        self.L.or_generate_dense(_ptr(np.asarray(dims, np.int64)), rank, seed, _ptr(a), _ptr(b), _ptr(c))
        return a, b, c


class Reference:
    """The reference library itself (compiled in place from /root/reference)."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing (build in a container that has /root/reference)")
        L = C.CDLL(str(REF_SO))
        sig = {
            "xref_last_payload": (_I64, []),
            "xref_set_blas_threads": (None, [C.c_int]),
            "xref_rng_u64": (None, [_U64, _I64, _P]),
            "xref_rng_normal": (None, [_U64, _I64, _P]),
            "xref_derive": (_U64, [_U64, _U64]),
            "xref_log_many": (None, [_P, _I64, _P]),
            "xref_replica_count": (C.c_int, [_P, _P, _I64, _P]),
            "xref_gen_gaussian": (C.c_int, [_I64, _I64, _U64, _P]),
            "xref_gen_sparse_projection": (C.c_int, [_I64, _I64, _D, _U64, _P]),
            "xref_make_ensemble": (C.c_int, [_P, _P, _I64, _I64, C.c_int, _D, _D, _D, _D, C.c_int, _D, _U64]
                                   + [_P] * 9),
            "xref_comp": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "xref_comp_mixed": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, C.c_int, _P]),
            "xref_comp_from_factors": (C.c_int, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64, _P,
                                                 _I64, _P]),
            "xref_reconstruct": (C.c_int, [_P, _P, _P, _I64, _I64, _I64, _I64, _P]),
            "xref_comp_blocked": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P, _P, C.c_int, C.c_int, _P]),
            "xref_cp_als": (C.c_int, [_P, _I64, _I64, _I64, _I64, _I64, _D, _U64, C.c_int, _P, _P, _P, _P, _P,
                                      _P]),
            "xref_relative_error": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _I64, _P]),
            "xref_solve_stacked_ls": (C.c_int, [_I64, _P, _I64, _I64, _P, _P, _P]),
            "xref_max_trace_assignment": (C.c_int, [_P, _I64, _P]),
            "xref_normalize_shared": (C.c_int, [_P, _I64, _I64, _I64, _P, _P]),
            "xref_align_replicas": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P]),
            "xref_recover_perm_scale": (C.c_int, [_P, _P, _I64, _I64, _P, _P]),
            "xref_generate": (C.c_int, [_P, _I64, C.c_int, _I64, _U64, _P, _P, _P]),
            "xref_decompose": (C.c_int, [_P, _P, _P, _P, _I64, _P, _P, _P, _U64, _P, _P, _P, _P]),
            "xref_evaluate": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
            "xref_double_to_half_bits": (C.c_int, [_D, _P]),
            "xref_write_tensor_file": (C.c_int, [C.c_char_p, _P, _I64, _I64, _I64]),
            "xref_write_factor_file": (C.c_int, [C.c_char_p, _P, _P, _P, _I64, _I64, _I64, _I64]),
            "xref_split": (C.c_int, [_P, _I64, C.c_int, _P, _P]),
            "xref_half_gemm": (C.c_int, [_P, _I64, _I64, _P, _I64, _P]),
            "xref_comp_half": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "xref_comp_naive_half": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
            "xref_comp_mixed": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, C.c_int, _P]),
        }
        for n, (r, a) in sig.items():
            fn = getattr(L, n)
            fn.restype = r
            fn.argtypes = a
        self.L = L

    def _ok(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"reference {what} failed with status {rc} (payload {self.L.xref_last_payload()})")

    def rng_normal(self, seed, n):
        out = np.zeros(n)
        self.L.xref_rng_normal(seed, n, _ptr(out))
        return out

    def log_many(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros_like(x)
        self.L.xref_log_many(_ptr(x), x.size, _ptr(out))
        return out

    def make_ensemble(self, dims, red, count, shared, seed, kind=0, s=1.0, alpha=1.6, beta=1.6, gamma=1.6,
                      inner_kind=1, inner_s=1.0):
        dims = np.asarray(dims, np.int64)
        red = np.asarray(red, np.int64)
        bufs = [np.zeros(count * red[m] * dims[m]) for m in range(3)]
        self._ok(self.L.xref_make_ensemble(_ptr(dims), _ptr(red), count, shared, kind, s, alpha, beta, gamma,
                                           inner_kind, inner_s, seed, *[_ptr(b) for b in bufs],
                                           *([None] * 6)), "make_ensemble")
        per = [int(red[m] * dims[m]) for m in range(3)]
        return [[bufs[m][p * per[m]:(p + 1) * per[m]].reshape(int(red[m]), int(dims[m]), order="F")
                 for p in range(count)] for m in range(3)]

    def ensemble_cols(self, dims, red, count, shared, seed, cols=None, kind=0, s=1.0, threads=None):
        """make_ensemble (gaussian/sparse kinds, compression.cpp:115-155)
        restricted to the columns cols[m] (sorted int64 indices; None = all)
        of each mode; the (mode, replica) matrices are generated on a thread
        pool (ctypes releases the GIL). Returns [mode][p] -> red[m] x len(cols[m])."""
        from concurrent.futures import ThreadPoolExecutor
        import os
        cols = [np.arange(int(dims[m]), dtype=np.int64) if cols is None or cols[m] is None
                else np.ascontiguousarray(cols[m], dtype=np.int64) for m in range(3)]
        out = [[np.zeros((int(red[m]), len(cols[m])), order="F") for _ in range(count)] for m in range(3)]

        def one(mp):
            m, p = mp
            self.L.or_gen_replica_cols(int(red[m]), p, shared, kind, s, self.derive(seed, 101 + m), seed, m,
                                       len(cols[m]), _ptr(cols[m]), _ptr(out[m][p]))

        with ThreadPoolExecutor(threads or os.cpu_count() or 4) as ex:
            list(ex.map(one, [(m, p) for m in range(3) for p in range(count)]))
        return out

    def comp(self, t, u, v, w):
        t, u, v, w = _f(t), _f(u), _f(v), _f(w)
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self._ok(self.L.xref_comp(_ptr(t), *t.shape, _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w),
                                  w.shape[0], _ptr(y)), "comp")
        return y

    def write_tensor_file(self, path, t):
        t = _f(t)
        self._ok(self.L.xref_write_tensor_file(str(path).encode(), _ptr(t), *t.shape), "write_tensor_file")

    def write_factor_file(self, path, a, b, c):
        a, b, c = _f(a), _f(b), _f(c)
        self._ok(self.L.xref_write_factor_file(str(path).encode(), _ptr(a), _ptr(b), _ptr(c), a.shape[0], b.shape[0],
                                               c.shape[0], a.shape[1]), "write_factor_file")

    def half_bits(self, x):
        out = np.zeros(1, np.uint16)
        rc = self.L.xref_double_to_half_bits(float(x), _ptr(out))
        return None if rc != 0 else int(out[0])

    def split(self, x, mode):
        x = _f(x)
        half = np.zeros(x.shape, order="F")
        res = np.zeros(x.shape, order="F")
        if self.L.xref_split(_ptr(x), x.size, mode, _ptr(half), _ptr(res)) != 0:
            raise OverflowError("HalfRangeError")
        return half, res

    def half_gemm(self, a, b):
        a, b = _f(a), _f(b)
        out = np.zeros((a.shape[0], b.shape[1]), order="F")
        self._ok(self.L.xref_half_gemm(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(out)),
                 "half_gemm")
        return out

    def _comp3(self, fn, t, u, v, w, *extra):
        t, u, v, w = _f(t), _f(u), _f(v), _f(w)
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self._ok(fn(_ptr(t), *t.shape, _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w), w.shape[0], *extra,
                    _ptr(y)), fn.__name__)
        return y

    def comp_half(self, t, u, v, w):
        return self._comp3(self.L.xref_comp_half, t, u, v, w)

    def comp_naive_half(self, t, u, v, w):
        return self._comp3(self.L.xref_comp_naive_half, t, u, v, w)

    def comp_mixed(self, t, u, v, w, stored_residual=False):
        """comp_mixed(split_tensor(t), split_matrix(u), ...) from the unsplit operands."""
        return self._comp3(self.L.xref_comp_mixed, t, u, v, w, int(stored_residual))

    def comp_from_factors(self, a, b, c, u, v, w):
        a, b, c, u, v, w = map(_f, (a, b, c, u, v, w))
        y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
        self._ok(self.L.xref_comp_from_factors(_ptr(a), _ptr(b), _ptr(c), a.shape[0], b.shape[0], c.shape[0],
                                               a.shape[1], _ptr(u), u.shape[0], _ptr(v), v.shape[0], _ptr(w),
                                               w.shape[0], _ptr(y)), "comp_from_factors")
        return y

    def comp_blocked(self, t, block, ens, deterministic=True, workers=1):
        t = _f(t)
        dims = np.asarray(t.shape, np.int64)
        P = len(ens[0])
        red = np.asarray([ens[0][0].shape[0], ens[1][0].shape[0], ens[2][0].shape[0]], np.int64)
        flat = [np.concatenate([x.ravel(order="F") for x in ens[m]]) for m in range(3)]
        y = np.zeros(P * int(np.prod(red)))
        self._ok(self.L.xref_comp_blocked(_ptr(t), _ptr(dims), _ptr(np.asarray(block, np.int64)), P, _ptr(red),
                                          *[_ptr(f) for f in flat], int(deterministic), workers, _ptr(y)),
                 "comp_blocked")
        n = int(np.prod(red))
        return [y[p * n:(p + 1) * n].reshape(tuple(red), order="F") for p in range(P)]

    def generate(self, dims, rank, seed, law=0, nnz_per_col=0):
        a = np.zeros((dims[0], rank), order="F")
        b = np.zeros((dims[1], rank), order="F")
        c = np.zeros((dims[2], rank), order="F")
        self._ok(self.L.xref_generate(_ptr(np.asarray(dims, np.int64)), rank, law, nnz_per_col, seed, _ptr(a),
                                      _ptr(b), _ptr(c)), "generate")
        return a, b, c

    def evaluate(self, truth, recovered):
        """pipeline.cpp:577-609 -> (mode_rel_err[3], sample_mse)"""
        t = [_f(x) for x in truth]
        r = [_f(x) for x in recovered]
        out = np.zeros(4)
        self._ok(self.L.xref_evaluate(_ptr(np.asarray([x.shape[0] for x in t], np.int64)), t[0].shape[1],
                                      *[_ptr(x) for x in t], *[_ptr(x) for x in r], _ptr(out)), "evaluate")
        return list(out[:3]), float(out[3])

    def cp_als(self, t, rank, max_iters=500, tol=1e-10, seed=0, init=0):
        t = _f(t)
        a = np.zeros((t.shape[0], rank), order="F")
        b = np.zeros((t.shape[1], rank), order="F")
        c = np.zeros((t.shape[2], rank), order="F")
        it = np.zeros(1, np.int64)
        conv = np.zeros(1, np.int32)
        hist = np.zeros(max_iters)
        self._ok(self.L.xref_cp_als(_ptr(t), *t.shape, rank, max_iters, tol, seed, init, _ptr(a), _ptr(b), _ptr(c),
                                    _ptr(it), _ptr(conv), _ptr(hist)), "cp_als")
        return (a, b, c), int(it[0]), list(hist[:int(it[0])]), bool(conv[0])

    def solve_stacked_ls(self, fs, us):
        fs = [_f(f) for f in fs]
        us = [_f(u) for u in us]
        rows = np.asarray([f.shape[0] for f in fs], np.int64)
        r, cols = fs[0].shape[1], us[0].shape[1]
        x = np.zeros((cols, r), order="F")
        rc = self.L.xref_solve_stacked_ls(len(fs), _ptr(rows), r, cols,
                                          _ptr(np.concatenate([f.ravel(order="F") for f in fs])),
                                          _ptr(np.concatenate([u.ravel(order="F") for u in us])), _ptr(x))
        return rc, int(self.L.xref_last_payload()), x

    def decompose(self, factors, dims, reduced, rank, replicas, shared, seed, tensor=None, block=(0, 0, 0),
                  mode=0, omp_sparsity=0, sample_b=0, precision=0, deterministic=0, als_max_iters=500,
                  als_restarts=3, workers=1, slack=10, alpha=1.6, beta=1.6, gamma=1.6, projection_s=0.0,
                  omp_tol=1e-9, als_tol=1e-10, fit_tol=1e-6):
        a, b, c = map(_f, factors)
        dims = np.asarray(dims, np.int64)
        cfg_i = np.asarray([reduced[0], reduced[1], reduced[2], rank, replicas, slack, shared, block[0], block[1],
                            block[2], mode, omp_sparsity, sample_b, precision, deterministic, als_max_iters,
                            als_restarts, workers], np.int64)
        cfg_d = np.asarray([alpha, beta, gamma, projection_s, omp_tol, als_tol, fit_tol], np.float64)
        oa, ob, oc = np.zeros_like(a), np.zeros_like(b), np.zeros_like(c)
        st = np.zeros(11)
        t = None if tensor is None else _f(tensor)
        rc = self.L.xref_decompose(_ptr(a), _ptr(b), _ptr(c), _ptr(dims), a.shape[1], _ptr(t), _ptr(cfg_i),
                                   _ptr(cfg_d), seed, _ptr(oa), _ptr(ob), _ptr(oc), _ptr(st))
        return rc, (oa, ob, oc), st


def rel_diff(a, b):
    """test_support.hpp:27-35"""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(a * a))
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))
