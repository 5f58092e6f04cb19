"""Python mirror of the reference entry points over the xtsg C ABI.

Layout convention follows xts::Matrix / xts::Tensor3 (tensor.hpp:10-44):
matrices and tensors are numpy arrays in Fortran (column-major) order, so
``m[i, j]`` is the reference's ``m(i, j)`` and the memory image is identical.
Device-resident inputs (torch CUDA tensors) are passed through untouched.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from ._lib import (AlsConfig, EnsembleSpec, PlanDesc, PipelineConfigC, PipelineMetricsC, DTYPE_BF16,
                   DTYPE_F32, DTYPE_F64, KIND_GAUSSIAN, KIND_SPARSE, KIND_TWO_STAGE, LAW_DENSE, LAW_SPARSE,
                   MODE_DENSE, MODE_SPARSE, MODE_TWO_STAGE, PREC_BF16, PREC_FP64, DTYPE_F16, check, lib, ptr, UsageError)

_KINDS = {"gaussian": KIND_GAUSSIAN, "sparse": KIND_SPARSE, "two_stage": KIND_TWO_STAGE}


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _arr3(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64).reshape(3))


def device_ready() -> bool:
    return bool(lib.xtsg_device_ready())


def launch_count() -> int:
    return int(lib.xtsg_launch_count())


def compute_replica_count(dims, reduced, slack: int) -> int:
    """compression.cpp:82-95"""
    out = np.zeros(1, np.int64)
    check(lib.xtsg_replica_count(ptr(_arr3(dims)), ptr(_arr3(reduced)), int(slack), ptr(out)))
    return int(out[0])


def gen_gaussian(rows: int, cols: int, seed: int) -> np.ndarray:
    """compression.cpp:97-103"""
    out = np.zeros((max(rows, 0), max(cols, 0)), order="F")
    check(lib.xtsg_gen_gaussian(int(rows), int(cols), C.c_uint64(seed), ptr(out)))
    return out


def gen_sparse_projection(rows: int, cols: int, s: float, seed: int) -> np.ndarray:
    """compression.cpp:105-113"""
    out = np.zeros((max(rows, 0), max(cols, 0)), order="F")
    check(lib.xtsg_gen_sparse_projection(int(rows), int(cols), float(s), C.c_uint64(seed), ptr(out)))
    return out


def _spec(kind="gaussian", s=1.0, alpha=1.6, beta=1.6, gamma=1.6, inner_kind="sparse",
          inner_s=1.0) -> EnsembleSpec:
    k = _KINDS[kind] if isinstance(kind, str) else int(kind)
    ik = _KINDS[inner_kind] if isinstance(inner_kind, str) else int(inner_kind)
    return EnsembleSpec(k, ik, float(s), float(alpha), float(beta), float(gamma), float(inner_s))


@dataclass
class Ensemble:
    """CompressionEnsemble (compression.hpp:33-65)."""
    count: int
    shared_rows: int
    seed: int
    u: list
    v: list
    w: list
    two_stage: Optional[dict] = None


def make_ensemble(dims, reduced, count: int, shared_rows: int, seed: int, kind="gaussian",
                  **spec) -> Ensemble:
    """compression.cpp:115-200 (bit-exact on the device)."""
    dims, reduced = _arr3(dims), _arr3(reduced)
    sp = _spec(kind, **spec)
    P = max(int(count), 0)
    inner = outer = None
    if sp.kind == KIND_TWO_STAGE:
        ratio = [sp.alpha, sp.beta, sp.gamma]
        ir = [int(np.floor(ratio[m] * reduced[m] + 0.5)) for m in range(3)]
        inner = [np.zeros(ir[m] * int(dims[m])) for m in range(3)]
        outer = [np.zeros(P * int(reduced[m]) * ir[m]) for m in range(3)]
    raw = [np.zeros(P * int(reduced[m]) * int(dims[m])) for m in range(3)]
    args = raw + (inner if inner else [None] * 3) + (outer if outer else [None] * 3)
    check(lib.xtsg_make_ensemble(ptr(dims), ptr(reduced), int(count), int(shared_rows),
                                 C.byref(sp), C.c_uint64(seed), *[ptr(a) for a in args]))
    per = [int(reduced[m] * dims[m]) for m in range(3)]
    lists = [[raw[m][p * per[m]:(p + 1) * per[m]].reshape(int(reduced[m]), int(dims[m]), order="F")
              for p in range(P)] for m in range(3)]
    ts = None
    if inner:
        ts = {
            "inner": [inner[m].reshape(ir[m], int(dims[m]), order="F") for m in range(3)],
            "outer": [[outer[m][p * reduced[m] * ir[m]:(p + 1) * reduced[m] * ir[m]].reshape(
                int(reduced[m]), ir[m], order="F") for p in range(P)] for m in range(3)],
        }
    return Ensemble(int(count), int(shared_rows), int(seed), lists[0], lists[1], lists[2], ts)


def comp(t, u, v, w) -> np.ndarray:
    """compression.cpp:211-213 (fp64 on the device)."""
    t, u, v, w = _f64(t), _f64(u), _f64(v), _f64(w)
    if t.ndim != 3 or u.shape[1] != t.shape[0] or v.shape[1] != t.shape[1] or w.shape[1] != t.shape[2]:
        from ._lib import UsageError
        raise UsageError("comp: compression matrix columns must match tensor dims")
    y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
    check(lib.xtsg_comp(ptr(t), *t.shape, ptr(u), u.shape[0], ptr(v), v.shape[0], ptr(w),
                        w.shape[0], ptr(y)))
    return y


def _split(x, mode):
    x = _f64(x)
    half = np.zeros(x.shape, order="F")
    res = np.zeros(x.shape, order="F") if mode else None
    check(lib.xtsg_split_half(ptr(x), x.size, mode, ptr(half), ptr(res) if mode else None))
    return half, res


def round_to_half(x) -> np.ndarray:
    """round_matrix_to_half / round_tensor_to_half (mixed.cpp:47-61); HalfRangeError out of range."""
    return _split(x, 0)[0]


def split_half(x, stored_residual: bool = False):
    """split_matrix / split_tensor (mixed.cpp:27-45): (half, residual) arrays."""
    return _split(x, 2 if stored_residual else 1)


def half_gemm(a, b) -> np.ndarray:
    """half_gemm (mixed.cpp:63-76), bit-exact on the device."""
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0], b.shape[1]), order="F")
    check(lib.xtsg_half_gemm(ptr(a), a.shape[0], a.shape[1], ptr(b), b.shape[0], b.shape[1], ptr(out)))
    return out


def _comp_shapes(t, u, v, w):
    if t.ndim != 3 or u.shape[1] != t.shape[0] or v.shape[1] != t.shape[1] or w.shape[1] != t.shape[2]:
        from ._lib import UsageError
        raise UsageError("comp: compression matrix columns must match tensor dims")
    return np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")


def comp_half(t, u, v, w) -> np.ndarray:
    """comp_with(t, u, v, w, &half_gemm) (mixed.cpp:84-86)."""
    t, u, v, w = _f64(t), _f64(u), _f64(v), _f64(w)
    y = _comp_shapes(t, u, v, w)
    check(lib.xtsg_comp_half(ptr(t), *t.shape, ptr(u), u.shape[0], ptr(v), v.shape[0], ptr(w),
                             w.shape[0], ptr(y)))
    return y


def comp_mixed(t, u, v, w) -> np.ndarray:
    """comp_mixed (mixed.cpp:88-98). Each argument is a (half, residual) pair
    as returned by split_half."""
    (th, tr), (uh, ur), (vh, vr), (wh, wr) = [(_f64(a), _f64(b)) for a, b in (t, u, v, w)]
    y = _comp_shapes(th, uh, vh, wh)
    check(lib.xtsg_comp_mixed(ptr(th), ptr(tr), *th.shape, ptr(uh), ptr(ur), uh.shape[0], ptr(vh), ptr(vr),
                              vh.shape[0], ptr(wh), ptr(wr), wh.shape[0], ptr(y)))
    return y


def comp_naive_half(t, u, v, w) -> np.ndarray:
    """comp_naive_half (mixed.cpp:100-104)."""
    t, u, v, w = _f64(t), _f64(u), _f64(v), _f64(w)
    y = _comp_shapes(t, u, v, w)
    check(lib.xtsg_comp_naive_half(ptr(t), *t.shape, ptr(u), u.shape[0], ptr(v), v.shape[0], ptr(w),
                                   w.shape[0], ptr(y)))
    return y


def reconstruct(a, b, c) -> np.ndarray:
    """tensor.cpp:133-150"""
    a, b, c = _f64(a), _f64(b), _f64(c)
    out = np.zeros((a.shape[0], b.shape[0], c.shape[0]), order="F")
    check(lib.xtsg_reconstruct(ptr(a), ptr(b), ptr(c), a.shape[0], b.shape[0], c.shape[0],
                               a.shape[1], ptr(out)))
    return out


def comp_from_factors(factors, u, v, w) -> np.ndarray:
    """compression.cpp:215-220"""
    a, b, c = (_f64(x) for x in factors)
    u, v, w = _f64(u), _f64(v), _f64(w)
    if u.shape[1] != a.shape[0] or v.shape[1] != b.shape[0] or w.shape[1] != c.shape[0]:
        from ._lib import UsageError
        raise UsageError("comp_from_factors: compression matrix columns must match factors")
    y = np.zeros((u.shape[0], v.shape[0], w.shape[0]), order="F")
    check(lib.xtsg_comp_from_factors(ptr(a), ptr(b), ptr(c), a.shape[0], b.shape[0], c.shape[0],
                                     a.shape[1], ptr(u), u.shape[0], ptr(v), v.shape[0], ptr(w),
                                     w.shape[0], ptr(y)))
    return y


def comp_blocked(dims, block, source: Iterable, ensemble: Ensemble, deterministic: bool = True,
                 regions: Iterable = ()):
    """compression.cpp:332-404. ``source`` yields (cell, block_tensor) records;
    ``regions`` are (element offset, tensor) pieces of whole cells pushed first
    (xtsg_blocked_push_region, deterministic mode)."""
    dims, block = _arr3(dims), _arr3(block)
    P = ensemble.count
    red = _arr3([ensemble.u[0].shape[0], ensemble.v[0].shape[0], ensemble.w[0].shape[0]])
    src_dims = [ensemble.u[0].shape[1], ensemble.v[0].shape[1], ensemble.w[0].shape[1]]
    if list(src_dims) != [int(d) for d in dims]:
        from ._lib import UsageError
        raise UsageError("comp_blocked: ensemble does not match grid dims")
    u = np.concatenate([x.ravel(order="F") for x in ensemble.u])
    v = np.concatenate([x.ravel(order="F") for x in ensemble.v])
    w = np.concatenate([x.ravel(order="F") for x in ensemble.w])
    h = C.c_void_p()
    check(lib.xtsg_blocked_begin(ptr(dims), ptr(block), P, ptr(red), ptr(u), ptr(v), ptr(w),
                                 1 if deterministic else 0, C.byref(h)))
    try:
        for off, data in regions:
            data = _f64(data)
            check(lib.xtsg_blocked_push_region(h, ptr(_arr3(off)), ptr(_arr3(data.shape)), ptr(data)))
        for cell, data in source:
            data = _f64(data)
            check(lib.xtsg_blocked_push(h, ptr(_arr3(cell)), ptr(_arr3(data.shape)), ptr(data)))
        out = np.zeros(P * int(np.prod(red)))
        check(lib.xtsg_blocked_finish(h, ptr(out)))
    finally:
        lib.xtsg_blocked_destroy(h)
    n = int(np.prod(red))
    return [out[p * n:(p + 1) * n].reshape(tuple(red), order="F") for p in range(P)]


def _torch_dtype_code(t):
    import torch
    return {torch.bfloat16: DTYPE_BF16, torch.float32: DTYPE_F32, torch.float64: DTYPE_F64,
            torch.float16: DTYPE_F16}[t.dtype]


_CUDA_STREAM_LEGACY = 0x1   # cudaStreamLegacy: the explicit handle of the legacy default stream


def _stream_arg(stream, *arrays):
    """The CUDA stream a plan call runs on. An explicit ``stream`` (torch
    stream or raw handle) wins; otherwise, when any argument is a torch CUDA
    tensor, the call joins torch's current stream (the legacy default stream
    by its explicit handle, since 0 means "the library's own per-thread
    stream" in the C ABI) so the results are ordered with later torch work;
    host-only calls run on the library's stream and return synchronised."""
    if stream is not None:
        h = getattr(stream, "cuda_stream", stream)
        return C.c_void_p(h if h else _CUDA_STREAM_LEGACY)
    for a in arrays:
        if getattr(a, "is_cuda", False):
            import torch
            h = torch.cuda.current_stream(a.device).cuda_stream
            return C.c_void_p(h if h else _CUDA_STREAM_LEGACY)
    return None


class Plan:
    """Device-resident compression plan (include/xtsg.h, xtsg_plan_*)."""

    def __init__(self, dims, reduced, count: int, shared_rows: int, seed: int,
                 precision: int = PREC_BF16, kind="gaussian", **spec):
        d = PlanDesc()
        for m in range(3):
            d.dims[m] = int(dims[m])
            d.reduced[m] = int(reduced[m])
        d.count = int(count)
        d.shared_rows = int(shared_rows)
        d.spec = _spec(kind, **spec)
        d.seed = C.c_uint64(seed).value
        d.precision = int(precision)
        self.desc = d
        self.dims = tuple(int(x) for x in dims)
        self.reduced = tuple(int(x) for x in reduced)
        self.count = int(count)
        self.precision = int(precision)
        self._h = C.c_void_p()
        check(lib.xtsg_plan_create(C.byref(d), C.byref(self._h)))

    def close(self):
        if self._h:
            lib.xtsg_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def out_shape(self):
        return (self.count,) + self.reduced

    def compress(self, x, y=None, offset=(0, 0, 0), extent=None, ld=None, accumulate=False,
                 stream=None):
        """Compress block ``x`` (column-major (i,j,k) block, numpy or torch) at ``offset``.

        Returns y: (P, L, M, N) with each replica column-major, i.e. an array whose
        ``y[p]`` memory image is the reference Tensor3 of replica p.
        """
        if isinstance(x, np.ndarray):
            if x.dtype not in (np.float32, np.float64):
                raise TypeError("numpy input must be float32/float64")
            xa = np.asfortranarray(x)
            code = DTYPE_F64 if xa.dtype == np.float64 else DTYPE_F32
            shape = xa.shape
            strides = [s // xa.itemsize for s in xa.strides]
        else:
            xa = x
            code = _torch_dtype_code(x)
            shape = tuple(x.shape)
            strides = list(x.stride())
        if extent is None:
            extent = shape
        if ld is None:
            if strides[0] != 1:
                raise ValueError("x must be column-major (i fastest)")
            ld = (strides[1], strides[2])
        ydt = np.float64 if self.precision == PREC_FP64 else np.float32
        if y is None:
            if isinstance(x, np.ndarray):
                y = np.zeros(self.count * int(np.prod(self.reduced)), ydt)
            else:
                import torch
                y = torch.zeros(self.count * int(np.prod(self.reduced)),
                                dtype=torch.float64 if ydt == np.float64 else torch.float32,
                                device=x.device)
        st = _stream_arg(stream, x, y)
        check(lib.xtsg_plan_compress(self._h, ptr(xa), code, ptr(np.asarray(ld, np.int64)),
                                     ptr(_arr3(offset)), ptr(_arr3(extent)), ptr(y),
                                     1 if accumulate else 0, st))
        return y

    def _y(self, like_device, y):
        if y is not None:
            return y
        n = self.count * int(np.prod(self.reduced))
        if like_device is None:
            return np.zeros(n, np.float32)
        import torch
        return torch.zeros(n, dtype=torch.float32, device=like_device)

    def compress_factors(self, factors, k0=0, k1=None, y=None, accumulate=False, stream=None, device=None):
        """xtsg_plan_compress_factors: X = reconstruct(a, b, c) generated on the device slab by slab."""
        a, b, c = (_f64(x) for x in factors)
        k1 = self.dims[2] if k1 is None else k1
        y = self._y(device, y)
        st = _stream_arg(stream, y)
        check(lib.xtsg_plan_compress_factors(self._h, ptr(a), ptr(b), ptr(c), a.shape[1], int(k0), int(k1), ptr(y),
                                             1 if accumulate else 0, st))
        return y

    def compress_coo(self, i, j, k, val, y=None, accumulate=False, stream=None, device=None):
        """xtsg_plan_compress_coo: COO nonzeros (int32 coordinates, fp32 values; duplicates sum)."""
        def as_arr(v, dt):
            if isinstance(v, np.ndarray) or not hasattr(v, "data_ptr"):
                return np.ascontiguousarray(np.asarray(v, dt))
            return v
        i, j, k = as_arr(i, np.int32), as_arr(j, np.int32), as_arr(k, np.int32)
        val = as_arr(val, np.float32)
        nnz = int(val.shape[0])
        y = self._y(device, y)
        st = _stream_arg(stream, y, i, val)
        check(lib.xtsg_plan_compress_coo(self._h, ptr(i), ptr(j), ptr(k), ptr(val), nnz, ptr(y),
                                         1 if accumulate else 0, st))
        return y

    def compress_csf(self, slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val, y=None, accumulate=False,
                     stream=None, device=None):
        """xtsg_plan_compress_csf: CSF input (slices k -> fibers j -> nonzeros i), no sort pass."""
        def as_arr(v, dt):
            if isinstance(v, np.ndarray) or not hasattr(v, "data_ptr"):
                return np.ascontiguousarray(np.asarray(v, dt))
            return v
        slice_k, fiber_j, nz_i = (as_arr(v, np.int32) for v in (slice_k, fiber_j, nz_i))
        slice_ptr, fiber_ptr = (as_arr(v, np.int64) for v in (slice_ptr, fiber_ptr))
        val = as_arr(val, np.float32)
        _csf_shape_check(slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val)
        y = self._y(device, y)
        st = _stream_arg(stream, y, nz_i, val)
        check(lib.xtsg_plan_compress_csf(self._h, int(slice_k.shape[0]), ptr(slice_k), ptr(slice_ptr),
                                         int(fiber_j.shape[0]), ptr(fiber_j), ptr(fiber_ptr), int(val.shape[0]),
                                         ptr(nz_i), ptr(val), ptr(y), 1 if accumulate else 0, st))
        return y

    @staticmethod
    def coo_to_csf(i, j, k, val):
        """Host helper: COO -> CSF (stable sort by (k, j), slices and fibers of equal keys)."""
        i, j, k = (np.asarray(a, np.int64) for a in (i, j, k))
        order = np.lexsort((j, k))
        i, j, k, v = i[order], j[order], k[order], np.asarray(val, np.float32)[order]
        new_f = np.ones(len(k), bool)
        new_f[1:] = (k[1:] != k[:-1]) | (j[1:] != j[:-1])
        fstart = np.nonzero(new_f)[0]
        fiber_ptr = np.append(fstart, len(k)).astype(np.int64)
        fk = k[fstart]
        new_s = np.ones(len(fstart), bool)
        new_s[1:] = fk[1:] != fk[:-1]
        sstart = np.nonzero(new_s)[0]
        slice_ptr = np.append(sstart, len(fstart)).astype(np.int64)
        return (fk[sstart].astype(np.int32), slice_ptr, j[fstart].astype(np.int32), fiber_ptr, i.astype(np.int32),
                v)

    def compress_file(self, path, y=None, accumulate=False, stream=None, device=None, slab_bytes=0):
        """xtsg_plan_compress_file: compress a .xts file (dense or factor triple) straight from disk."""
        ydt = np.float64 if self.precision == PREC_FP64 else np.float32
        if y is None:
            n = self.count * int(np.prod(self.reduced))
            if device is None:
                y = np.zeros(n, ydt)
            else:
                import torch
                y = torch.zeros(n, dtype=torch.float64 if ydt == np.float64 else torch.float32, device=device)
        st = _stream_arg(stream, y)
        check(lib.xtsg_plan_compress_file(self._h, str(path).encode(), int(slab_bytes), ptr(y),
                                          1 if accumulate else 0, st))
        return y

    def set_profiling(self, on: bool = True):
        check(lib.xtsg_plan_set_profiling(self._h, 1 if on else 0))

    def profile(self, reset: bool = True) -> dict:
        out = np.zeros(6)
        check(lib.xtsg_plan_profile(self._h, 1 if reset else 0, ptr(out)))
        return {"fused_ms": out[0], "fused_launches": int(out[1]), "mode3_ms": out[2],
                "mode3_launches": int(out[3]), "fused_flops": out[4], "mode3_flops": out[5]}

    @staticmethod
    def replicas(y, count, reduced):
        """Split a flat output into per-replica column-major tensors (numpy)."""
        n = int(np.prod(reduced))
        y = np.asarray(y)
        return [y[p * n:(p + 1) * n].reshape(tuple(reduced), order="F") for p in range(count)]


def _csf_shape_check(slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val):
    """The C ABI reads slice_ptr[n_slices] and fiber_ptr[n_fibers]: the pointer
    arrays must be one longer than their index arrays."""
    if (slice_ptr.shape[0] != slice_k.shape[0] + 1 or fiber_ptr.shape[0] != fiber_j.shape[0] + 1
            or nz_i.shape[0] != val.shape[0]):
        raise UsageError("compress_csf: need len(slice_ptr) = len(slice_k) + 1, "
                         "len(fiber_ptr) = len(fiber_j) + 1 and len(nz_i) = len(val)")


class MultiPlan:
    """xtsg_multi_*: one plan per GPU of the node, mode-3 slabs per GPU and one
    NCCL reduce of the replicas onto the first GPU (SURVEY §8 e), driven from
    one process through the C ABI (no torch.distributed)."""

    def __init__(self, dims, reduced, count: int, shared_rows: int, seed: int, gpus=(0,),
                 precision: int = PREC_BF16, kind="gaussian", **spec):
        d = PlanDesc()
        for m in range(3):
            d.dims[m] = int(dims[m])
            d.reduced[m] = int(reduced[m])
        d.count, d.shared_rows = int(count), int(shared_rows)
        d.spec = _spec(kind, **spec)
        d.seed = C.c_uint64(seed).value
        d.precision = int(precision)
        self.desc, self.count, self.reduced = d, int(count), tuple(int(x) for x in reduced)
        self.gpus = np.asarray(gpus, np.int32)
        # load torch (and with it torch's NCCL) first: the library dlopens
        # whatever libnccl.so.2 the process already has, and a different
        # system NCCL loaded first would break a later `import torch`
        import torch  # noqa: F401
        self._h = C.c_void_p()
        check(lib.xtsg_multi_create(C.byref(d), len(self.gpus), ptr(self.gpus), C.byref(self._h)))

    def close(self):
        if self._h:
            lib.xtsg_multi_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _y(self, y):
        return np.zeros(self.count * int(np.prod(self.reduced)), np.float32) if y is None else y

    def compress_factors(self, factors, y=None, accumulate=False):
        a, b, c = (_f64(x) for x in factors)
        y = self._y(y)
        check(lib.xtsg_multi_compress_factors(self._h, ptr(a), ptr(b), ptr(c), a.shape[1], ptr(y),
                                              1 if accumulate else 0))
        return y

    def compress(self, x, y=None, accumulate=False):
        xa = np.asfortranarray(x)
        code = {np.dtype(np.float64): DTYPE_F64, np.dtype(np.float32): DTYPE_F32}[xa.dtype]
        ld = np.asarray([xa.shape[0], xa.shape[0] * xa.shape[1]], np.int64)
        y = self._y(y)
        check(lib.xtsg_multi_compress(self._h, ptr(xa), code, ptr(ld), ptr(y), 1 if accumulate else 0))
        return y

    def compress_coo(self, i, j, k, val, y=None, accumulate=False):
        """xtsg_multi_compress_coo: host COO nonzeros, contiguous nonzero ranges per GPU."""
        i, j, k = (np.ascontiguousarray(np.asarray(a, np.int32)) for a in (i, j, k))
        val = np.ascontiguousarray(np.asarray(val, np.float32))
        y = self._y(y)
        check(lib.xtsg_multi_compress_coo(self._h, ptr(i), ptr(j), ptr(k), ptr(val), int(val.shape[0]), ptr(y),
                                          1 if accumulate else 0))
        return y

    def compress_csf(self, slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val, y=None, accumulate=False):
        """xtsg_multi_compress_csf: host CSF, nonzero-balanced slice ranges per GPU."""
        slice_k, fiber_j, nz_i = (np.ascontiguousarray(np.asarray(a, np.int32)) for a in (slice_k, fiber_j, nz_i))
        slice_ptr, fiber_ptr = (np.ascontiguousarray(np.asarray(a, np.int64)) for a in (slice_ptr, fiber_ptr))
        val = np.ascontiguousarray(np.asarray(val, np.float32))
        _csf_shape_check(slice_k, slice_ptr, fiber_j, fiber_ptr, nz_i, val)
        y = self._y(y)
        check(lib.xtsg_multi_compress_csf(self._h, int(slice_k.shape[0]), ptr(slice_k), ptr(slice_ptr),
                                          int(fiber_j.shape[0]), ptr(fiber_j), ptr(fiber_ptr), int(val.shape[0]),
                                          ptr(nz_i), ptr(val), ptr(y), 1 if accumulate else 0))
        return y

    def last_ms(self) -> float:
        out = np.zeros(1)
        check(lib.xtsg_multi_last_ms(self._h, ptr(out)))
        return float(out[0])


def nccl_version() -> int:
    import torch  # noqa: F401  (see MultiPlan)
    v = np.zeros(1, np.int32)
    check(lib.xtsg_nccl_version(ptr(v)))
    return int(v[0])


# ---------------------------------------------------------------------------
# CP-ALS (cp_als.hpp:10-40)

@dataclass
class AlsResult:
    factors: tuple
    iters: int
    error_history: list
    converged: bool

    def final_error(self) -> float:
        return self.error_history[-1] if self.error_history else 1.0


def cp_als_batched(tensors: Sequence, rank: int, max_iters: int = 500, tol: float = 1e-10,
                   seeds: Sequence[int] | int = 0, init: Sequence[int] | int = 0):
    """cp_als over a batch of same-shape tensors; ``seeds``/``init`` are one
    value for every tensor or one per tensor."""
    ts = [_f64(t) for t in tensors]
    n = len(ts)
    if n == 0:
        return []
    n1, n2, n3 = ts[0].shape
    if any(t.shape != ts[0].shape for t in ts):
        from ._lib import UsageError
        raise UsageError("cp_als_batched: every tensor must have the same shape")
    seeds = [int(seeds)] * n if isinstance(seeds, (int, np.integer)) else list(seeds)
    inits = [int(init)] * n if isinstance(init, (int, np.integer)) else list(init)
    if len(seeds) != n or len(inits) != n:
        from ._lib import UsageError
        raise UsageError("cp_als_batched: seeds/init must be a scalar or one per tensor")
    cfgs = (AlsConfig * n)()
    for q in range(n):
        cfgs[q] = AlsConfig(int(rank), int(max_iters), float(tol), C.c_uint64(seeds[q]).value,
                            int(inits[q]), 0)
    flat = np.concatenate([t.ravel(order="F") for t in ts]) if n else np.zeros(0)
    a = np.zeros(n * n1 * rank); b = np.zeros(n * n2 * rank); c = np.zeros(n * n3 * rank)
    iters = np.zeros(n, np.int64); conv = np.zeros(n, np.int32); hist = np.zeros(n * max_iters)
    check(lib.xtsg_cp_als_batched(n, ptr(flat), n1, n2, n3, cfgs, ptr(a), ptr(b), ptr(c),
                                  ptr(iters), ptr(conv), ptr(hist)))
    out = []
    for q in range(n):
        fa = a[q * n1 * rank:(q + 1) * n1 * rank].reshape(n1, rank, order="F")
        fb = b[q * n2 * rank:(q + 1) * n2 * rank].reshape(n2, rank, order="F")
        fc = c[q * n3 * rank:(q + 1) * n3 * rank].reshape(n3, rank, order="F")
        it = int(iters[q])
        out.append(AlsResult((fa, fb, fc), it, list(hist[q * max_iters:q * max_iters + it]), bool(conv[q])))
    return out


def cp_als(t, rank: int, max_iters: int = 500, tol: float = 1e-10, seed: int = 0, init: int = 0):
    """cp_als.cpp:46-111"""
    return cp_als_batched([t], rank, max_iters, tol, [seed], [init])[0]


def relative_error(t, factors) -> float:
    """cp_als.cpp:37-44"""
    t = _f64(t)
    a, b, c = (_f64(x) for x in factors)
    out = np.zeros(1)
    check(lib.xtsg_relative_error(ptr(t), *t.shape, ptr(a), ptr(b), ptr(c), a.shape[1], ptr(out)))
    return float(out[0])


# ---------------------------------------------------------------------------
# alignment & recovery (alignment.hpp)

def normalize_shared(m, shared_rows: int):
    m = _f64(m)
    out = np.zeros_like(m, order="F")
    piv = np.zeros(m.shape[1])
    check(lib.xtsg_normalize_shared(ptr(m), m.shape[0], m.shape[1], int(shared_rows), ptr(out), ptr(piv)))
    return out, piv


def max_trace_assignment(objective) -> list:
    o = _f64(objective)
    if o.ndim != 2 or o.shape[0] != o.shape[1]:
        from ._lib import UsageError
        raise UsageError("max_trace_assignment: objective must be square")
    perm = np.zeros(o.shape[0], np.int64)
    check(lib.xtsg_max_trace_assignment(ptr(o), o.shape[0], ptr(perm)))
    return [int(x) for x in perm]


def align_replicas(factors: Sequence, shared_rows: int, min_survivors: int = 1):
    """alignment.cpp:154-218 -> (aligned, dropped, survivors)"""
    P = len(factors)
    if P == 0:
        from ._lib import UsageError
        raise UsageError("align_replicas: no replicas")
    dims = _arr3([f[0].shape[0] for f in [factors[0]]] + [factors[0][1].shape[0], factors[0][2].shape[0]])
    r = factors[0][0].shape[1]
    flat = np.concatenate([np.concatenate([_f64(x).ravel(order="F") for x in f]) for f in factors])
    per = int(dims.sum()) * r
    aligned = np.zeros(P * per)
    dropped = np.zeros(P, np.int32)
    surv = np.zeros(P, np.int64)
    ns = np.zeros(1, np.int64)
    check(lib.xtsg_align_replicas(P, ptr(dims), r, ptr(flat), int(shared_rows), int(min_survivors),
                                  ptr(aligned), ptr(dropped), ptr(surv), ptr(ns)))
    out = []
    for i in range(int(ns[0])):
        base = aligned[i * per:(i + 1) * per]
        o0 = dims[0] * r
        o1 = o0 + dims[1] * r
        out.append((base[:o0].reshape(dims[0], r, order="F"), base[o0:o1].reshape(dims[1], r, order="F"),
                    base[o1:].reshape(dims[2], r, order="F")))
    return out, [bool(x) for x in dropped], [int(x) for x in surv[:int(ns[0])]]


def solve_stacked_ls(stacked_factors: Sequence, stacked_compressors: Sequence) -> np.ndarray:
    """alignment.cpp:220-252"""
    if len(stacked_factors) == 0 or len(stacked_factors) != len(stacked_compressors):
        from ._lib import UsageError
        raise UsageError("solve_stacked_ls: factor/compressor counts differ")
    fs = [_f64(f) for f in stacked_factors]
    us = [_f64(u) for u in stacked_compressors]
    r = fs[0].shape[1]
    cols = us[0].shape[1]
    rows = np.array([f.shape[0] for f in fs], np.int64)
    for f, u in zip(fs, us):
        if f.shape[1] != r or u.shape[1] != cols or f.shape[0] != u.shape[0]:
            from ._lib import UsageError
            raise UsageError("solve_stacked_ls: inconsistent block shapes")
    f = np.concatenate([x.ravel(order="F") for x in fs])
    u = np.concatenate([x.ravel(order="F") for x in us])
    x = np.zeros((cols, r), order="F")
    check(lib.xtsg_solve_stacked_ls(len(fs), ptr(rows), r, cols, ptr(f), ptr(u), ptr(x)))
    return x


def recover_perm_scale(global_head, sampled):
    g, s = _f64(global_head), _f64(sampled)
    if g.shape != s.shape:
        from ._lib import UsageError
        raise UsageError("recover_perm_scale: blocks must share shape")
    perm = np.zeros(g.shape[1], np.int64)
    scale = np.zeros(g.shape[1])
    check(lib.xtsg_recover_perm_scale(ptr(g), ptr(s), g.shape[0], g.shape[1], ptr(perm), ptr(scale)))
    return [int(x) for x in perm], [float(x) for x in scale]


def apply_forward(m, perm, scale) -> np.ndarray:
    """alignment.cpp:280-291: column r = m[:, perm[r]] * scale[r]"""
    m = _f64(m)
    return np.asfortranarray(m[:, list(perm)] * np.asarray(scale)[None, :])


def apply_recovery(m, perm, scale) -> np.ndarray:
    """alignment.cpp:293-304"""
    m = _f64(m)
    out = np.zeros_like(m, order="F")
    out[:, list(perm)] = m / np.asarray(scale)[None, :]
    return out


# ---------------------------------------------------------------------------
# synthetic problems and the end-to-end pipeline (pipeline.hpp)

def xts_header(path):
    """Header of a .xts file (io.cpp:94-125): (kind 'tensor'|'factors', dims, rank)."""
    kind = C.c_int32()
    dims = np.zeros(3, np.int64)
    rank = C.c_int64()
    check(lib.xtsg_xts_header(str(path).encode(), C.byref(kind), ptr(dims), C.byref(rank)))
    return ("tensor" if kind.value == 0 else "factors"), tuple(int(d) for d in dims), int(rank.value)


def generate_factors(dims, rank: int, law: str = "dense", nnz_per_col: int = 0, seed: int = 0):
    """generate (pipeline.cpp:176-207) without materialization: the factor triple."""
    d = _arr3(dims)
    outs = [np.zeros((int(d[m]), int(rank)), order="F") for m in range(3)]
    code = {"dense": LAW_DENSE, "sparse": LAW_SPARSE}[law] if isinstance(law, str) else int(law)
    check(lib.xtsg_generate_factors(ptr(d), int(rank), code, int(nnz_per_col), C.c_uint64(seed),
                                    *[ptr(o) for o in outs]))
    return tuple(outs)


_MODES = {"dense": MODE_DENSE, "sparse": MODE_SPARSE, "two_stage": MODE_TWO_STAGE}


@dataclass
class PipelineConfig:
    """PipelineConfig (pipeline.hpp:16-45) for the device pipeline, same defaults,
    plus ``precision`` (PREC_FP64 = the reference's full precision, PREC_BF16 =
    tcgen05 compression; then ``replica_fit_tol`` must admit the bf16 error)."""
    reduced: tuple = (0, 0, 0)
    rank: int = 1
    replicas: int = 0
    slack: int = 10
    shared: int = 0
    mode: str = "dense"
    precision: int = PREC_FP64
    alpha: float = 1.6
    beta: float = 1.6
    gamma: float = 1.6
    projection_s: float = 0.0
    omp_sparsity: int = 0
    omp_residual_tol: float = 1e-9
    sample_b: int = 0
    seed: int = 0
    als_max_iters: int = 500
    als_tol: float = 1e-10
    replica_fit_tol: float = 1e-6
    als_restarts: int = 3

    def to_c(self) -> PipelineConfigC:
        c = PipelineConfigC()
        for m in range(3):
            c.reduced[m] = int(self.reduced[m])
        c.rank, c.replicas, c.slack, c.shared = int(self.rank), int(self.replicas), int(self.slack), int(self.shared)
        c.mode = _MODES[self.mode] if isinstance(self.mode, str) else int(self.mode)
        c.precision = int(self.precision)
        c.alpha, c.beta, c.gamma = float(self.alpha), float(self.beta), float(self.gamma)
        c.projection_s = float(self.projection_s)
        c.omp_sparsity, c.omp_residual_tol = int(self.omp_sparsity), float(self.omp_residual_tol)
        c.sample_b = int(self.sample_b)
        c.seed = C.c_uint64(self.seed).value
        c.als_max_iters, c.als_tol = int(self.als_max_iters), float(self.als_tol)
        c.replica_fit_tol, c.als_restarts = float(self.replica_fit_tol), int(self.als_restarts)
        return c


@dataclass
class RunMetrics:
    """RunMetrics subset (metrics.hpp): per-stage seconds/status, survivors, sample MSE."""
    stage_seconds: dict
    stage_status: dict
    replicas_total: int
    replicas_dropped: int
    sample_mse: float
    block_fit: float
    als_sweeps: int


_STAGES = ("compression", "decomposition", "alignment", "recovery")
_STATUS = {0: "skipped", 1: "ok", 2: "error"}


def _metrics(m: PipelineMetricsC) -> RunMetrics:
    return RunMetrics({s: m.stage_seconds[i] for i, s in enumerate(_STAGES)},
                      {s: _STATUS.get(m.stage_status[i], "?") for i, s in enumerate(_STAGES)},
                      int(m.replicas_total), int(m.replicas_dropped), float(m.sample_mse),
                      float(m.block_fit), int(m.als_sweeps))


def _source(tensor, factors):
    if tensor is not None:
        t = tensor if not isinstance(tensor, np.ndarray) else _f64(tensor)
        return t, tuple(int(x) for x in t.shape), (None, None, None), 0
    f = tuple(_f64(x) for x in factors)
    return None, (f[0].shape[0], f[1].shape[0], f[2].shape[0]), f, f[0].shape[1]


def decompose(cfg: PipelineConfig, tensor=None, factors=None):
    """decompose (pipeline.cpp:245-573) on the device -> (factors, RunMetrics).

    ``tensor``: column-major fp64 array (numpy or a CUDA tensor); or ``factors``
    (a, b, c) standing in for a tensor too large to hold (TensorSource)."""
    t, dims, f, frank = _source(tensor, factors)
    d = _arr3(dims)
    outs = [np.zeros((int(d[m]), int(cfg.rank)), order="F") for m in range(3)]
    met = PipelineMetricsC()
    c = cfg.to_c()
    rc = lib.xtsg_decompose(C.byref(c), ptr(d), ptr(t), *[ptr(x) for x in f], int(frank),
                            *[ptr(o) for o in outs], C.byref(met))
    check(rc)
    return tuple(outs), _metrics(met)


def decompose_replicas(cfg: PipelineConfig, replicas, tensor=None, factors=None):
    """Stages 1-3 of decompose on caller-compressed replicas (flat P*L*M*N, f32/f64,
    numpy or CUDA tensor), e.g. after a mode-3-sharded multi-GPU compression."""
    t, dims, f, frank = _source(tensor, factors)
    d = _arr3(dims)
    if isinstance(replicas, np.ndarray):
        y = np.ascontiguousarray(replicas)
        code = DTYPE_F64 if y.dtype == np.float64 else DTYPE_F32
        if y.dtype not in (np.float32, np.float64):
            raise TypeError("replicas must be float32/float64")
    else:
        y = replicas.contiguous()
        code = _torch_dtype_code(y)
    outs = [np.zeros((int(d[m]), int(cfg.rank)), order="F") for m in range(3)]
    met = PipelineMetricsC()
    c = cfg.to_c()
    check(lib.xtsg_decompose_replicas(C.byref(c), ptr(d), ptr(y), code, ptr(t), *[ptr(x) for x in f],
                                      int(frank), *[ptr(o) for o in outs], C.byref(met)))
    return tuple(outs), _metrics(met)


def _replicas_arg(replicas):
    if isinstance(replicas, np.ndarray):
        if replicas.dtype not in (np.float32, np.float64):
            raise TypeError("replicas must be float32/float64")
        y = np.ascontiguousarray(replicas)
        return y, (DTYPE_F64 if y.dtype == np.float64 else DTYPE_F32)
    y = replicas.contiguous()
    return y, _torch_dtype_code(y)


@dataclass
class Stage1Result:
    """Per-replica stage-1 results (xtsg_decompose_stage1): factors (n, (L+M+N)*R),
    fit errors, convergence flags, sweeps — the exchange unit of a multi-GPU pipeline."""
    ids: np.ndarray
    factors: np.ndarray
    fit_err: np.ndarray
    converged: np.ndarray
    sweeps: np.ndarray


def decompose_stage1(cfg: PipelineConfig, dims, replicas, ids) -> Stage1Result:
    """Stage 1 of decompose (pipeline.cpp:410-446) for the replicas with global indices ``ids``
    (``replicas``: len(ids) replicas back to back)."""
    d = _arr3(dims)
    ids = np.ascontiguousarray(np.asarray(ids, np.int64))
    n = int(ids.size)
    per_f = int(sum(cfg.reduced)) * int(cfg.rank)
    out = Stage1Result(ids, np.zeros((n, per_f)), np.ones(n), np.zeros(n, np.int32), np.zeros(n, np.int64))
    y, code = _replicas_arg(replicas)
    c = cfg.to_c()
    check(lib.xtsg_decompose_stage1(C.byref(c), ptr(d), n, ptr(ids), ptr(y), code, ptr(out.factors),
                                    ptr(out.fit_err), ptr(out.converged), ptr(out.sweeps)))
    return out


def decompose_finish(cfg: PipelineConfig, stage1: Stage1Result, tensor=None, factors=None):
    """Stages 1 (survivor rule) - 3 from the stage-1 results of all replicas (any order of ids)."""
    t, dims, f, frank = _source(tensor, factors)
    d = _arr3(dims)
    order = np.argsort(stage1.ids, kind="stable")
    fac = np.ascontiguousarray(stage1.factors[order])
    err = np.ascontiguousarray(stage1.fit_err[order])
    conv = np.ascontiguousarray(stage1.converged[order].astype(np.int32))
    sw = np.ascontiguousarray(stage1.sweeps[order].astype(np.int64))
    outs = [np.zeros((int(d[m]), int(cfg.rank)), order="F") for m in range(3)]
    met = PipelineMetricsC()
    c = cfg.to_c()
    check(lib.xtsg_decompose_finish(C.byref(c), ptr(d), ptr(fac), ptr(err), ptr(conv), ptr(sw), ptr(t),
                                    *[ptr(x) for x in f], int(frank), *[ptr(o) for o in outs], C.byref(met)))
    return tuple(outs), _metrics(met)


@dataclass
class EvalReport:
    mode_rel_err: list
    sample_mse: float
    aligned: tuple


def evaluate(truth, recovered, sample: int = 0) -> EvalReport:
    """evaluate (pipeline.cpp:577-609) for a factor-triple truth."""
    t = [_f64(x) for x in truth]
    r = [_f64(x) for x in recovered]
    d = _arr3([x.shape[0] for x in t])
    rank = t[0].shape[1]
    if any(x.shape != y.shape for x, y in zip(t, r)):
        from ._lib import UsageError
        raise UsageError("evaluate: factor dimensions disagree")
    errs = np.zeros(3)
    mse = np.zeros(1)
    al = [np.zeros_like(x, order="F") for x in t]
    check(lib.xtsg_evaluate(ptr(d), rank, *[ptr(x) for x in t], *[ptr(x) for x in r], int(sample),
                            ptr(errs), ptr(mse), *[ptr(x) for x in al]))
    return EvalReport([float(x) for x in errs], float(mse[0]), tuple(al))
