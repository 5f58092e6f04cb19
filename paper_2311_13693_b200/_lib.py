"""ctypes binding of libxtsg.so (include/xtsg.h) and the xts exception taxonomy.

Exception classes mirror /root/reference/proj/include/xts/errors.hpp:10-59.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libxtsg.so"

KIND_GAUSSIAN, KIND_SPARSE, KIND_TWO_STAGE = 0, 1, 2
PREC_FP64, PREC_BF16, PREC_FP16, PREC_FP16X3 = 0, 1, 2, 3
DTYPE_BF16, DTYPE_F32, DTYPE_F64, DTYPE_F16 = 0, 1, 2, 3
LAW_DENSE, LAW_SPARSE = 0, 1
MODE_DENSE, MODE_SPARSE, MODE_TWO_STAGE = 0, 1, 2


class XtsError(RuntimeError):
    pass


class UsageError(XtsError, ValueError):
    """xts::UsageError (std::invalid_argument)."""


class DataError(XtsError):
    pass


class IllPosedError(XtsError):
    def __init__(self, msg, effective_rank):
        super().__init__(msg)
        self.effective_rank = effective_rank


class DegenerateColumnError(XtsError):
    def __init__(self, msg, column):
        super().__init__(msg)
        self.column = column


class InsufficientReplicasError(XtsError):
    def __init__(self, msg, survivors, required):
        super().__init__(msg)
        self.survivors = survivors
        self.required = required


class HalfRangeError(XtsError):
    pass


class StageError(XtsError):
    def __init__(self, msg, stage):
        super().__init__(msg)
        self.stage = stage


class CudaError(XtsError):
    """No usable sm_100 device or a CUDA runtime failure (no CPU fallback)."""


class EnsembleSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("inner_kind", C.c_int32), ("s", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("inner_s", C.c_double)]


class PlanDesc(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("reduced", C.c_int64 * 3), ("count", C.c_int64),
                ("shared_rows", C.c_int64), ("spec", EnsembleSpec), ("seed", C.c_uint64),
                ("precision", C.c_int32), ("reserved", C.c_int32)]


class AlsConfig(C.Structure):
    _fields_ = [("rank", C.c_int64), ("max_iters", C.c_int64), ("tol", C.c_double),
                ("seed", C.c_uint64), ("init", C.c_int32), ("reserved", C.c_int32)]


class PipelineConfigC(C.Structure):
    _fields_ = [("reduced", C.c_int64 * 3), ("rank", C.c_int64), ("replicas", C.c_int64),
                ("slack", C.c_int64), ("shared", C.c_int64), ("mode", C.c_int32),
                ("precision", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
                ("gamma", C.c_double), ("projection_s", C.c_double), ("omp_sparsity", C.c_int64),
                ("omp_residual_tol", C.c_double), ("sample_b", C.c_int64), ("seed", C.c_uint64),
                ("als_max_iters", C.c_int64), ("als_tol", C.c_double),
                ("replica_fit_tol", C.c_double), ("als_restarts", C.c_int64)]


class PipelineMetricsC(C.Structure):
    _fields_ = [("stage_seconds", C.c_double * 4), ("stage_status", C.c_int32 * 4),
                ("replicas_total", C.c_int64), ("replicas_dropped", C.c_int64),
                ("sample_mse", C.c_double), ("block_fit", C.c_double), ("als_sweeps", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_U64 = C.c_uint64
_D = C.c_double

_SIGS = {
    "xtsg_last_error": (C.c_char_p, []),
    "xtsg_last_payload": (_I64, [_I32]),
    "xtsg_version": (_I32, []),
    "xtsg_device_ready": (_I32, []),
    "xtsg_warmup": (_I32, []),
    "xtsg_gemm": (_I32, [_I32, _I32, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64]),
    "xtsg_pseudo_inverse": (_I32, [_P, _I64, _I64, _D, _P]),
    "xtsg_leading_left_singular_vectors": (_I32, [_P, _I64, _I64, _I64, _P]),
    "xtsg_solve_least_squares": (_I32, [_P, _I64, _I64, _P, _I64, _P]),
    "xtsg_omp_recover": (_I32, [_P, _I64, _I64, _P, _I64, _I64, _D, _P]),
    "xtsg_launch_count": (_I64, []),
    "xtsg_replica_count": (_I32, [_P, _P, _I64, _P]),
    "xtsg_gen_gaussian": (_I32, [_I64, _I64, _U64, _P]),
    "xtsg_gen_sparse_projection": (_I32, [_I64, _I64, _D, _U64, _P]),
    "xtsg_make_ensemble": (_I32, [_P, _P, _I64, _I64, _P, _U64] + [_P] * 9),
    "xtsg_comp": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "xtsg_comp_from_factors": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64,
                                      _P, _I64, _P]),
    "xtsg_reconstruct": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P]),
    "xtsg_split_half": (_I32, [_P, _I64, _I32, _P, _P]),
    "xtsg_half_gemm": (_I32, [_P, _I64, _I64, _P, _I64, _I64, _P]),
    "xtsg_comp_half": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "xtsg_comp_mixed": (_I32, [_P, _P, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P]),
    "xtsg_comp_naive_half": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "xtsg_blocked_begin": (_I32, [_P, _P, _I64, _P, _P, _P, _P, _I32, _P]),
    "xtsg_blocked_push": (_I32, [_P, _P, _P, _P]),
    "xtsg_blocked_push_region": (_I32, [_P, _P, _P, _P]),
    "xtsg_blocked_finish": (_I32, [_P, _P]),
    "xtsg_blocked_destroy": (None, [_P]),
    "xtsg_plan_create": (_I32, [_P, _P]),
    "xtsg_plan_destroy": (None, [_P]),
    "xtsg_plan_compress": (_I32, [_P, _P, _I32, _P, _P, _P, _P, _I32, _P]),
    "xtsg_plan_set_profiling": (_I32, [_P, _I32]),
    "xtsg_plan_profile": (_I32, [_P, _I32, _P]),
    "xtsg_plan_compress_factors": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _I32, _P]),
    "xtsg_multi_create": (_I32, [_P, _I32, _P, _P]),
    "xtsg_multi_destroy": (None, [_P]),
    "xtsg_multi_compress_factors": (_I32, [_P, _P, _P, _P, _I64, _P, _I32]),
    "xtsg_multi_compress": (_I32, [_P, _P, _I32, _P, _P, _I32]),
    "xtsg_multi_compress_coo": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _I32]),
    "xtsg_multi_compress_csf": (_I32, [_P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, _P, _I32]),
    "xtsg_multi_last_ms": (_I32, [_P, _P]),
    "xtsg_nccl_version": (_I32, [_P]),
    "xtsg_plan_compress_coo": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _I32, _P]),
    "xtsg_xts_header": (_I32, [C.c_char_p, _P, _P, _P]),
    "xtsg_plan_compress_csf": (_I32, [_P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, _P, _I32, _P]),
    "xtsg_plan_compress_file": (_I32, [_P, C.c_char_p, _I64, _P, _I32, _P]),
    "xtsg_relative_error": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _I64, _P]),
    "xtsg_cp_als_batched": (_I32, [_I64, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "xtsg_normalize_shared": (_I32, [_P, _I64, _I64, _I64, _P, _P]),
    "xtsg_max_trace_assignment": (_I32, [_P, _I64, _P]),
    "xtsg_align_replicas": (_I32, [_I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P]),
    "xtsg_solve_stacked_ls": (_I32, [_I64, _P, _I64, _I64, _P, _P, _P]),
    "xtsg_recover_perm_scale": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "xtsg_generate_factors": (_I32, [_P, _I64, _I32, _I64, _U64, _P, _P, _P]),
    "xtsg_decompose": (_I32, [_P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "xtsg_decompose_replicas": (_I32, [_P, _P, _P, _I32, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "xtsg_decompose_stage1": (_I32, [_P, _P, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "xtsg_decompose_finish": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "xtsg_evaluate": (_I32, [_P, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P]),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.xtsg_last_error().decode(errors="replace")
    p0, p1 = lib.xtsg_last_payload(0), lib.xtsg_last_payload(1)
    if rc == 1:
        raise UsageError(msg)
    if rc == 2:
        raise DataError(msg)
    if rc == 3:
        raise IllPosedError(msg, p0)
    if rc == 4:
        raise DegenerateColumnError(msg, p0)
    if rc == 5:
        raise InsufficientReplicasError(msg, p0, p1)
    if rc == 6:
        raise HalfRangeError(msg)
    if rc == 7:
        raise StageError(msg, p0)
    if rc == 8:
        raise CudaError(msg)
    raise XtsError(f"xtsg internal error {rc}: {msg}")


def ptr(a):
    """Raw pointer of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())  # torch.Tensor
