"""xtsg — B200-native Exascale-Tensor compression path (Python mirror of the C ABI).

The product is ``libxtsg.so`` (CUDA sm_100a kernels + the C ABI declared in
``include/xtsg.h``). This module is a thin ctypes binding that mirrors the
reference's C++ entry points (``/root/reference/proj/include/xts``) with the
same names, argument meaning and exception types, so tests and the bench read
like the reference's own. There is no CPU fallback: every compute call goes
through the CUDA library and raises :class:`CudaError` without a B200.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from ._lib import (  # noqa: F401
    CudaError, DataError, DegenerateColumnError, HalfRangeError, IllPosedError,
    InsufficientReplicasError, StageError, UsageError, XtsError, lib, check, ptr,
    KIND_GAUSSIAN, KIND_SPARSE, KIND_TWO_STAGE, PREC_FP64, PREC_BF16, PREC_FP16, PREC_FP16X3,
    DTYPE_BF16, DTYPE_F32, DTYPE_F64, DTYPE_F16, EnsembleSpec, PlanDesc, AlsConfig,
    LAW_DENSE, LAW_SPARSE, MODE_DENSE, MODE_SPARSE, MODE_TWO_STAGE,
)
from .api import (  # noqa: F401
    compute_replica_count, gen_gaussian, gen_sparse_projection, make_ensemble, comp,
    comp_from_factors, reconstruct, round_to_half, split_half, half_gemm, comp_half, comp_mixed,
    comp_naive_half, comp_blocked, Plan, MultiPlan, nccl_version, launch_count, device_ready,
    cp_als, cp_als_batched, relative_error, normalize_shared, max_trace_assignment,
    align_replicas, solve_stacked_ls, recover_perm_scale, apply_forward, apply_recovery,
    generate_factors, xts_header, PipelineConfig, RunMetrics, decompose, decompose_replicas, decompose_stage1,
    decompose_finish, Stage1Result, evaluate, EvalReport,
)

__all__ = [n for n in dir() if not n.startswith("_")]
