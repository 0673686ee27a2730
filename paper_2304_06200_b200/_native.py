"""ctypes binding of the C ABI declared in include/leangrape_b200.h.

This is the only bridge between the Python mirror of the reference API and
the sm_100a library.  There is no CPU fallback: if the library cannot be
loaded, or no CUDA device is present when a problem is created, the call
raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib_debug" if os.environ.get("LG_DEBUG") else "_lib", "libleangrape_b200.so")

LG_OK = 0
LG_INVALID_ARG = 1
LG_PLANNING_INFEASIBLE = 2
LG_CUDA_ERROR = 3
LG_NCCL_ERROR = 4
LG_INDEX_ERROR = 5
LG_UNSUPPORTED = 6

EXPORTED = (
    "lg_problem_create", "lg_problem_destroy", "lg_eval", "lg_cost", "lg_cost_batch", "lg_eval_device", "lg_plan_table",
    "lg_forward_states", "lg_step_derivative", "lg_matvec", "lg_raw_size", "lg_raw_get", "lg_finalize_host", "lg_make_plan",
    "lg_make_plans_device", "lg_finalize_raw", "lg_np_cabs_host", "lg_np_pairwise_host", "lg_np_reduce_host",
    "lg_set_stream", "lg_set_timing", "lg_get_timing", "lg_bench_zgemm", "lg_device_count", "lg_last_error", "lg_version",
)


class lg_matrix(C.Structure):
    _fields_ = [
        ("dense", C.c_int32),
        ("n", C.c_int64),
        ("nnz", C.c_int64),
        ("row_offsets", C.POINTER(C.c_int64)),
        ("col_indices", C.POINTER(C.c_int64)),
        ("values", C.POINTER(C.c_double)),
    ]


class lg_cost_term(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("weight", C.c_double),
        ("targets", C.POINTER(C.c_double)),
        ("penalty", lg_matrix),
    ]


class lg_problem_desc(C.Structure):
    _fields_ = [
        ("h_static", lg_matrix),
        ("n_channels", C.c_int32),
        ("h_controls", C.POINTER(lg_matrix)),
        ("tau", C.c_double),
        ("n_states", C.c_int64),
        ("initial_states", C.POINTER(C.c_double)),
        ("n_basis", C.c_int64),
        ("basis", C.POINTER(C.c_double)),
        ("n_terms", C.c_int32),
        ("terms", C.POINTER(lg_cost_term)),
        ("device", C.c_int32),
        ("shard_begin", C.c_int64),
        ("shard_end", C.c_int64),
        ("backend", C.c_int32),
    ]


_lib = None


# int (*lg_allreduce_fn)(double* d_buf, int64_t count, void* stream, void* user)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


def load() -> C.CDLL:
    """Load (once) the in-tree library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2304_06200_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    dp = C.POINTER(C.c_double)
    i64p = C.POINTER(C.c_int64)
    i32p = C.POINTER(C.c_int32)
    lib.lg_problem_create.argtypes = [C.POINTER(lg_problem_desc), C.POINTER(P)]
    lib.lg_problem_destroy.argtypes = [P]
    lib.lg_problem_destroy.restype = None
    lib.lg_eval.argtypes = [P, C.c_int64, C.c_double, dp, dp, dp, i64p]
    lib.lg_cost.argtypes = [P, C.c_int64, C.c_double, dp, dp]
    lib.lg_cost_batch.argtypes = [P, C.c_int32, C.c_int64, C.c_double, dp, dp]
    lib.lg_eval_device.argtypes = [P, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.lg_plan_table.argtypes = [P, C.c_int64, C.c_double, dp, dp, i64p, i32p, i32p, dp, i64p, i32p, i32p]
    lib.lg_forward_states.argtypes = [P, C.c_int64, C.c_double, dp, dp]
    lib.lg_step_derivative.argtypes = [P, C.c_int64, C.c_double, dp, C.c_int64, C.c_int32, dp, dp]
    lib.lg_raw_size.argtypes = [P, C.c_int64]
    lib.lg_raw_size.restype = C.c_int64
    lib.lg_raw_get.argtypes = [P, dp]
    lib.lg_finalize_host.argtypes = [P, C.c_int64, dp, dp, dp]
    lib.lg_set_raw_buffer.argtypes = [P, C.c_void_p, C.c_int64]
    lib.lg_expm_plan_inputs.argtypes = [C.POINTER(lg_matrix), dp, i64p]
    lib.lg_expm_apply.argtypes = [C.POINTER(lg_matrix), C.c_int64, dp, C.c_int32, C.c_int32, dp, C.c_int32]
    lib.lg_matvec.argtypes = [C.POINTER(lg_matrix), C.c_int64, dp, dp, C.c_int32]
    lib.lg_eval_sharded.argtypes = [P, C.c_int64, C.c_double, dp, ALLREDUCE_FN, C.c_void_p, dp, dp]
    lib.lg_cost_sharded.argtypes = [P, C.c_int64, C.c_double, dp, ALLREDUCE_FN, C.c_void_p, dp]
    lib.lg_make_plan.argtypes = [C.c_double, C.c_int64, C.c_double, C.c_int32, C.c_int32, i32p, i32p, dp]
    lib.lg_make_plans_device.argtypes = [C.c_int64, dp, i64p, C.c_double, i32p, i32p, i32p, i32p]
    lib.lg_finalize_raw.argtypes = [C.c_int32, i32p, dp, i32p, i32p, C.c_int64, C.c_int32, C.c_int32, dp, dp, dp]
    lib.lg_np_cabs_host.argtypes = [C.c_int64, dp, dp]
    lib.lg_np_cabs_host.restype = None
    lib.lg_np_pairwise_host.argtypes = [C.c_int64, dp]
    lib.lg_np_pairwise_host.restype = C.c_double
    lib.lg_np_reduce_host.argtypes = [C.c_int64, dp]
    lib.lg_np_reduce_host.restype = C.c_double
    lib.lg_set_stream.argtypes = [P, C.c_void_p]
    lib.lg_bench_zgemm.argtypes = [C.c_int32, C.c_int32, C.c_int32, dp]
    lib.lg_set_timing.argtypes = [P, C.c_int]
    lib.lg_get_timing.argtypes = [P, dp, i64p]
    lib.lg_device_count.argtypes = []
    lib.lg_engine_name.argtypes = [P]
    lib.lg_engine_name.restype = C.c_char_p
    lib.lg_diag_solver_name.argtypes = [P]
    lib.lg_diag_solver_name.restype = C.c_char_p
    lib.lg_live_vector_peak.argtypes = [P]
    lib.lg_live_vector_peak.restype = C.c_int64
    lib.lg_launch_count.argtypes = []
    lib.lg_launch_count.restype = C.c_int64
    lib.lg_last_error.restype = C.c_char_p
    lib.lg_version.restype = C.c_char_p
    _lib = lib
    return lib


def last_error() -> str:
    return load().lg_last_error().decode()


def check(rc: int) -> None:
    """Map a status code onto the reference's exception types."""
    if rc == LG_OK:
        return
    msg = last_error()
    if rc == LG_INVALID_ARG:
        raise ValueError(msg)
    if rc == LG_PLANNING_INFEASIBLE:
        from .expm import PlanningError

        raise PlanningError(msg)
    if rc == LG_INDEX_ERROR:
        raise IndexError(msg)
    if rc == LG_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))
