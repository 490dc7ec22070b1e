"""ctypes binding of the C ABI in include/halp.h (libhalp_b200.so).

There is no fallback: if the in-tree library is missing or cannot be loaded
this module raises, and every compute call on a machine without a B200
returns HALP_CUDA_ERROR, which the Python layer raises as HalpCudaError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HALP_LIB") or os.path.join(HERE, "libhalp_b200.so")  # HALP_LIB: A/B a variant build

HALP_OK, HALP_INVALID_INPUT, HALP_DIVERGED, HALP_CUDA_ERROR, HALP_NCCL_ERROR, HALP_CAPACITY, HALP_UNSUPPORTED = range(7)
F64, F32, BF16 = 0, 1, 2
SQUARED, SOFTMAX = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1


class ProblemDesc(C.Structure):
    _fields_ = [
        ("X", C.c_void_p), ("dtype", C.c_int32), ("mem", C.c_int32), ("n", C.c_int64), ("d", C.c_int32),
        ("loss", C.c_int32), ("num_classes", C.c_int32), ("y", C.c_void_p), ("labels", C.c_void_p),
        ("l2", C.c_double), ("device", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
        ("nccl_id", C.c_void_p), ("collective", C.c_int32), ("qcodes", C.c_void_p), ("qbits", C.c_int32),
        ("qdelta", C.c_double),
    ]


class Config(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("epochs", C.c_int32), ("inner_steps", C.c_int64), ("bits", C.c_int32),
        ("mu", C.c_double), ("option", C.c_int32), ("full_grad_period", C.c_int32), ("seed", C.c_uint64),
        ("metric_every_passes", C.c_double), ("delta_min", C.c_double), ("divergence_limit", C.c_double),
        ("init", C.c_void_p), ("delta", C.c_double), ("algorithm", C.c_int32),
    ]


class Row(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("pass_", "seconds", "loss", "grad_norm", "delta")] + [
        ("iterate_hash", C.c_uint64), ("delta_inner", C.c_double), ("delta_aux", C.c_double)
    ]


class Record(C.Structure):
    _fields_ = [
        ("rows", C.POINTER(Row)), ("rows_cap", C.c_int32), ("rows_n", C.c_int32), ("final_iterate", C.c_void_p),
        ("status", C.c_int32), ("steps_taken", C.c_int64), ("inner_fp_vector_ops", C.c_uint64),
        ("inner_lp_vector_ops", C.c_uint64),
    ]


class Timing(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("fullgrad_ms", "finalize_ms", "inner_ms", "sample_ms")] + [
        (k, C.c_int64) for k in ("fullgrad_launches", "inner_launches", "kernel_launches", "inner_steps",
                                "h2d_bytes", "d2h_bytes")
    ]


class Plan(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("fg_threads", "fg_vec", "fg_splits", "in_ctas", "in_threads", "in_per",
                                         "fg_rows_per_stage", "fg_stages")] + [
        ("fg_split_begin", C.c_int64), ("fg_split_end", C.c_int64), ("in_levels", C.c_int32)
    ]


class BatchDesc(C.Structure):
    _fields_ = [
        ("X", C.c_void_p), ("dtype", C.c_int32), ("mem", C.c_int32), ("n", C.c_int64), ("d", C.c_int32),
        ("nprob", C.c_int32), ("y", C.c_void_p), ("l2", C.c_double), ("device", C.c_int32), ("shared", C.c_int32),
    ]


class DatagenDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n", C.c_int64), ("d", C.c_int32), ("num_classes", C.c_int32), ("dtype", C.c_int32),
        ("noise_sd", C.c_double), ("x_scale", C.c_double), ("density", C.c_double), ("seed", C.c_uint64),
    ]


# every symbol include/halp.h declares (checked by tests/test_capi_symbols.py)
SYMBOLS = [
    "halp_last_error", "halp_abi_version", "halp_problem_create", "halp_problem_destroy", "halp_problem_plan",
    "halp_run", "halp_full_gradient", "halp_set_trace", "halp_last_timing", "halp_bench_full_gradient",
    "halp_batch_create", "halp_batch_destroy", "halp_batch_run", "halp_datagen", "halp_shard_plan",
    "halp_rng_state_after", "halp_plan_for", "halp_batch_plan", "halp_rank_partial", "halp_finalize_gathered",
    "halp_make_regression", "halp_make_classification", "halp_normals", "halp_quantize_dataset",
]

_lib = None


def lib():
    """Load the in-tree libhalp_b200.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1803_03383_b200.build` (no CPU fallback)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P = C.c_void_p
    L.halp_last_error.restype = C.c_char_p
    L.halp_abi_version.restype = C.c_int32
    L.halp_problem_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(P)]
    L.halp_problem_destroy.argtypes = [P]
    L.halp_problem_destroy.restype = None
    L.halp_problem_plan.argtypes = [P, C.POINTER(Plan)]
    L.halp_run.argtypes = [P, C.POINTER(Config), C.POINTER(Record)]
    L.halp_full_gradient.argtypes = [P, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
    L.halp_set_trace.argtypes = [P, C.c_void_p, C.c_int64]
    L.halp_last_timing.argtypes = [P, C.POINTER(Timing)]
    L.halp_bench_full_gradient.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    L.halp_batch_create.argtypes = [C.POINTER(BatchDesc), C.POINTER(P)]
    L.halp_batch_destroy.argtypes = [P]
    L.halp_batch_destroy.restype = None
    L.halp_batch_run.argtypes = [P, C.POINTER(Config), C.POINTER(Record), C.POINTER(C.c_double)]
    L.halp_batch_plan.argtypes = [P, C.POINTER(Plan)]
    L.halp_datagen.argtypes = [C.POINTER(DatagenDesc), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    L.halp_shard_plan.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32] + [
        C.POINTER(C.c_int64)] * 5
    L.halp_plan_for.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Plan)]
    L.halp_rank_partial.argtypes = [P, C.c_void_p, C.c_void_p]
    L.halp_finalize_gathered.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
    L.halp_make_regression.argtypes = [C.c_int64, C.c_int32, C.c_double, C.c_uint64, C.c_void_p, C.c_void_p]
    L.halp_make_classification.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_void_p,
                                           C.c_void_p]
    L.halp_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
    L.halp_quantize_dataset.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p,
                                        C.POINTER(C.c_double)]
    L.halp_rng_state_after.restype = C.c_uint64
    L.halp_rng_state_after.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    _lib = L
    return L


def last_error() -> str:
    return lib().halp_last_error().decode()
