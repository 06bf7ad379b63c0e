"""ctypes mirror of include/parsa_b200.h (the C-ABI drop-in boundary).

Struct layouts here must match the header field for field; tests/test_abi.py
checks sizes and offsets against the compiled library.
"""
from __future__ import annotations

import ctypes as C
import os

ABI_VERSION = 2  # include/parsa_b200.h PSA_ABI_VERSION (2: psa_objective.param, PSA_FN_CONSTANT)
PSA_OK = 0
PSA_ERR_INVALID_ARGUMENT = 1
PSA_ERR_OUT_OF_RANGE = 2
PSA_ERR_LOGIC = 3
PSA_ERR_CUDA = 4
PSA_ERR_NO_DEVICE = 5

PSA_F64 = 0
PSA_F32 = 1
PSA_SHARED_POINT = 0
PSA_RANDOM_PER_CHAIN = 1

FAMILIES = [
    "SCHWEFEL", "ACKLEY", "BRANIN", "COSINE_MIXTURE", "DEKKERS_AARTS", "EASOM",
    "EXPONENTIAL", "GOLDSTEIN_PRICE", "GRIEWANK", "HIMMELBLAU", "LEVY_MONTALVO",
    "MOD_LANGERMAN", "MICHALEWICZ", "RASTRIGIN", "ROSENBROCK", "SALOMON",
    "SIX_HUMP_CAMEL", "SHUBERT", "SHEKEL5", "SHEKEL7", "SHEKEL10", "SHEKEL_FOXHOLES",
    "SPHERE", "CONSTANT",
]
FAMILY = {name: i for i, name in enumerate(FAMILIES)}


class psa_objective(C.Structure):
    _fields_ = [
        ("id", C.c_char_p),
        ("family", C.c_int32),
        ("dim", C.c_int32),
        ("lower", C.POINTER(C.c_double)),
        ("upper", C.POINTER(C.c_double)),
        ("param", C.c_double),
    ]


class psa_schedule(C.Structure):
    _fields_ = [
        ("t0", C.c_double),
        ("t_min", C.c_double),
        ("rho", C.c_double),
        ("sweep_length", C.c_int32),
        ("reserved", C.c_int32),
    ]


class psa_engine_config(C.Structure):
    _fields_ = [
        ("n_chains", C.c_int32),
        ("start_mode", C.c_int32),
        ("start_point", C.POINTER(C.c_double)),
        ("start_point_len", C.c_int32),
        ("precision", C.c_int32),
        ("seed", C.c_uint64),
        ("workers", C.c_int32),
        ("reserved", C.c_int32),
        ("schedule", psa_schedule),
    ]


class psa_trace_point(C.Structure):
    _fields_ = [
        ("level", C.c_int32),
        ("reserved", C.c_int32),
        ("cumulative_evals", C.c_uint64),
        ("best_f", C.c_double),
    ]


class psa_run_result(C.Structure):
    _fields_ = [
        ("best_x", C.POINTER(C.c_double)),
        ("trace", C.POINTER(psa_trace_point)),
        ("trace_capacity", C.c_int32),
        ("trace_len", C.c_int32),
        ("best_f", C.c_double),
        ("evaluations", C.c_uint64),
        ("wall_time_s", C.c_double),
        ("winning_chain", C.c_int32),
        ("has_phases", C.c_int32),
        ("rng_draws", C.c_uint64),
        ("sa_evaluations", C.c_uint64),
        ("refine_evaluations", C.c_uint64),
        ("sa_best_f", C.c_double),
    ]


class psa_nm_config(C.Structure):
    _fields_ = [
        ("reflect", C.c_double),
        ("expand", C.c_double),
        ("contract", C.c_double),
        ("shrink", C.c_double),
        ("f_tol", C.c_double),
        ("x_tol", C.c_double),
        ("max_iters", C.c_int32),
        ("reserved", C.c_int32),
    ]


class psa_plan_options(C.Structure):
    _fields_ = [
        ("max_blocks", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("reserved", C.c_int32),
    ]


class psa_nm_result(C.Structure):
    _fields_ = [
        ("x_best", C.POINTER(C.c_double)),
        ("f_best", C.c_double),
        ("iterations", C.c_int32),
        ("reserved", C.c_int32),
        ("evaluations", C.c_uint64),
    ]


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSA_LIB_PATH") or os.path.join(PKG_DIR, "libparsa_b200.so")

_lib = None


def _declare(lib):
    P = C.POINTER
    st = C.c_int32
    sig = {
        "psa_abi_version": (C.c_int32, []),
        "psa_last_error": (C.c_char_p, []),
        "psa_device_count": (C.c_int32, []),
        "psa_schedule_validate": (st, [P(psa_schedule)]),
        "psa_ladder": (st, [P(psa_schedule), P(C.c_double), C.c_int32, P(C.c_int32)]),
        "psa_expected_evaluations": (st, [P(psa_schedule), C.c_int32, P(C.c_uint64)]),
        "psa_reduce_min": (st, [P(C.c_double), P(C.c_int32), C.c_int32, P(C.c_int32)]),
        "psa_run_sequential": (st, [P(psa_objective), P(psa_engine_config), P(psa_run_result)]),
        "psa_run_asynchronous": (st, [P(psa_objective), P(psa_engine_config), P(psa_run_result)]),
        "psa_run_synchronous": (st, [P(psa_objective), P(psa_engine_config), P(psa_run_result)]),
        "psa_nelder_mead_minimize": (st, [P(psa_objective), P(C.c_double), P(psa_nm_config), P(psa_nm_result)]),
        "psa_hybrid_run": (st, [P(psa_objective), P(psa_engine_config), P(psa_schedule), P(psa_nm_config), P(psa_run_result)]),
        "psa_plan_create": (st, [P(psa_objective), P(psa_engine_config), C.c_int32, C.c_int32, C.c_int32, P(C.c_void_p)]),
        "psa_plan_launch": (st, [C.c_void_p, C.c_void_p]),
        "psa_plan_fetch": (st, [C.c_void_p, C.c_void_p, P(psa_run_result)]),
        "psa_plan_info": (st, [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32)]),
        "psa_plan_destroy": (st, [C.c_void_p]),
        "psa_device_uniforms": (st, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int32, P(C.c_double)]),
        "psa_device_philox": (st, [P(C.c_uint32), P(C.c_uint32), C.c_int32, P(C.c_uint32)]),
        "psa_device_evaluate": (st, [P(psa_objective), C.c_int32, P(C.c_double), C.c_int32, P(C.c_double)]),
        "psa_libm_sinf": (C.c_float, [C.c_float]),
        "psa_libm_cosf": (C.c_float, [C.c_float]),
        "psa_libm_expf": (C.c_float, [C.c_float]),
        "psa_libm_sin": (C.c_double, [C.c_double]),
        "psa_libm_cos": (C.c_double, [C.c_double]),
        "psa_libm_exp": (C.c_double, [C.c_double]),
        "psa_plan_level_detail": (st, [C.c_void_p, P(C.c_int32), P(C.c_double), C.c_int32]),
        "psa_device_libm_f32": (st, [C.c_int32, P(C.c_float), C.c_int32, P(C.c_float), P(C.c_int32)]),
        "psa_device_libm_f64": (st, [C.c_int32, P(C.c_double), C.c_int32, P(C.c_double)]),
        "psa_plan_create_ex": (st, [P(psa_objective), P(psa_engine_config), C.c_int32, C.c_int32, C.c_int32,
                                    P(psa_plan_options), P(C.c_void_p)]),
        "psa_plan_mailbox": (st, [C.c_void_p, P(C.c_void_p), P(C.c_uint64)]),
        "psa_plan_mailbox_ipc_handle": (st, [C.c_void_p, C.c_void_p]),
        "psa_ipc_open": (st, [C.c_void_p, P(C.c_void_p)]),
        "psa_ipc_close": (st, [C.c_void_p]),
        "psa_plan_set_peers": (st, [C.c_void_p, P(C.c_void_p), C.c_int32]),
        "psa_plan_describe": (st, [C.c_void_p, C.c_char_p, C.c_int32]),
        "psa_plan_stats": (st, [C.c_void_p, P(C.c_uint64)]),
        "psa_device_metropolis_check": (st, [C.c_int32, C.c_uint64, C.c_uint64, P(C.c_uint64)]),
        "psa_nelder_mead_batch": (st, [P(psa_objective), P(C.c_double), C.c_int32, P(psa_nm_config), P(C.c_double),
                                       P(C.c_double), P(C.c_int32), P(C.c_uint64)]),
        "psa_metropolis_sweep": (st, [P(psa_objective), C.c_int32, P(C.c_double), P(C.c_double), C.c_uint64,
                                      C.c_uint32, C.c_uint32, P(C.c_uint64), C.c_double, C.c_int32,
                                      P(C.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return sig


# Every symbol include/parsa_b200.h declares (tests/test_abi.py checks the
# header and the library against this list).
EXPORTED_SYMBOLS = [
    "psa_abi_version", "psa_last_error", "psa_device_count", "psa_schedule_validate",
    "psa_ladder", "psa_expected_evaluations", "psa_reduce_min", "psa_run_sequential",
    "psa_run_asynchronous", "psa_run_synchronous", "psa_nelder_mead_minimize",
    "psa_hybrid_run", "psa_plan_create", "psa_plan_launch", "psa_plan_fetch", "psa_plan_info",
    "psa_plan_destroy", "psa_device_uniforms", "psa_device_philox", "psa_device_evaluate",
    "psa_libm_sinf", "psa_libm_cosf", "psa_libm_expf", "psa_libm_sin", "psa_libm_cos",
    "psa_libm_exp", "psa_plan_level_detail", "psa_device_libm_f32", "psa_device_libm_f64",
    "psa_plan_create_ex", "psa_plan_mailbox", "psa_plan_mailbox_ipc_handle", "psa_ipc_open",
    "psa_ipc_close", "psa_plan_set_peers", "psa_plan_describe", "psa_metropolis_sweep", "psa_nelder_mead_batch",
    "psa_plan_stats", "psa_device_metropolis_check",
]


def load_library(path: str | None = None):
    """Load the compiled CUDA library.  There is no fallback: a missing
    library is an error (build it with `python -c "import __graft_entry__ as g; g.build()"`)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"parsa_b200: CUDA library {p} is missing; run __graft_entry__.build()")
    lib = C.CDLL(p)
    _declare(lib)
    if lib.psa_abi_version() != ABI_VERSION:
        raise RuntimeError("parsa_b200: ABI version mismatch")
    if path is None:
        _lib = lib
    return lib
