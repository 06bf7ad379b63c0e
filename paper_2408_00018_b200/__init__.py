"""paper_2408_00018_b200 — B200-native synchronous parallel simulated annealing.

The hot path (run_synchronous and friends) lives in libparsa_b200.so: CUDA
kernels for sm_100a behind the C-ABI declared in include/parsa_b200.h.  This
package is the Python face of that ABI, mirroring the reference `parsa`
C++ API (see api.py).
"""
from .api import (  # noqa: F401
    AnnealSchedule,
    BoxDomain,
    Candidate,
    DeviceError,
    EngineConfig,
    InvalidArgument,
    LadderInfo,
    LogicError,
    NelderMeadConfig,
    NelderMeadResult,
    ObjectiveFunction,
    OutOfRange,
    PhaseBreakdown,
    Plan,
    Precision,
    ReferenceOptimum,
    RunResult,
    StartMode,
    TracePoint,
    contains,
    evaluate,
    evaluate_batch,
    evaluate_single,
    expected_evaluations,
    hybrid_run,
    ladder,
    location_error,
    nelder_mead_batch,
    nelder_mead_minimize,
    reduce_min,
    registry,
    registry_get,
    run_asynchronous,
    run_sequential,
    run_synchronous,
)
