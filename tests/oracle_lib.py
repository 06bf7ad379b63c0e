"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``oracle()``  -> oracle/liboracle.so, the plain-C restatement (sa_oracle.c)
* ``ref()``     -> oracle/_ref/libparsa_ref.so, the reference's own sources
  compiled unchanged (None when it was never built, e.g. a box that did not
  receive it).

Also holds small marshalling helpers shared by the tests so that oracle, ref
and the product library are driven with identical C structs.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2408_00018_b200 import _abi  # noqa: E402
from paper_2408_00018_b200._abi import (  # noqa: E402
    psa_engine_config,
    psa_nm_config,
    psa_nm_result,
    psa_objective,
    psa_run_result,
    psa_schedule,
    psa_trace_point,
)

ORACLE_PATH = os.path.join(ROOT, "oracle", "liboracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libparsa_ref.so")

_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_PATH):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_PATH)
        P = C.POINTER
        lib.orc_philox4x32_10.argtypes = [P(C.c_uint32), C.c_uint32, C.c_uint32, P(C.c_uint32)]
        lib.orc_uniforms.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int32, P(C.c_double)]
        lib.orc_coordinate_index.restype = C.c_int32
        lib.orc_coordinate_index.argtypes = [C.c_double, C.c_int32]
        lib.orc_schedule_validate.argtypes = [P(psa_schedule)]
        lib.orc_ladder.restype = C.c_int32
        lib.orc_ladder.argtypes = [P(psa_schedule), P(C.c_double), C.c_int32]
        lib.orc_expected_evaluations.restype = C.c_uint64
        lib.orc_expected_evaluations.argtypes = [P(psa_schedule), C.c_int32]
        lib.orc_evaluate.restype = C.c_double
        lib.orc_evaluate.argtypes = [C.c_int32, C.c_int32, P(C.c_double)]
        lib.orc_evaluate_single.restype = C.c_double
        lib.orc_evaluate_single.argtypes = [C.c_int32, C.c_int32, P(C.c_double)]
        lib.orc_reduce_min.restype = C.c_int32
        lib.orc_reduce_min.argtypes = [P(C.c_double), P(C.c_int32), C.c_int32]
        lib.orc_run_synchronous.argtypes = [P(psa_objective), P(psa_engine_config), P(psa_run_result), C.c_void_p]
        lib.orc_run_asynchronous.argtypes = [P(psa_objective), P(psa_engine_config), P(psa_run_result)]
        lib.orc_nelder_mead_minimize.argtypes = [P(psa_objective), P(C.c_double), P(psa_nm_config), P(psa_nm_result)]
        lib.orc_hybrid_run.argtypes = [P(psa_objective), P(psa_engine_config), P(psa_schedule), P(psa_nm_config), P(psa_run_result)]
        _oracle = lib
    return _oracle


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        lib = C.CDLL(REF_PATH)
        P = C.POINTER
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_max_threads.restype = C.c_int32
        lib.ref_philox4x32_10.argtypes = [P(C.c_uint32), C.c_uint32, C.c_uint32, P(C.c_uint32)]
        lib.ref_uniforms.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, P(C.c_double)]
        lib.ref_coordinate_indices.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, P(C.c_int32)]
        lib.ref_ladder.argtypes = [P(psa_schedule), P(C.c_double), C.c_int32, P(C.c_int32)]
        lib.ref_expected_evaluations.argtypes = [P(psa_schedule), C.c_int32, P(C.c_uint64)]
        lib.ref_evaluate.argtypes = [P(psa_objective), C.c_int32, P(C.c_double), C.c_int32, P(C.c_double)]
        lib.ref_reduce_min.argtypes = [P(C.c_double), P(C.c_int32), C.c_int32, P(C.c_int32)]
        lib.ref_run.argtypes = [C.c_int32, P(psa_objective), P(psa_engine_config), P(psa_run_result)]
        lib.ref_hybrid_run.argtypes = [P(psa_objective), P(psa_engine_config), P(psa_schedule), P(psa_nm_config), P(psa_run_result)]
        lib.ref_nelder_mead.argtypes = [P(psa_objective), P(C.c_double), P(psa_nm_config), P(psa_nm_result)]
        _ref = lib
    return _ref


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Problem:
    """Keeps the numpy buffers behind a psa_objective alive."""

    def __init__(self, family: str | int, dim: int, lo: float | np.ndarray, hi: float | np.ndarray,
                 ident: str = "fn", param: float = 0.0):
        self.family = _abi.FAMILY[family] if isinstance(family, str) else int(family)
        self.dim = int(dim)
        self.lower = np.ascontiguousarray(np.broadcast_to(np.asarray(lo, dtype=np.float64), (dim,)))
        self.upper = np.ascontiguousarray(np.broadcast_to(np.asarray(hi, dtype=np.float64), (dim,)))
        self._id = ident.encode()
        self.c = psa_objective(self._id, self.family, self.dim, dptr(self.lower), dptr(self.upper), float(param))


class Config:
    def __init__(self, chains: int, schedule=(5.0, 0.5, 0.7, 10), seed: int = 0, precision: int = 0,
                 start_mode: int = 0, start_point=None, workers: int = 1):
        self.sp = None if start_point is None else np.ascontiguousarray(start_point, dtype=np.float64)
        t0, tmin, rho, n = schedule
        self.c = psa_engine_config(
            n_chains=chains, start_mode=start_mode,
            start_point=dptr(self.sp) if self.sp is not None else None,
            start_point_len=0 if self.sp is None else len(self.sp),
            precision=precision, seed=seed, workers=workers,
            schedule=psa_schedule(t0, tmin, rho, n, 0))


class Result:
    def __init__(self, dim: int, trace_capacity: int):
        self.best_x = np.zeros(dim, dtype=np.float64)
        self.trace = (psa_trace_point * max(1, trace_capacity))()
        self.c = psa_run_result()
        self.c.best_x = dptr(self.best_x)
        self.c.trace = self.trace
        self.c.trace_capacity = trace_capacity

    def as_dict(self):
        r = self.c
        n = min(r.trace_len, r.trace_capacity)
        return {
            "best_x": self.best_x.copy(),
            "best_f": r.best_f,
            "evaluations": r.evaluations,
            "winning_chain": r.winning_chain,
            "rng_draws": r.rng_draws,
            "trace": [(self.trace[i].level, self.trace[i].cumulative_evals, self.trace[i].best_f)
                      for i in range(n)],
            "trace_len": r.trace_len,
            "has_phases": r.has_phases,
            "sa_evaluations": r.sa_evaluations,
            "refine_evaluations": r.refine_evaluations,
            "sa_best_f": r.sa_best_f,
            "wall_time_s": r.wall_time_s,
        }


def levels_of(schedule) -> int:
    t0, tmin, rho, n = schedule
    s = psa_schedule(t0, tmin, rho, n, 0)
    return oracle().orc_ladder(C.byref(s), None, 0)


def oracle_sync(prob: Problem, cfg: Config, detail: bool = False):
    L = levels_of_cfg(cfg)
    res = Result(prob.dim, L + 1)
    if detail:
        winners = np.zeros(L, dtype=np.int32)
        wf = np.zeros(L, dtype=np.float64)

        class Detail(C.Structure):
            _fields_ = [("winner", C.POINTER(C.c_int32)), ("winner_f", C.POINTER(C.c_double)),
                        ("accept_mask", C.POINTER(C.c_uint32))]

        d = Detail(winners.ctypes.data_as(C.POINTER(C.c_int32)), dptr(wf), None)
        rc = oracle().orc_run_synchronous(C.byref(prob.c), C.byref(cfg.c), C.byref(res.c), C.byref(d))
        out = res.as_dict()
        out["level_winner"] = winners
        out["level_winner_f"] = wf
    else:
        rc = oracle().orc_run_synchronous(C.byref(prob.c), C.byref(cfg.c), C.byref(res.c), None)
        out = res.as_dict()
    out["rc"] = rc
    return out


def oracle_async(prob: Problem, cfg: Config):
    L = levels_of_cfg(cfg)
    res = Result(prob.dim, L + 1)
    rc = oracle().orc_run_asynchronous(C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
    out = res.as_dict()
    out["rc"] = rc
    return out


def ref_run(engine: int, prob: Problem, cfg: Config):
    L = levels_of_cfg(cfg)
    res = Result(prob.dim, L + 1)
    rc = ref().ref_run(engine, C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
    out = res.as_dict()
    out["rc"] = rc
    out["err"] = ref().ref_last_error().decode() if rc else ""
    return out


def levels_of_cfg(cfg: Config) -> int:
    s = cfg.c.schedule
    return oracle().orc_ladder(C.byref(s), None, 0)


def same_run(a: dict, b: dict, check_wall: bool = False) -> list[str]:
    """Bitwise comparison of two run dicts; returns the differing fields."""
    diffs = []
    if not np.array_equal(a["best_x"].view(np.uint64), b["best_x"].view(np.uint64)):
        diffs.append("best_x")
    for k in ("best_f", "evaluations", "winning_chain", "rng_draws", "trace_len"):
        x, y = a[k], b[k]
        if isinstance(x, float):
            if np.float64(x).view(np.uint64) != np.float64(y).view(np.uint64):
                diffs.append(k)
        elif x != y:
            diffs.append(k)
    ta, tb = a["trace"], b["trace"]
    if len(ta) != len(tb):
        diffs.append("trace")
    else:
        for (la, ca, fa), (lb, cb, fb) in zip(ta, tb):
            if la != lb or ca != cb or np.float64(fa).view(np.uint64) != np.float64(fb).view(np.uint64):
                diffs.append("trace")
                break
    return diffs
