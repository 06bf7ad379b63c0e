"""Python mirror of the reference `parsa` C++ API over the B200 C-ABI.

Names, fields, defaults and error behaviour follow the reference headers
(proj/include/parsa/{objectives,sa_core,engines,nelder_mead}.hpp) so that a
reference user (and the parity tests) can switch over unchanged:

    f = registry_get("F0_b")
    cfg = EngineConfig(n_chains=1024, schedule=AnnealSchedule(1000, 0.01, 0.99, 100))
    res = run_synchronous(f, cfg)

Every engine call goes through libparsa_b200.so (CUDA, sm_100a).  There is
no CPU fallback: on a host without a B200 the engines raise DeviceError.
Exceptions map the reference's: std::invalid_argument -> InvalidArgument
(a ValueError), std::out_of_range -> OutOfRange (a LookupError),
std::logic_error -> LogicError.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (
    psa_engine_config,
    psa_nm_config,
    psa_nm_result,
    psa_objective,
    psa_run_result,
    psa_schedule,
    psa_trace_point,
)


# ---------------------------------------------------------------------------
# errors
# ---------------------------------------------------------------------------

class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(LookupError):
    """std::out_of_range"""


class LogicError(RuntimeError):
    """std::logic_error"""


class DeviceError(RuntimeError):
    """CUDA failure or no usable B200 (the library has no CPU fallback)."""


def _raise(lib, status: int):
    if status == _abi.PSA_OK:
        return
    msg = lib.psa_last_error().decode()
    if status == _abi.PSA_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _abi.PSA_ERR_OUT_OF_RANGE:
        raise OutOfRange(msg)
    if status == _abi.PSA_ERR_LOGIC:
        raise LogicError(msg)
    raise DeviceError(msg)


def _lib():
    return _abi.load_library()


# ---------------------------------------------------------------------------
# objectives.hpp
# ---------------------------------------------------------------------------

class Precision(IntEnum):
    f64 = 0
    f32 = 1


class StartMode(IntEnum):
    shared_point = 0
    random_per_chain = 1


@dataclass
class BoxDomain:
    lower: list
    upper: list

    def dim(self) -> int:
        return len(self.lower)

    def width(self, k: int) -> float:
        return self.upper[k] - self.lower[k]

    def center(self) -> list:
        return [0.5 * (lo + hi) for lo, hi in zip(self.lower, self.upper)]


@dataclass
class ReferenceOptimum:
    f_star: float = 0.0
    minimizers: list = field(default_factory=list)
    location_known: bool = False
    location_at_origin: bool = False


@dataclass
class ObjectiveFunction:
    """ObjectiveFunction (objectives.hpp:31-39).  Instead of host eval
    pointers the descriptor names the device cost family (`family`, one of
    _abi.FAMILIES); any dim/domain may be set, as with the reference."""
    id: str
    name: str
    dim: int
    domain: BoxDomain
    family: str
    reference: ReferenceOptimum = field(default_factory=ReferenceOptimum)
    param: float = 0.0  # family parameter: the value of family "CONSTANT"

    def with_dim(self, n: int, lo: Optional[float] = None, hi: Optional[float] = None) -> "ObjectiveFunction":
        """Copy resized to n dimensions on a uniform box (how the configs use
        Schwefel at n = 10 / 100 / 500)."""
        lo = self.domain.lower[0] if lo is None else lo
        hi = self.domain.upper[0] if hi is None else hi
        return ObjectiveFunction(self.id, self.name, n, BoxDomain([lo] * n, [hi] * n), self.family,
                                 ReferenceOptimum(self.reference.f_star,
                                                  [[m[0]] * n for m in self.reference.minimizers[:1]]
                                                  if self.reference.minimizers else [],
                                                  self.reference.location_known,
                                                  self.reference.location_at_origin), self.param)


def _uniform(n, lo, hi):
    return BoxDomain([float(lo)] * n, [float(hi)] * n)


def _at_origin(n, f_star):
    return ReferenceOptimum(f_star, [[0.0] * n], True, True)


def _at_points(f_star, pts):
    return ReferenceOptimum(f_star, [list(map(float, p)) for p in pts], True, False)


def _value_only(f_star):
    return ReferenceOptimum(f_star, [], False, False)


def _build_registry() -> list:
    """The 41 entries of the reference registry (objectives.cpp:337-469)."""
    pi = math.pi
    reg = []
    for sfx, n in (("a", 8), ("b", 16), ("c", 32), ("d", 64), ("e", 128), ("f", 256), ("g", 512)):
        reg.append(ObjectiveFunction(f"F0_{sfx}", "Schwefel (normalized)", n, _uniform(n, -512, 512),
                                     "SCHWEFEL", _at_points(-418.982887, [[420.968746] * n])))
    for sfx, n in (("a", 30), ("b", 100), ("c", 200), ("d", 400)):
        reg.append(ObjectiveFunction(f"F1_{sfx}", "Ackley", n, _uniform(n, -30, 30), "ACKLEY", _at_origin(n, 0.0)))
    reg.append(ObjectiveFunction("F2", "Branin", 2, _uniform(2, -20, 20), "BRANIN",
                                 _at_points(0.397887, [[-pi, 12.275], [pi, 2.275], [9.425, 2.475]])))
    reg.append(ObjectiveFunction("F3_a", "Cosine mixture", 2, _uniform(2, -1, 1), "COSINE_MIXTURE", _at_origin(2, -0.2)))
    reg.append(ObjectiveFunction("F3_b", "Cosine mixture", 4, _uniform(4, -1, 1), "COSINE_MIXTURE", _at_origin(4, -0.4)))
    reg.append(ObjectiveFunction("F4", "Dekkers and Aarts", 2, _uniform(2, -20, 20), "DEKKERS_AARTS",
                                 _at_points(-24776.518, [[0.0, -14.945], [0.0, 14.945]])))
    reg.append(ObjectiveFunction("F5", "Easom", 2, _uniform(2, -10, 10), "EASOM", _at_points(-1.0, [[pi, pi]])))
    reg.append(ObjectiveFunction("F6", "Exponential", 4, _uniform(4, -1, 1), "EXPONENTIAL", _at_origin(4, -1.0)))
    reg.append(ObjectiveFunction("F7", "Goldstein and Price", 2, _uniform(2, -2, 2), "GOLDSTEIN_PRICE",
                                 _at_points(3.0, [[0.0, -1.0]])))
    for sfx, n in (("a", 100), ("b", 200), ("c", 400)):
        reg.append(ObjectiveFunction(f"F8_{sfx}", "Griewank", n, _uniform(n, -600, 600), "GRIEWANK", _at_origin(n, 0.0)))
    reg.append(ObjectiveFunction("F9", "Himmelblau", 2, _uniform(2, -6, 6), "HIMMELBLAU",
                                 _at_points(0.0, [[3.0, 2.0], [-2.805118, 3.131312], [-3.779310, -3.283186],
                                                  [3.584428, -1.848126]])))
    for sfx, n in (("a", 2), ("b", 5), ("c", 10)):
        reg.append(ObjectiveFunction(f"F10_{sfx}", "Levy and Montalvo", n, _uniform(n, -10, 10), "LEVY_MONTALVO",
                                     _at_points(0.0, [[-1.0] * n])))
    reg.append(ObjectiveFunction("F11_a", "Modified Langerman", 2, _uniform(2, 0, 10), "MOD_LANGERMAN",
                                 _at_points(-1.080938, [[9.6810707, 0.6666515]])))
    reg.append(ObjectiveFunction("F11_b", "Modified Langerman", 5, _uniform(5, 0, 10), "MOD_LANGERMAN",
                                 _at_points(-0.964999, [[8.074000, 8.777001, 3.467004, 1.863013, 6.707995]])))
    for sfx, n, fs in (("a", 2, -1.8013), ("b", 5, -4.6877), ("c", 10, -9.6602)):
        reg.append(ObjectiveFunction(f"F12_{sfx}", "Michalewicz", n, _uniform(n, 0, pi), "MICHALEWICZ", _value_only(fs)))
    reg.append(ObjectiveFunction("F13_a", "Rastrigin", 100, _uniform(100, -5.12, 5.12), "RASTRIGIN", _at_origin(100, 0.0)))
    reg.append(ObjectiveFunction("F13_b", "Rastrigin", 400, _uniform(400, -5.12, 5.12), "RASTRIGIN", _at_origin(400, 0.0)))
    reg.append(ObjectiveFunction("F14", "Generalized Rosenbrock", 4, _uniform(4, -2.048, 2.048), "ROSENBROCK",
                                 _at_points(0.0, [[1.0, 1.0, 1.0, 1.0]])))
    reg.append(ObjectiveFunction("F15", "Salomon", 10, _uniform(10, -100, 100), "SALOMON", _at_origin(10, 0.0)))
    reg.append(ObjectiveFunction("F16", "Six-Hump Camel Back", 2, BoxDomain([-3.0, -2.0], [3.0, 2.0]), "SIX_HUMP_CAMEL",
                                 _at_points(-1.0316, [[-0.0898, 0.7126], [0.0898, -0.7126]])))
    reg.append(ObjectiveFunction("F17", "Shubert", 2, _uniform(2, -10, 10), "SHUBERT", _at_points(-186.7309, [
        [-7.0835, 4.8580], [-7.0835, -7.7083], [-1.4251, -7.0835], [5.4828, 4.8580], [-1.4251, -0.8003],
        [4.8580, 5.4828], [-7.7083, -7.0835], [-7.0835, -1.4251], [-7.7083, -0.8003], [-7.7083, 5.4828],
        [-0.8003, -7.7083], [-0.8003, -1.4251], [-0.8003, 4.8580], [-1.4251, 5.4828], [5.4828, -7.7083],
        [4.8580, -7.0835], [5.4828, -1.4251], [4.8580, -0.8003]])))
    for sfx, fam, fs in (("a", "SHEKEL5", -10.1532), ("b", "SHEKEL7", -10.4029), ("c", "SHEKEL10", -10.5364)):
        m = {"SHEKEL5": 5, "SHEKEL7": 7, "SHEKEL10": 10}[fam]
        reg.append(ObjectiveFunction(f"F18_{sfx}", f"Shekel {m}", 4, _uniform(4, 0, 10), fam,
                                     _at_points(fs, [[4.0, 4.0, 4.0, 4.0]])))
    reg.append(ObjectiveFunction("F19_a", "Modified Shekel Foxholes", 2, _uniform(2, -5, 15), "SHEKEL_FOXHOLES",
                                 _at_points(-12.1190, [[8.024, 9.146]])))
    reg.append(ObjectiveFunction("F19_b", "Modified Shekel Foxholes", 5, _uniform(5, -5, 15), "SHEKEL_FOXHOLES",
                                 _at_points(-10.4056, [[8.025, 9.152, 5.114, 7.621, 4.564]])))
    return reg


_REGISTRY = _build_registry()


def registry() -> list:
    return _REGISTRY


def registry_get(ident: str) -> ObjectiveFunction:
    """objectives.cpp:539-551"""
    for f in _REGISTRY:
        if f.id == ident:
            return f
    raise OutOfRange(f"unknown function id '{ident}'; valid ids: " + " ".join(f.id for f in _REGISTRY))


def contains(domain: BoxDomain, x: Sequence[float]) -> bool:
    """objectives.cpp:490-496"""
    if len(x) != domain.dim():
        raise InvalidArgument(f"contains: expected dimension {domain.dim()}, got {len(x)}")
    return all(lo <= v <= hi for v, lo, hi in zip(x, domain.lower, domain.upper))


def evaluate(f: ObjectiveFunction, x: Sequence[float], precision: Precision = Precision.f64) -> float:
    """f(x) computed by the DEVICE cost kernel (objectives.cpp:498-510 semantics:
    f32 rounds every coordinate to float and evaluates in float)."""
    if len(x) != f.dim:
        what = "evaluate_single" if precision == Precision.f32 else "evaluate"
        raise InvalidArgument(f"{what}: expected dimension {f.dim}, got {len(x)}")
    return float(evaluate_batch(f, np.asarray([x], dtype=np.float64), precision)[0])


def evaluate_single(f: ObjectiveFunction, x: Sequence[float]) -> float:
    return evaluate(f, x, Precision.f32)


def evaluate_batch(f: ObjectiveFunction, X: np.ndarray, precision: Precision = Precision.f64) -> np.ndarray:
    lib = _lib()
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.zeros(X.shape[0], dtype=np.float64)
    h = _Objective(f)
    _raise(lib, lib.psa_device_evaluate(C.byref(h.c), int(precision),
                                        X.ctypes.data_as(C.POINTER(C.c_double)), X.shape[0],
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def location_error(f: ObjectiveFunction, x: Sequence[float]) -> float:
    """objectives.cpp:512-530"""
    if len(x) != f.dim:
        raise InvalidArgument(f"location_error: expected dimension {f.dim}, got {len(x)}")
    if not f.reference.location_known:
        raise InvalidArgument("location_error: exact minimizer unknown for " + f.id)
    best = math.inf
    for m in f.reference.minimizers:
        d2 = 0.0
        n2 = 0.0
        for k in range(f.dim):
            d = x[k] - m[k]
            d2 += d * d
            n2 += m[k] * m[k]
        err = math.sqrt(d2)
        if not f.reference.location_at_origin:
            err /= math.sqrt(n2)
        best = min(best, err)
    return best


# ---------------------------------------------------------------------------
# sa_core.hpp
# ---------------------------------------------------------------------------

@dataclass
class AnnealSchedule:
    t0: float = 1.0
    t_min: float = 1e-3
    rho: float = 0.99
    sweep_length: int = 100

    def _c(self):
        return psa_schedule(float(self.t0), float(self.t_min), float(self.rho), int(self.sweep_length), 0)

    def validate(self):
        lib = _lib()
        s = self._c()
        _raise(lib, lib.psa_schedule_validate(C.byref(s)))


@dataclass
class LadderInfo:
    levels: int
    temperatures: list


def ladder(sched: AnnealSchedule) -> LadderInfo:
    lib = _lib()
    s = sched._c()
    n = C.c_int32()
    _raise(lib, lib.psa_ladder(C.byref(s), None, 0, C.byref(n)))
    buf = (C.c_double * n.value)()
    _raise(lib, lib.psa_ladder(C.byref(s), buf, n.value, C.byref(n)))
    return LadderInfo(n.value, list(buf))


def expected_evaluations(sched: AnnealSchedule, n_chains: int) -> int:
    lib = _lib()
    s = sched._c()
    out = C.c_uint64()
    _raise(lib, lib.psa_expected_evaluations(C.byref(s), int(n_chains), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# engines.hpp
# ---------------------------------------------------------------------------

@dataclass
class EngineConfig:
    n_chains: int = 1
    start_mode: StartMode = StartMode.shared_point
    start_point: list = field(default_factory=list)
    schedule: AnnealSchedule = field(default_factory=AnnealSchedule)
    precision: Precision = Precision.f64
    seed: int = 0
    workers: int = 0


@dataclass
class TracePoint:
    level: int = 0
    cumulative_evals: int = 0
    best_f: float = 0.0


@dataclass
class PhaseBreakdown:
    sa_evaluations: int = 0
    refine_evaluations: int = 0
    sa_best_f: float = 0.0


@dataclass
class RunResult:
    best_x: list = field(default_factory=list)
    best_f: float = 0.0
    evaluations: int = 0
    wall_time_s: float = 0.0
    trace: list = field(default_factory=list)
    winning_chain: int = 0
    rng_draws: int = 0
    phases: Optional[PhaseBreakdown] = None


@dataclass
class Candidate:
    x: list
    f_value: float
    chain_index: int


def reduce_min(candidates: Sequence[Candidate]) -> Candidate:
    """engines.cpp:55-64 (host selection rule; the device uses the same order)."""
    lib = _lib()
    if len(candidates) == 0:
        raise InvalidArgument("reduce_min: empty candidate list")
    f = (C.c_double * len(candidates))(*[c.f_value for c in candidates])
    ch = (C.c_int32 * len(candidates))(*[c.chain_index for c in candidates])
    pos = C.c_int32()
    _raise(lib, lib.psa_reduce_min(f, ch, len(candidates), C.byref(pos)))
    return candidates[pos.value]


class _Objective:
    """Keeps the buffers behind a psa_objective alive."""

    def __init__(self, f: ObjectiveFunction):
        if f.family not in _abi.FAMILY:
            raise InvalidArgument(f"parsa_b200: no device implementation for objective '{f.id}'")
        self.lower = np.ascontiguousarray(f.domain.lower, dtype=np.float64)
        self.upper = np.ascontiguousarray(f.domain.upper, dtype=np.float64)
        if len(self.lower) != f.dim or len(self.upper) != f.dim:
            raise InvalidArgument(f"parsa_b200: domain of '{f.id}' does not match dim {f.dim}")
        self._id = f.id.encode()
        self.c = psa_objective(self._id, _abi.FAMILY[f.family], int(f.dim),
                               self.lower.ctypes.data_as(C.POINTER(C.c_double)),
                               self.upper.ctypes.data_as(C.POINTER(C.c_double)), float(f.param))


class _Config:
    def __init__(self, cfg: EngineConfig):
        self.sp = np.ascontiguousarray(cfg.start_point, dtype=np.float64) if len(cfg.start_point) else None
        self.c = psa_engine_config(
            n_chains=int(cfg.n_chains), start_mode=int(cfg.start_mode),
            start_point=self.sp.ctypes.data_as(C.POINTER(C.c_double)) if self.sp is not None else None,
            start_point_len=0 if self.sp is None else len(self.sp),
            precision=int(cfg.precision), seed=int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, workers=int(cfg.workers),
            schedule=cfg.schedule._c())


class _Result:
    def __init__(self, dim: int, capacity: int):
        self.best_x = np.zeros(dim, dtype=np.float64)
        self.trace = (psa_trace_point * max(1, capacity))()
        self.c = psa_run_result()
        self.c.best_x = self.best_x.ctypes.data_as(C.POINTER(C.c_double))
        self.c.trace = self.trace
        self.c.trace_capacity = capacity

    def to_run_result(self) -> RunResult:
        r = self.c
        n = min(r.trace_len, r.trace_capacity)
        return RunResult(
            best_x=self.best_x.tolist(), best_f=r.best_f, evaluations=r.evaluations,
            wall_time_s=r.wall_time_s,
            trace=[TracePoint(self.trace[i].level, self.trace[i].cumulative_evals, self.trace[i].best_f)
                   for i in range(n)],
            winning_chain=r.winning_chain, rng_draws=r.rng_draws,
            phases=PhaseBreakdown(r.sa_evaluations, r.refine_evaluations, r.sa_best_f) if r.has_phases else None)


def _levels_or_raise(sched: AnnealSchedule) -> int:
    lib = _lib()
    s = sched._c()
    n = C.c_int32()
    st = lib.psa_ladder(C.byref(s), None, 0, C.byref(n))
    return n.value if st == 0 else 1


def _run(fn_name: str, f: ObjectiveFunction, cfg: EngineConfig, extra_trace: int = 0) -> RunResult:
    lib = _lib()
    h = _Objective(f)
    c = _Config(cfg)
    r = _Result(f.dim, _levels_or_raise(cfg.schedule) + extra_trace)
    _raise(lib, getattr(lib, fn_name)(C.byref(h.c), C.byref(c.c), C.byref(r.c)))
    return r.to_run_result()


def run_sequential(f: ObjectiveFunction, cfg: EngineConfig) -> RunResult:
    """engines.cpp:125-129"""
    return _run("psa_run_sequential", f, cfg)


def run_asynchronous(f: ObjectiveFunction, cfg: EngineConfig) -> RunResult:
    """engines.cpp:66-123"""
    return _run("psa_run_asynchronous", f, cfg)


def run_synchronous(f: ObjectiveFunction, cfg: EngineConfig) -> RunResult:
    """engines.cpp:131-207"""
    return _run("psa_run_synchronous", f, cfg)


# ---------------------------------------------------------------------------
# nelder_mead.hpp
# ---------------------------------------------------------------------------

@dataclass
class NelderMeadConfig:
    reflect: float = 1.0
    expand: float = 2.0
    contract: float = 0.5
    shrink: float = 0.5
    f_tol: float = 1e-12
    x_tol: float = 1e-10
    max_iters: int = 0  # 0 => 50000 * n

    def effective_max_iters(self, n: int) -> int:
        return self.max_iters if self.max_iters > 0 else 50000 * n

    def _c(self):
        return psa_nm_config(self.reflect, self.expand, self.contract, self.shrink, self.f_tol, self.x_tol,
                             int(self.max_iters), 0)


@dataclass
class NelderMeadResult:
    x_best: list
    f_best: float
    iterations: int
    evaluations: int


def nelder_mead_minimize(f: ObjectiveFunction, x_start: Sequence[float],
                         cfg: Optional[NelderMeadConfig] = None) -> NelderMeadResult:
    """nelder_mead.cpp:37-115, on the device (one cooperative block)."""
    lib = _lib()
    cfg = cfg or NelderMeadConfig()
    h = _Objective(f)
    x0 = np.ascontiguousarray(x_start, dtype=np.float64)
    if len(x0) != f.dim:
        raise InvalidArgument(f"contains: expected dimension {f.dim}, got {len(x0)}")
    xb = np.zeros(f.dim)
    r = psa_nm_result(xb.ctypes.data_as(C.POINTER(C.c_double)), 0.0, 0, 0, 0)
    c = cfg._c()
    _raise(lib, lib.psa_nelder_mead_minimize(C.byref(h.c), x0.ctypes.data_as(C.POINTER(C.c_double)),
                                             C.byref(c), C.byref(r)))
    return NelderMeadResult(xb.tolist(), r.f_best, r.iterations, r.evaluations)


def nelder_mead_batch(f: ObjectiveFunction, x_starts, cfg: NelderMeadConfig = None) -> list:
    """Many independent nelder_mead_minimize runs on the device, one thread
    each (psa_nelder_mead_batch); each result is bit-identical to the
    reference's run from that start.  x_starts: (count, dim) array-like."""
    cfg = cfg or NelderMeadConfig()
    lib = _lib()
    X = np.ascontiguousarray(np.asarray(x_starts, dtype=np.float64).reshape(-1, f.dim))
    m = X.shape[0]
    xb = np.zeros((m, f.dim))
    fb = np.zeros(m)
    it = np.zeros(m, dtype=np.int32)
    ev = np.zeros(m, dtype=np.uint64)
    h = _Objective(f)
    _raise(lib, lib.psa_nelder_mead_batch(C.byref(h.c), X.ctypes.data_as(C.POINTER(C.c_double)), m,
                                          C.byref(cfg._c()), xb.ctypes.data_as(C.POINTER(C.c_double)),
                                          fb.ctypes.data_as(C.POINTER(C.c_double)),
                                          it.ctypes.data_as(C.POINTER(C.c_int32)),
                                          ev.ctypes.data_as(C.POINTER(C.c_uint64))))
    return [NelderMeadResult(list(xb[i]), float(fb[i]), int(it[i]), int(ev[i])) for i in range(m)]


def hybrid_run(f: ObjectiveFunction, cfg: EngineConfig, truncated_sched: AnnealSchedule,
               nm_cfg: Optional[NelderMeadConfig] = None) -> RunResult:
    """nelder_mead.cpp:117-136: truncated synchronous SA, then the polish."""
    lib = _lib()
    nm_cfg = nm_cfg or NelderMeadConfig()
    h = _Objective(f)
    c = _Config(cfg)
    r = _Result(f.dim, _levels_or_raise(truncated_sched) + 1)
    ts = truncated_sched._c()
    nm = nm_cfg._c()
    _raise(lib, lib.psa_hybrid_run(C.byref(h.c), C.byref(c.c), C.byref(ts), C.byref(nm), C.byref(r.c)))
    return r.to_run_result()


# ---------------------------------------------------------------------------
# device-resident plans (benchmarks, multi-GPU shards)
# ---------------------------------------------------------------------------

class Plan:
    """A device-resident engine run: upload once, launch many times on a
    caller-supplied CUDA stream (`stream` is an int cudaStream_t handle, e.g.
    torch.cuda.current_stream().cuda_stream), fetch the RunResult.

    `rank`/`world` make the plan one shard of a multi-GPU synchronous run
    (chains [chain_begin, chain_end) of the global range); connect the ranks'
    mailboxes with `set_peers` before the first launch (see dist.py)."""

    def __init__(self, f: ObjectiveFunction, cfg: EngineConfig, engine: int = 2,
                 chain_begin: int = 0, chain_end: Optional[int] = None,
                 rank: int = 0, world: int = 1, max_blocks: int = 0):
        self._lib = _lib()
        self._h = _Objective(f)
        self._c = _Config(cfg)
        self.f = f
        self.cfg = cfg
        self.rank, self.world = rank, world
        end = cfg.n_chains if chain_end is None else chain_end
        p = C.c_void_p()
        opt = _abi.psa_plan_options(int(max_blocks), int(rank), int(world), 0)
        _raise(self._lib, self._lib.psa_plan_create_ex(C.byref(self._h.c), C.byref(self._c.c), int(engine),
                                                       int(chain_begin), int(end), C.byref(opt), C.byref(p)))
        self._p = p
        lv, ch, la = C.c_int32(), C.c_int32(), C.c_int32()
        _raise(self._lib, self._lib.psa_plan_info(p, C.byref(lv), C.byref(ch), C.byref(la)))
        self.levels, self.chains, self.launches_per_run = lv.value, ch.value, la.value
        buf = C.create_string_buffer(256)
        _raise(self._lib, self._lib.psa_plan_describe(p, buf, 256))
        self.description = buf.value.decode()
        self._opened = []

    def mailbox(self) -> int:
        ptr = C.c_void_p()
        _raise(self._lib, self._lib.psa_plan_mailbox(self._p, C.byref(ptr), None))
        return ptr.value

    def mailbox_ipc_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        _raise(self._lib, self._lib.psa_plan_mailbox_ipc_handle(self._p, buf))
        return bytes(buf)

    def open_ipc(self, handle: bytes) -> int:
        ptr = C.c_void_p()
        _raise(self._lib, self._lib.psa_ipc_open(C.create_string_buffer(handle, 64), C.byref(ptr)))
        self._opened.append(ptr.value)
        return ptr.value

    def set_peers(self, mailboxes):
        arr = (C.c_void_p * len(mailboxes))(*mailboxes)
        _raise(self._lib, self._lib.psa_plan_set_peers(self._p, arr, len(mailboxes)))

    def launch(self, stream: int = 0):
        _raise(self._lib, self._lib.psa_plan_launch(self._p, C.c_void_p(stream)))

    def fetch(self, stream: int = 0) -> RunResult:
        r = _Result(self.f.dim, self.levels)
        _raise(self._lib, self._lib.psa_plan_fetch(self._p, C.c_void_p(stream), C.byref(r.c)))
        return r.to_run_result()

    def level_detail(self):
        w = np.zeros(self.levels, dtype=np.int32)
        e = np.zeros(self.levels, dtype=np.float64)
        _raise(self._lib, self._lib.psa_plan_level_detail(self._p, w.ctypes.data_as(C.POINTER(C.c_int32)),
                                                          e.ctypes.data_as(C.POINTER(C.c_double)), self.levels))
        return w, e

    def exact_settles(self) -> int:
        """Deferred-fold plans: trials of the last fetched run whose decision
        needed exact folds (psa_plan_stats)."""
        v = C.c_uint64()
        _raise(self._lib, self._lib.psa_plan_stats(self._p, C.byref(v)))
        return v.value

    def close(self, _sync: bool = True):
        # a multi-process shard waits for every rank before it unmaps the
        # peers' mailboxes and frees its own (dist.make_sharded_plan)
        hook = getattr(self, "_before_close", None)
        if _sync and hook is not None and self._p:
            self._before_close = None
            hook()
        for ptr in getattr(self, "_opened", []):
            self._lib.psa_ipc_close(C.c_void_p(ptr))
        self._opened = []
        if self._p:
            self._lib.psa_plan_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close(_sync=False)
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
