"""Host-side behaviour of the drop-in API (CPU, no device): schedule, ladder,
budgets, reduce_min, registry and the reference's error messages.  Mirrors
test_sa_core.cpp:27-62, test_engines.cpp:39-68,180-190, test_objectives.cpp:25-60."""
import ctypes as C

import numpy as np
import pytest

import paper_2408_00018_b200 as psa
from oracle_lib import oracle
from paper_2408_00018_b200._abi import psa_schedule


def test_ladder_follows_the_do_while_loop():
    info = psa.ladder(psa.AnnealSchedule(5, 0.5, 0.7, 5))
    assert info.levels == 7
    assert info.temperatures[0] == 5.0
    assert abs(info.temperatures[-1] - 0.588245) < 1e-6
    assert all(b < a for a, b in zip(info.temperatures, info.temperatures[1:]))
    assert info.temperatures[-1] > 0.5 and info.temperatures[-1] * 0.7 <= 0.5
    assert psa.ladder(psa.AnnealSchedule(1000, 0.01, 0.99, 100)).levels == 1146
    assert psa.ladder(psa.AnnealSchedule(1, 0.9, 0.5, 1)).levels == 1
    # bitwise equal to the oracle's ladder
    for s in [(1000, 0.01, 0.99, 100), (1000, 32, 0.9, 100), (3.7, 1e-3, 0.937, 3)]:
        t = psa.ladder(psa.AnnealSchedule(*s)).temperatures
        buf = (C.c_double * 4096)()
        n = oracle().orc_ladder(C.byref(psa_schedule(*s, 0)), buf, 4096)
        assert t == list(buf[:n])


@pytest.mark.parametrize("bad,msg", [((1, 2, 0.5, 1), "schedule: need 0 < t_min < t0"),
                                     ((1, 0.5, 1.5, 1), "schedule: need rho in (0,1)"),
                                     ((1, 0.5, 0.9, 0), "schedule: need sweep_length >= 1"),
                                     ((-1, 0.5, 0.9, 1), "schedule: need 0 < t_min < t0"),
                                     ((1, 0.5, float("nan"), 1), "schedule: need rho in (0,1)")])
def test_invalid_schedules(bad, msg):
    with pytest.raises(psa.InvalidArgument, match=msg.replace("(", r"\(").replace(")", r"\)")):
        psa.ladder(psa.AnnealSchedule(*bad))


def test_budgets():
    small = psa.AnnealSchedule(5, 0.5, 0.7, 5)
    assert psa.expected_evaluations(small, 768) == 27648
    assert psa.expected_evaluations(small, 76800) == 2_764_800
    assert psa.expected_evaluations(small, 7_680_000) == 276_480_000
    large = psa.AnnealSchedule(1000, 0.01, 0.99, 100)
    assert psa.expected_evaluations(large, 16384) == 1_877_622_784
    assert psa.expected_evaluations(large, 1 << 20) == 120_167_858_176  # C2
    with pytest.raises(psa.InvalidArgument, match="need n_chains >= 1"):
        psa.expected_evaluations(large, 0)


def test_reduce_min_tie_break_and_grouping():
    Cd = psa.Candidate
    cands = [Cd([1.0], 3.0, 0), Cd([2.0], 1.0, 1), Cd([3.0], 2.0, 2)]
    assert psa.reduce_min(cands).chain_index == 1
    ties = [Cd([1.0], 5.0, 2), Cd([2.0], 5.0, 0), Cd([3.0], 5.0, 1)]
    assert psa.reduce_min(ties).chain_index == 0
    perm = [cands[2], cands[0], cands[1]]
    assert psa.reduce_min(perm).chain_index == psa.reduce_min(cands).chain_index
    with pytest.raises(psa.InvalidArgument, match="reduce_min: empty candidate list"):
        psa.reduce_min([])
    vals = [4.0, 2.0, 7.0, 2.0, 9.0, 2.0, 5.0]
    cs = [Cd([float(i)], v, i) for i, v in enumerate(vals)]
    whole = psa.reduce_min(cs)
    for split in range(1, len(cs) - 1):
        grouped = [psa.reduce_min(cs[:split]), psa.reduce_min(cs[split:])]
        assert psa.reduce_min(grouped).chain_index == whole.chain_index
    # -0.0 == +0.0 ties go to the smaller chain
    z = [Cd([0.0], 0.0, 3), Cd([0.0], -0.0, 1)]
    assert psa.reduce_min(z).chain_index == 1


def test_registry():
    ids = [f.id for f in psa.registry()]
    assert len(ids) == 41 and len(set(ids)) == 41
    s = psa.registry_get("F0_a")
    assert s.dim == 8 and s.domain.lower == [-512.0] * 8 and s.domain.upper == [512.0] * 8
    assert abs(s.reference.f_star - (-418.982887)) < 1e-9
    b = psa.registry_get("F2")
    assert b.dim == 2 and b.domain.lower[0] == -20.0 and len(b.reference.minimizers) == 3
    sh = psa.registry_get("F18_a")
    assert sh.dim == 4 and sh.reference.minimizers == [[4.0, 4.0, 4.0, 4.0]]
    with pytest.raises(psa.OutOfRange) as e:
        psa.registry_get("F20")
    assert "F0_a" in str(e.value) and "F19_b" in str(e.value)
    f100 = psa.registry_get("F0_a").with_dim(100)
    assert f100.dim == 100 and f100.domain.lower == [-512.0] * 100


def test_contains_and_location_error():
    d = psa.BoxDomain([-512.0] * 8, [512.0] * 8)
    assert psa.contains(d, [0.0] * 8)
    assert not psa.contains(d, [513.0] + [0.0] * 7)
    assert psa.contains(psa.BoxDomain([0.0] * 4, [10.0] * 4), [0, 10, 0, 10])
    with pytest.raises(psa.InvalidArgument, match="contains: expected dimension 8, got 3"):
        psa.contains(d, [0.0] * 3)
    f = psa.registry_get("F0_a")
    assert psa.location_error(f, [420.968746] * 8) == 0.0
    with pytest.raises(psa.InvalidArgument, match="exact minimizer unknown for F12_a"):
        psa.location_error(psa.registry_get("F12_a"), [1.0, 1.0])


def test_engine_argument_errors_precede_device_checks():
    """Validation order and messages of engines.cpp:131-140 / :125-127, and
    rejection of descriptors without a device twin (no CPU fallback)."""
    f = psa.registry_get("F0_a")
    base = psa.AnnealSchedule(5.0, 0.5, 0.7, 10)
    with pytest.raises(psa.InvalidArgument, match="infeasible start point for F0_a"):
        psa.run_synchronous(f, psa.EngineConfig(n_chains=2, schedule=base, start_point=[600.0] * 8))
    with pytest.raises(psa.InvalidArgument, match="infeasible start point for F0_a"):
        psa.run_asynchronous(f, psa.EngineConfig(n_chains=2, schedule=base, start_point=[600.0] * 8))
    with pytest.raises(psa.InvalidArgument, match="run_synchronous: need n_chains >= 1"):
        psa.run_synchronous(f, psa.EngineConfig(n_chains=0, schedule=base))
    with pytest.raises(psa.InvalidArgument, match="run_asynchronous: need n_chains >= 1"):
        psa.run_asynchronous(f, psa.EngineConfig(n_chains=0, schedule=base))
    with pytest.raises(psa.InvalidArgument, match="run_sequential: requires n_chains == 1"):
        psa.run_sequential(f, psa.EngineConfig(n_chains=4, schedule=base))
    with pytest.raises(psa.InvalidArgument, match="schedule: need 0 < t_min < t0"):
        psa.run_synchronous(f, psa.EngineConfig(n_chains=4, schedule=psa.AnnealSchedule(1, 2, 0.5, 1)))
    custom = psa.ObjectiveFunction("lambda", "user lambda", 1, psa.BoxDomain([-1.0], [1.0]), "HOST_LAMBDA")
    with pytest.raises(psa.InvalidArgument, match="no device implementation"):
        psa.run_synchronous(custom, psa.EngineConfig(n_chains=1, schedule=base))
