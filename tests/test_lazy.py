"""Deferred-fold engine (v2_lazy_kernel, engine.cuh sweep_lazy) against the
reference (GPU tests).

The deferred fold settles a Metropolis decision from an energy interval and
folds the chain's terms only when the interval straddles the threshold, so
its risk is the bound: a radius that is too small gives a wrong decision.
These cases aim at the places where the interval is tight or undecided:

  * very low temperatures (every uphill decision sits near the band),
  * tiny boxes (energy differences of the order of the radius itself, so
    most decisions take the exact path),
  * non-uniform boxes, random starts, f32 and f64, compile-time and runtime n,
    shared-memory and HBM rows,
and compare bit for bit with the C oracle (oracle/sa_oracle.c, pinned to the
reference) and with the fold-every-trial kernels (PSA_LAZY=0).
"""
import numpy as np
import pytest

import paper_2408_00018_b200 as psa
from oracle_lib import Config, Problem, oracle_sync, same_run
from test_gpu_parity import device_run

pytestmark = pytest.mark.gpu

@pytest.fixture(autouse=True, params=["lazy1", "lazypair", "lazypc"])
def _lazy_kernel(request, monkeypatch):
    """these tests pin each deferred-fold kernel: one chain per thread
    (lazy1), chain pairs (lazypair; binary32 only — f64 plans fall back to
    lazy1) and the producer/consumer blocks with the deferred-fold consumer
    (lazypc, the default at small chain counts)"""
    monkeypatch.setenv("PSA_V2_MODE", request.param)
    return request.param


LAZY = [("SCHWEFEL", -512.0, 512.0), ("RASTRIGIN", -5.12, 5.12), ("SPHERE", -2.0, 2.0),
        ("MICHALEWICZ", 0.0, 3.141592653589793)]


def _plan_desc(family, dim, lo, hi, chains, sched, prec):
    f = psa.ObjectiveFunction("lazy", "lazy", dim, psa.BoxDomain([lo] * dim, [hi] * dim), family)
    cfg = psa.EngineConfig(n_chains=chains, schedule=psa.AnnealSchedule(*sched), precision=prec)
    with psa.Plan(f, cfg) as p:
        return p.description


@pytest.mark.parametrize("family,lo,hi", LAZY)
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("dim", [10, 100, 7])
def test_lazy_matches_oracle(gpu_lib, family, lo, hi, prec, dim):
    prob = Problem(family, dim, lo, hi)
    for start, sched in ((0, (50.0, 0.05, 0.7, 40)), (1, (1e-3, 1e-7, 0.25, 64))):
        cfg = Config(517, sched, 5 + start, prec, start)
        got = device_run(2, prob, cfg)
        want = oracle_sync(prob, cfg)
        assert not same_run(got, want), (family, dim, prec, start, same_run(got, want))


def test_lazy_kernel_is_the_default_for_affine_families(gpu_lib, monkeypatch):
    monkeypatch.delenv("PSA_V2_MODE", raising=False)
    d = _plan_desc("SCHWEFEL", 100, -512.0, 512.0, 1 << 16, (1000.0, 989.01, 0.99, 100),
                   psa.Precision.f32)
    assert d.startswith("v2_lazy_kernel"), d


@pytest.mark.parametrize("adapt", ["0", "1"])
@pytest.mark.parametrize("prec", [0, 1])
def test_tiny_box_forces_exact_settles(gpu_lib, monkeypatch, prec, adapt):
    """Energy differences of the order of the radius: most decisions need the
    exact folds, and the result must still be the reference's — with every
    settle taken in the deferred-fold sweep (adapt 0) and with the blocks
    falling back to a fold per trial after the first level (adapt 1)."""
    monkeypatch.setenv("PSA_LAZY_ADAPT", adapt)
    # f32 radius ~ 2^-24 of the energy; f64 ~ the double tracking error
    lo, hi = 1.0, 1.0 + (2.0 ** -18 if prec == 1 else 2.0 ** -44)
    prob = Problem("SPHERE", 30, lo, hi)
    cfg = Config(300, (1e-6, 1e-9, 0.3, 50), 3, prec, 1)
    got = device_run(2, prob, cfg)
    want = oracle_sync(prob, cfg)
    assert not same_run(got, want), same_run(got, want)
    f = psa.ObjectiveFunction("t", "t", 30, psa.BoxDomain([lo] * 30, [hi] * 30), "SPHERE")
    ecfg = psa.EngineConfig(n_chains=300, schedule=psa.AnnealSchedule(1e-6, 1e-9, 0.3, 50), seed=3,
                            precision=psa.Precision(prec), start_mode=psa.StartMode.random_per_chain)
    with psa.Plan(f, ecfg) as p:
        p.launch()
        p.fetch()
        settles = p.exact_settles()
    assert settles > 0


def test_nonuniform_box_matches_oracle(gpu_lib):
    rng = np.random.default_rng(7)
    dim = 40
    lo = -rng.uniform(1, 600, dim)
    hi = rng.uniform(1, 600, dim)
    prob = Problem("SCHWEFEL", dim, lo, hi)
    for prec in (0, 1):
        cfg = Config(1000, (300.0, 0.01, 0.8, 60), 9, prec, 1)
        got = device_run(2, prob, cfg)
        want = oracle_sync(prob, cfg)
        assert not same_run(got, want), (prec, same_run(got, want))


@pytest.mark.parametrize("prec", [0, 1])
def test_lazy_equals_fold_every_trial_at_scale(gpu_lib, monkeypatch, prec):
    """65536 chains, n = 100, 40 levels of the paper ladder's tail (the low
    temperatures where the interval is tightest): bitwise equal to the
    fold-every-trial kernel."""
    prob = Problem("SCHWEFEL", 100, -512.0, 512.0)
    cfg = Config(1 << 16, (0.5, 0.01, 0.9, 100), 21, prec, 1)
    monkeypatch.delenv("PSA_LAZY", raising=False)
    monkeypatch.delenv("PSA_V2_MODE", raising=False)
    lazy = device_run(2, prob, cfg)
    monkeypatch.setenv("PSA_LAZY", "0")
    full = device_run(2, prob, cfg)
    assert not same_run(lazy, full), same_run(lazy, full)


@pytest.mark.parametrize("prec", [0, 1])
def test_lazy_hbm_rows_match_oracle(gpu_lib, monkeypatch, prec):
    monkeypatch.setenv("PSA_FORCE_HBM_ROWS", "1")
    prob = Problem("RASTRIGIN", 45, -5.12, 5.12)
    cfg = Config(700, (20.0, 0.01, 0.75, 70), 4, prec, 1)
    got = device_run(2, prob, cfg)
    want = oracle_sync(prob, cfg)
    assert not same_run(got, want), same_run(got, want)


@pytest.mark.parametrize("prec", [0, 1])
def test_metropolis_pretest_never_contradicts_the_exact_test(gpu_lib, prec):
    """2^30 acceptance draws placed within 2^-40..2^-6 (relative) of the
    decision boundary -T ln(u), T in 2^-10..2^10: every decision the band
    pre-test calls certain equals the glibc-exact test (sa_core.cpp:46-55)."""
    import ctypes as C
    out = (C.c_uint64 * 3)()
    rc = gpu_lib.psa_device_metropolis_check(prec, 12345 + prec, 1 << 30, out)
    assert rc == 0, gpu_lib.psa_last_error().decode()
    certain, wrong, undecided = out
    assert certain + undecided == 1 << 30
    assert wrong == 0, (certain, wrong, undecided)
    assert certain > (1 << 30) // 8  # the draws away from the boundary are settled by the band


@pytest.mark.parametrize("prec", [0, 1])
def test_large_n_lazy_hbm_rows_match_oracle(gpu_lib, _lazy_kernel, prec):
    """n = 500 (C4's SA phase): the deferred fold keeps its rows in HBM
    (shared-memory rows would leave 3 warps per SM)."""
    if _lazy_kernel == "lazypc":
        pytest.skip("the producer/consumer kernel keeps its 32 rows in shared memory")
    prob = Problem("SCHWEFEL", 500, -512.0, 512.0)
    sched = (1000.0, 100.0, 0.5, 100)  # warm: binary32 keeps HBM rows only above rr * n
    cfg = Config(64, sched, 8, prec, 1)
    desc = _plan_desc("SCHWEFEL", 500, -512.0, 512.0, 64, sched, psa.Precision(prec))
    assert desc.startswith("v2_lazy_kernel (deferred fold, HBM SoA rows)"), desc
    got = device_run(2, prob, cfg)
    want = oracle_sync(prob, cfg)
    assert not same_run(got, want), same_run(got, want)


@pytest.mark.parametrize("prec", [0, 1])
def test_large_n_lazy_equals_fold_every_trial(gpu_lib, monkeypatch, prec):
    """n = 500 at 40000 chains over the C4 schedule's first and a low-T
    window: HBM-row deferred fold == fold-every-trial kernel, bitwise."""
    monkeypatch.delenv("PSA_V2_MODE", raising=False)
    prob = Problem("SCHWEFEL", 500, -512.0, 512.0)
    for sched in ((1000.0, 700.0, 0.9, 100), (0.5, 0.2, 0.8, 100)):
        cfg = Config(40000, sched, 13, prec, 1)
        lazy = device_run(2, prob, cfg)
        monkeypatch.setenv("PSA_LAZY", "0")
        full = device_run(2, prob, cfg)
        monkeypatch.delenv("PSA_LAZY")
        assert not same_run(lazy, full), (sched, same_run(lazy, full))


@pytest.mark.parametrize("family,lo,hi", LAZY)
@pytest.mark.parametrize("prec", [0, 1])
def test_v1_and_v0_lazy_consumer_match_oracle(gpu_lib, monkeypatch, family, lo, hi, prec):
    """The asynchronous engine's producer/consumer kernel with the deferred-
    fold consumer (v1_lazy_pc_kernel): level-end energies are exact folds
    (engines.cpp:90-106), every decision the reference's.  Also V0
    (run_sequential = one chain, engines.cpp:125-129)."""
    monkeypatch.setenv("PSA_V2_MODE", "lazypc")
    from oracle_lib import oracle_async
    prob = Problem(family, 30, lo, hi)
    for engine, chains, start in ((1, 333, 1), (1, 64, 0), (0, 1, 0)):
        cfg = Config(chains, (20.0, 0.002, 0.6, 50), 17, prec, start)
        got = device_run(engine, prob, cfg)
        want = oracle_async(prob, cfg)
        assert not same_run(got, want), (engine, chains, same_run(got, want))


@pytest.mark.parametrize("family,lo,hi", LAZY)
@pytest.mark.parametrize("prec", [0, 1])
def test_v0_latency_kernel_matches_oracle(gpu_lib, monkeypatch, family, lo, hi, prec):
    """run_sequential (engines.cpp:125-129) on the V0 latency kernel: the
    chain in one warp's registers, every decision the reference's, level-end
    energies exact folds; n = 1 / 10 / 32, shared and random starts, a
    non-uniform box and temperatures low enough to settle."""
    monkeypatch.delenv("PSA_V2_MODE", raising=False)
    from oracle_lib import oracle_async
    rng = np.random.default_rng(5)
    for dim, start, sched in ((10, 0, (20.0, 0.002, 0.8, 64)), (32, 1, (1e-3, 1e-7, 0.3, 100)), (1, 1, (5.0, 0.5, 0.5, 10))):
        lo_v = np.full(dim, lo) - rng.uniform(0, 0.1, dim) * (hi - lo) * (start == 1)
        prob = Problem(family, dim, lo_v, hi)
        cfg = Config(1, sched, 23 + dim, prec, start)
        got = device_run(0, prob, cfg)
        want = oracle_async(prob, cfg)
        assert not same_run(got, want), (dim, start, same_run(got, want))
    f = psa.ObjectiveFunction("v0", "v0", 10, psa.BoxDomain([lo] * 10, [hi] * 10), family)
    with psa.Plan(f, psa.EngineConfig(n_chains=1, schedule=psa.AnnealSchedule(5.0, 0.5, 0.5, 10)), engine=1) as p:
        assert p.description.startswith("v0_kernel"), p.description
