"""Parity AT the benchmark configurations (GPU tests).

tests/golden/bench_golden.json holds the UNMODIFIED reference's results
(oracle/_ref, tests/golden/make_bench_golden.py) at BASELINE.json's
configurations themselves, so the kernels the bench times are pinned at the
sizes it times them:

  C2  2^20 chains, Schwefel n=100, first 2 levels of the paper ladder,
      through the chain-pair kernel the bench launches (default plan choice)
      AND the one-chain kernel (PSA_V2_MODE=single)   — engines.cpp:131-207
  C3  16384 chains x 1146 levels, n=30, V1 and V2, Schwefel / Ackley /
      Rastrigin, f32 and f64                          — engines.cpp:66-207
  C4  hybrid at Table-8 scale: 16384 chains, n=500, 33 levels, then
      Nelder-Mead capped at 20000 iterations        — nelder_mead.cpp:117-136

Everything is compared bit for bit: best_x, best_f, winning chain,
evaluations, rng draws and every trace row.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle_lib import Config, Problem, Result, levels_of
from paper_2408_00018_b200 import _abi

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bench_golden.json")
SUITE = {"SCHWEFEL": (-512.0, 512.0, "F0_a"), "ACKLEY": (-30.0, 30.0, "F1"), "RASTRIGIN": (-5.12, 5.12, "F13")}


@pytest.fixture(scope="module")
def bench_golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def as_golden(d):
    return {"best_x": [float(v).hex() for v in d["best_x"]], "best_f": float(d["best_f"]).hex(),
            "winning_chain": d["winning_chain"], "evaluations": d["evaluations"], "rng_draws": d["rng_draws"],
            "trace": [[a, b, float(c).hex()] for a, b, c in d["trace"]]}


def assert_same(got, rec, what):
    for k in ("best_f", "winning_chain", "evaluations", "rng_draws"):
        assert got[k] == rec[k], (what, k, got[k], rec[k])
    assert got["best_x"] == rec["best_x"], (what, "best_x")
    assert got["trace"] == [list(t) for t in rec["trace"]], (what, "trace")


def device(gpu_lib, engine, family, dim, chains, sched, prec):
    lo, hi, ident = SUITE[family]
    prob = Problem(family, dim, lo, hi, ident=ident)
    cfg = Config(chains, tuple(sched), 0, prec, 0)
    res = Result(dim, levels_of(tuple(sched)) + 1)
    fn = gpu_lib.psa_run_synchronous if engine == 2 else gpu_lib.psa_run_asynchronous
    rc = fn(C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
    assert rc == 0, gpu_lib.psa_last_error().decode()
    return as_golden(res.as_dict())


@pytest.mark.parametrize("mode", ["", "single", "pair", "lazy1"])
@pytest.mark.parametrize("key", ["f32", "f64"])
def test_c2_full_chain_count_bitwise_vs_reference(gpu_lib, bench_golden, monkeypatch, key, mode):
    rec = bench_golden[f"c2_{key}"]
    if mode:
        monkeypatch.setenv("PSA_V2_MODE", mode)
    else:
        monkeypatch.delenv("PSA_V2_MODE", raising=False)
    got = device(gpu_lib, 2, "SCHWEFEL", rec["dim"], rec["chains"], rec["schedule"], 1 if key == "f32" else 0)
    assert_same(got, rec, f"c2 {key} {mode or 'default'}")


def test_c2_bench_kernel_is_the_lazy_kernel(gpu_lib):
    """The default plan at C2 (f32) is the deferred-fold kernel — the one the
    test above pins at full size (mode "single" pins the fold-every-trial
    kernel)."""
    import paper_2408_00018_b200 as psa
    f = psa.registry_get("F0_a").with_dim(100)
    cfg = psa.EngineConfig(n_chains=1 << 20, schedule=psa.AnnealSchedule(1000.0, 989.01, 0.99, 100),
                           precision=psa.Precision.f32)
    with psa.Plan(f, cfg) as p:
        assert p.description.startswith("v2_lazy_kernel"), p.description


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("family", ["SCHWEFEL", "ACKLEY", "RASTRIGIN"])
@pytest.mark.parametrize("key", ["f32", "f64"])
def test_c3_full_size_bitwise_vs_reference(gpu_lib, bench_golden, engine, family, key):
    name = f"c3_{family.lower()}_v{engine}_{key}"
    if name not in bench_golden:
        pytest.fail(f"golden {name} missing: run tests/golden/make_bench_golden.py c3")
    rec = bench_golden[name]
    got = device(gpu_lib, engine, family, rec["dim"], rec["chains"], rec["schedule"], 1 if key == "f32" else 0)
    assert_same(got, rec, name)


@pytest.mark.parametrize("key", ["f64", "f32"])
def test_c4_hybrid_table8_scale_bitwise_vs_reference(gpu_lib, bench_golden, key):
    rec = bench_golden[f"c4_{key}"]
    dim = rec["dim"]
    prob = Problem("SCHWEFEL", dim, -512.0, 512.0, ident="F0_a")
    cfg = Config(rec["chains"], tuple(rec["schedule"]), 0, 1 if key == "f32" else 0, 0)
    ts = _abi.psa_schedule(*rec["truncated"], 0)
    nm = _abi.psa_nm_config(1.0, 2.0, 0.5, 0.5, 1e-12, 1e-10, rec["nm_max_iters"], 0)
    res = Result(dim, levels_of(tuple(rec["truncated"])) + 2)
    rc = gpu_lib.psa_hybrid_run(C.byref(prob.c), C.byref(cfg.c), C.byref(ts), C.byref(nm), C.byref(res.c))
    assert rc == 0, gpu_lib.psa_last_error().decode()
    d = res.as_dict()
    got = as_golden(d)
    assert_same(got, rec, f"c4 {key}")
    assert d["sa_evaluations"] == rec["sa_evaluations"] and d["refine_evaluations"] == rec["refine_evaluations"]
    assert float(d["sa_best_f"]).hex() == rec["sa_best_f"]
    assert np.isfinite(d["best_f"])
