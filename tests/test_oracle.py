"""The CPU oracle (oracle/sa_oracle.c) pinned against the reference.

Two anchors: the committed golden fixtures generated from the unmodified
reference (tests/golden/reference_golden.json), and — when oracle/_ref was
built in this container — live side-by-side runs against the reference
library itself.  Mirrors the reference's own identities
(test_rng.cpp, test_sa_core.cpp, test_engines.cpp, acceptance A1/A5/A8/A9).
"""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import (Config, Problem, Result, levels_of_cfg, oracle, oracle_async, oracle_sync, ref,
                        ref_run, same_run)
from paper_2408_00018_b200._abi import FAMILY, psa_schedule


def fx(h):
    return float.fromhex(h)


def test_philox_kats(golden):
    o = oracle()
    for kat in golden["philox_kat"]:
        out = (C.c_uint32 * 4)()
        o.orc_philox4x32_10((C.c_uint32 * 4)(*kat["ctr"]), kat["key"][0], kat["key"][1], out)
        assert list(out) == kat["out"]
    # Random123 published vectors (also the survey's §8c values)
    assert golden["philox_kat"][0]["out"] == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert golden["philox_kat"][1]["out"] == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert golden["philox_kat"][2]["out"] == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_streams(golden):
    o = oracle()
    for s in golden["streams"]:
        u = np.zeros(64)
        o.orc_uniforms(s["seed"], s["chain"], s["level"], 0, 64, u.ctypes.data_as(C.POINTER(C.c_double)))
        assert [v.hex() for v in u] == s["uniforms"]
        assert [o.orc_coordinate_index(v, 100) for v in u] == s["coord_index_n100"]
    # rng.hpp:66-75: draw i is a pure function of (key, i) — skip-ahead equals sequential
    seq = np.zeros(50)
    o.orc_uniforms(77, 3, 9, 0, 50, seq.ctypes.data_as(C.POINTER(C.c_double)))
    tail = np.zeros(10)
    o.orc_uniforms(77, 3, 9, 40, 10, tail.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(seq[40:], tail)


def test_schedules(golden):
    o = oracle()
    for s in golden["schedules"]:
        t0, tmin, rho, n = s["schedule"]
        sc = psa_schedule(t0, tmin, rho, n, 0)
        temps = (C.c_double * 4096)()
        lv = o.orc_ladder(C.byref(sc), temps, 4096)
        assert lv == s["levels"]
        assert temps[lv - 1].hex() == s["last_t"]
        assert o.orc_expected_evaluations(C.byref(sc), s["chains"]) == s["expected_evaluations"]
    # test_sa_core.cpp:27-62 / acceptance A1
    by = {(tuple(s["schedule"]), s["chains"]): s for s in golden["schedules"]}
    assert by[((5, 0.5, 0.7, 5), 768)]["expected_evaluations"] == 27648
    assert by[((5, 0.5, 0.7, 5), 7680000)]["expected_evaluations"] == 276480000
    assert by[((1000, 0.01, 0.99, 100), 16384)]["expected_evaluations"] == 1877622784
    assert by[((1000, 0.01, 0.99, 100), 16384)]["levels"] == 1146
    assert by[((5, 0.5, 0.7, 5), 768)]["levels"] == 7
    assert by[((1, 0.9, 0.5, 1), 1)]["levels"] == 1


def test_evaluate_all_families(golden):
    o = oracle()
    for rec in golden["evaluate"]:
        fam = FAMILY[rec["family"]]
        for row, e64, e32 in zip(rec["x"], rec["f64"], rec["f32"]):
            x = np.array([fx(h) for h in row])
            xp = x.ctypes.data_as(C.POINTER(C.c_double))
            assert o.orc_evaluate(fam, rec["dim"], xp).hex() == e64, rec["family"]
            assert o.orc_evaluate_single(fam, rec["dim"], xp).hex() == e32, rec["family"]


def _run_from_golden(rec):
    prob = Problem(rec["family"], rec["dim"], rec["lo"], rec["hi"])
    cfg = Config(rec["chains"], tuple(rec["schedule"]), rec["seed"], rec["precision"], rec["start_mode"])
    return prob, cfg


def _golden_as_dict(rec):
    return {"best_x": np.array([fx(h) for h in rec["best_x"]]), "best_f": fx(rec["best_f"]),
            "evaluations": rec["evaluations"], "winning_chain": rec["winning_chain"],
            "rng_draws": rec["rng_draws"], "trace_len": len(rec["trace"]),
            "trace": [(a, b, fx(c)) for a, b, c in rec["trace"]]}


@pytest.mark.parametrize("name", [
    "v2_schwefel8_f64", "v2_schwefel8_f32", "v2_schwefel10_random_f64", "v2_schwefel16_f64",
    "v2_schwefel100_f32", "v2_rosenbrock4_f64", "v2_shekel5_random_f32", "v2_ackley30_f64",
    "v2_rastrigin30_f32", "v2_griewank50_f64", "v1_schwefel8_f64", "v1_schwefel30_f32",
    "v1_rastrigin30_f64", "v0_schwefel8_f64"])
def test_runs_bitwise(golden, name):
    rec = golden["runs"][name]
    prob, cfg = _run_from_golden(rec)
    got = oracle_sync(prob, cfg) if rec["engine"] == 2 else oracle_async(prob, cfg)
    assert got["rc"] == 0
    assert same_run(got, _golden_as_dict(rec)) == []


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1_v2_schwefel10_f32"])
def test_c1_bitwise(golden, name):
    """C1 of BASELINE.json (n=10, 1024 chains, 1146 levels): survey §8c golden."""
    rec = golden["runs"][name]
    prob, cfg = _run_from_golden(rec)
    got = oracle_sync(prob, cfg)
    assert same_run(got, _golden_as_dict(rec)) == []


def test_c1_golden_values(golden):
    r64 = golden["runs"]["c1_v2_schwefel10_f64"]
    r32 = golden["runs"]["c1_v2_schwefel10_f32"]
    assert fx(r64["best_f"]) == -418.98288724792656 and r64["winning_chain"] == 764
    assert fx(r32["best_f"]) == -418.98281860351562 and r32["winning_chain"] == 398
    assert r64["evaluations"] == 117351424


def test_draw_accounting_identities(golden):
    """test_engines.cpp:139,175-176 and acceptance A8"""
    for name, rec in golden["runs"].items():
        levels = len(rec["trace"])
        chains, n_steps = rec["chains"], rec["schedule"][3]
        assert rec["evaluations"] == chains * (1 + n_steps * levels)
        extra = chains * rec["dim"] if rec["start_mode"] == 1 else 0
        assert rec["rng_draws"] == 3 * (rec["evaluations"] - chains) + extra
        assert rec["trace"][-1][1] == rec["evaluations"]
        bf = [fx(t[2]) for t in rec["trace"]]
        if rec["engine"] == 2:
            assert all(b <= a for a, b in zip(bf, bf[1:])), name  # A9 monotone trace


def test_reduce_min_semantics():
    o = oracle()
    f = (C.c_double * 3)(3.0, 1.0, 2.0)
    ch = (C.c_int32 * 3)(0, 1, 2)
    assert o.orc_reduce_min(f, ch, 3) == 1
    f = (C.c_double * 3)(5.0, 5.0, 5.0)
    ch = (C.c_int32 * 3)(2, 0, 1)
    assert o.orc_reduce_min(f, ch, 3) == 1  # smallest chain index among ties


needs_ref = pytest.mark.skipif(ref() is None, reason="oracle/_ref not built (no reference tree here)")


@needs_ref
@pytest.mark.parametrize("seed", [11, 12])
def test_oracle_matches_reference_live(seed):
    rng = np.random.default_rng(seed)
    for fam, dim, lo, hi in [("SCHWEFEL", 12, -512, 512), ("LEVY_MONTALVO", 5, -10, 10),
                             ("MICHALEWICZ", 10, 0, np.pi), ("SALOMON", 10, -100, 100),
                             ("SHUBERT", 2, -10, 10), ("COSINE_MIXTURE", 4, -1, 1)]:
        for prec in (0, 1):
            sm = int(rng.integers(0, 2))
            prob = Problem(fam, dim, lo, hi)
            cfg = Config(int(rng.integers(3, 40)), (float(rng.uniform(5, 50)), 0.5, 0.8, int(rng.integers(2, 12))),
                         int(rng.integers(0, 2**40)), prec, sm)
            for engine in (1, 2):
                a = oracle_sync(prob, cfg) if engine == 2 else oracle_async(prob, cfg)
                b = ref_run(engine, prob, cfg)
                assert same_run(a, b) == [], (fam, prec, engine)


@needs_ref
def test_error_messages_match_reference():
    """The product must raise with the reference's messages (checked in
    test_api_cpu.py); here: the reference's own messages as the anchor."""
    prob = Problem("SCHWEFEL", 8, -512, 512, ident="F0_a")
    cfg = Config(2, (5.0, 0.5, 0.7, 10), start_point=[600.0] * 8)
    assert ref_run(2, prob, cfg)["err"] == "infeasible start point for F0_a"
    cfg = Config(0, (5.0, 0.5, 0.7, 10))
    assert ref_run(2, prob, cfg)["err"] == "run_synchronous: need n_chains >= 1"
    assert ref_run(1, prob, cfg)["err"] == "run_asynchronous: need n_chains >= 1"
    cfg = Config(2, (5.0, 6.0, 0.7, 10))
    assert ref_run(2, prob, cfg)["err"] == "schedule: need 0 < t_min < t0"
    cfg = Config(4, (5.0, 0.5, 0.7, 10))
    assert ref_run(0, prob, cfg)["err"] == "run_sequential: requires n_chains == 1"


def _nm_cfg(max_iters=0):
    from paper_2408_00018_b200._abi import psa_nm_config
    return psa_nm_config(1.0, 2.0, 0.5, 0.5, 1e-12, 1e-10, max_iters, 0)


@pytest.mark.parametrize("name", ["nm_sphere4", "nm_rosenbrock4", "nm_shekel5", "nm_schwefel8", "nm_griewank20",
                                  "nm_schwefel64_capped"])
def test_oracle_nelder_mead_bitwise(golden, name):
    from paper_2408_00018_b200._abi import psa_nm_result
    rec = golden["nelder_mead"][name]
    prob = Problem(rec["family"], rec["dim"], rec["lo"], rec["hi"])
    x0 = np.array([fx(h) for h in rec["x0"]])
    xb = np.zeros(rec["dim"])
    r = psa_nm_result(xb.ctypes.data_as(C.POINTER(C.c_double)), 0, 0, 0, 0)
    cfg = _nm_cfg(rec["max_iters"])
    assert oracle().orc_nelder_mead_minimize(C.byref(prob.c), x0.ctypes.data_as(C.POINTER(C.c_double)),
                                            C.byref(cfg), C.byref(r)) == 0
    assert [v.hex() for v in xb] == rec["x_best"]
    assert r.f_best.hex() == rec["f_best"]
    assert (r.iterations, r.evaluations) == (rec["iterations"], rec["evaluations"])


@pytest.mark.parametrize("name", ["hybrid_rosenbrock4", "hybrid_schwefel32", "hybrid_griewank10"])
def test_oracle_hybrid_bitwise(golden, name):
    from paper_2408_00018_b200._abi import psa_schedule
    rec = golden["hybrid"][name]
    prob = Problem(rec["family"], rec["dim"], rec["lo"], rec["hi"])
    cfg = Config(rec["chains"], tuple(rec["schedule"]), rec["seed"], 0, 0)
    ts = psa_schedule(*rec["truncated"], 0)
    L = levels_of_cfg(Config(rec["chains"], tuple(rec["truncated"])))
    res = Result(rec["dim"], L + 2)
    nm = _nm_cfg()
    assert oracle().orc_hybrid_run(C.byref(prob.c), C.byref(cfg.c), C.byref(ts), C.byref(nm), C.byref(res.c)) == 0
    d = res.as_dict()
    assert [v.hex() for v in d["best_x"]] == rec["best_x"]
    assert d["best_f"].hex() == rec["best_f"]
    assert d["evaluations"] == rec["evaluations"] and d["refine_evaluations"] == rec["refine_evaluations"]
    assert [[a, b, c.hex()] for a, b, c in d["trace"]] == rec["trace"]
