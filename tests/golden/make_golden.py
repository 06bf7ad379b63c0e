"""Generate tests/golden/*.json from the UNMODIFIED reference.

Runs oracle/_ref/libparsa_ref.so (the reference's own sources compiled by
oracle/Makefile) and records bit patterns (hex floats) so every parity test
can compare exactly.  Regenerate with:

    make -C oracle && python tests/golden/make_golden.py

The reference tree is only needed here, at generation time; the fixtures
are committed and travel to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Config, Problem, Result, levels_of_cfg, ref  # noqa: E402

from paper_2408_00018_b200 import _abi  # noqa: E402


def hx(v: float) -> str:
    return float(v).hex()


def run_ref(engine, prob, cfg):
    L = levels_of_cfg(cfg)
    res = Result(prob.dim, L + 1)
    rc = ref().ref_run(engine, C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
    assert rc == 0, ref().ref_last_error()
    d = res.as_dict()
    return {
        "best_x": [hx(v) for v in d["best_x"]],
        "best_f": hx(d["best_f"]),
        "evaluations": d["evaluations"],
        "winning_chain": d["winning_chain"],
        "rng_draws": d["rng_draws"],
        "trace": [[lv, ce, hx(bf)] for lv, ce, bf in d["trace"]],
    }


# (name, engine, family, dim, lo, hi, chains, schedule, seed, precision, start_mode)
RUNS = [
    ("v2_schwefel8_f64", 2, "SCHWEFEL", 8, -512, 512, 32, (5.0, 0.5, 0.7, 10), 3, 0, 0),
    ("v2_schwefel8_f32", 2, "SCHWEFEL", 8, -512, 512, 32, (5.0, 0.5, 0.7, 10), 3, 1, 0),
    ("v2_schwefel10_random_f64", 2, "SCHWEFEL", 10, -512, 512, 64, (1000, 0.01, 0.9, 20), 0, 0, 1),
    ("v2_schwefel16_f64", 2, "SCHWEFEL", 16, -512, 512, 512, (100, 0.01, 0.95, 30), 1, 0, 0),
    ("v2_schwefel100_f32", 2, "SCHWEFEL", 100, -512, 512, 256, (1000, 0.01, 0.9, 100), 0, 1, 0),
    ("v2_rosenbrock4_f64", 2, "ROSENBROCK", 4, -2.048, 2.048, 64, (10, 0.1, 0.9, 20), 1, 0, 0),
    ("v2_shekel5_random_f32", 2, "SHEKEL5", 4, 0, 10, 16, (10, 0.1, 0.8, 10), 5, 1, 1),
    ("v2_ackley30_f64", 2, "ACKLEY", 30, -30, 30, 128, (100, 0.1, 0.9, 20), 2, 0, 1),
    ("v2_rastrigin30_f32", 2, "RASTRIGIN", 30, -5.12, 5.12, 128, (100, 0.1, 0.9, 20), 4, 1, 1),
    ("v2_griewank50_f64", 2, "GRIEWANK", 50, -600, 600, 64, (1000, 1.0, 0.9, 20), 0, 0, 1),
    ("v1_schwefel8_f64", 1, "SCHWEFEL", 8, -512, 512, 32, (5.0, 0.5, 0.7, 10), 3, 0, 0),
    ("v1_schwefel30_f32", 1, "SCHWEFEL", 30, -512, 512, 256, (100, 0.01, 0.95, 20), 7, 1, 1),
    ("v1_rastrigin30_f64", 1, "RASTRIGIN", 30, -5.12, 5.12, 128, (100, 0.1, 0.9, 20), 4, 0, 1),
    ("v0_schwefel8_f64", 0, "SCHWEFEL", 8, -512, 512, 1, (5.0, 0.5, 0.7, 10), 42, 0, 0),
]

# the C1 configuration of BASELINE.json (survey §8c golden values)
C1_RUNS = [
    ("c1_v2_schwefel10_f64", 2, "SCHWEFEL", 10, -512, 512, 1024, (1000, 0.01, 0.99, 100), 0, 0, 0),
    ("c1_v2_schwefel10_f32", 2, "SCHWEFEL", 10, -512, 512, 1024, (1000, 0.01, 0.99, 100), 0, 1, 0),
]


def main():
    lib = ref()
    if lib is None:
        raise SystemExit("oracle/_ref/libparsa_ref.so missing: run `make -C oracle` (needs /root/reference)")
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference sources, unmodified)"}

    # Philox KATs (Random123 vectors) and stream draws
    kat_inputs = [([0, 0, 0, 0], [0, 0]),
                  ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
                  ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0])]
    kats = []
    for ctr, key in kat_inputs:
        o = (C.c_uint32 * 4)()
        lib.ref_philox4x32_10((C.c_uint32 * 4)(*ctr), key[0], key[1], o)
        kats.append({"ctr": ctr, "key": key, "out": list(o)})
    out["philox_kat"] = kats
    streams = []
    for seed, chain, level in [(0, 0, 0), (42, 7, 3), (2**63 + 12345, 4000000000, 77), (1, 2**20 - 1, 1145)]:
        u = (C.c_double * 64)()
        lib.ref_uniforms(seed, chain, level, 64, u)
        idx = (C.c_int32 * 64)()
        lib.ref_coordinate_indices(seed, chain, level, 100, 64, idx)
        streams.append({"seed": seed, "chain": chain, "level": level, "uniforms": [hx(v) for v in u],
                        "coord_index_n100": list(idx)})
    out["streams"] = streams

    # schedule identities (sa_core.cpp:17-35; test_sa_core.cpp:27-62)
    sched = []
    for t0, tmin, rho, n, chains in [(5, 0.5, 0.7, 5, 768), (5, 0.5, 0.7, 5, 76800), (5, 0.5, 0.7, 5, 7680000),
                                     (1000, 0.01, 0.99, 100, 16384), (1000, 0.01, 0.99, 100, 1024),
                                     (1000, 0.01, 0.99, 100, 2**20), (1, 0.9, 0.5, 1, 1),
                                     (1000, 32, 0.9, 100, 16384), (1000, 1, 0.9, 20, 512)]:
        s = _abi.psa_schedule(t0, tmin, rho, n, 0)
        lv = C.c_int32()
        temps = (C.c_double * 4096)()
        assert lib.ref_ladder(C.byref(s), temps, 4096, C.byref(lv)) == 0
        ev = C.c_uint64()
        assert lib.ref_expected_evaluations(C.byref(s), chains, C.byref(ev)) == 0
        sched.append({"schedule": [t0, tmin, rho, n], "chains": chains, "levels": lv.value,
                      "expected_evaluations": ev.value, "last_t": hx(temps[lv.value - 1]),
                      "temps_head": [hx(temps[i]) for i in range(min(5, lv.value))]})
    out["schedules"] = sched

    # cost functions at seeded points, both precisions, every family
    rng = np.random.default_rng(20240800)
    evals = []
    dims = {"SCHWEFEL": 10, "ACKLEY": 30, "COSINE_MIXTURE": 4, "EXPONENTIAL": 4, "GRIEWANK": 50,
            "MICHALEWICZ": 10, "RASTRIGIN": 30, "SALOMON": 10, "SHUBERT": 2, "SPHERE": 6, "BRANIN": 2,
            "DEKKERS_AARTS": 2, "EASOM": 2, "GOLDSTEIN_PRICE": 2, "HIMMELBLAU": 2, "LEVY_MONTALVO": 5,
            "MOD_LANGERMAN": 5, "ROSENBROCK": 4, "SIX_HUMP_CAMEL": 2, "SHEKEL5": 4, "SHEKEL7": 4,
            "SHEKEL10": 4, "SHEKEL_FOXHOLES": 5}
    boxes = {"SCHWEFEL": (-512, 512), "ACKLEY": (-30, 30), "COSINE_MIXTURE": (-1, 1), "EXPONENTIAL": (-1, 1),
             "GRIEWANK": (-600, 600), "MICHALEWICZ": (0, np.pi), "RASTRIGIN": (-5.12, 5.12),
             "SALOMON": (-100, 100), "SHUBERT": (-10, 10), "SPHERE": (-10, 10), "BRANIN": (-20, 20),
             "DEKKERS_AARTS": (-20, 20), "EASOM": (-10, 10), "GOLDSTEIN_PRICE": (-2, 2), "HIMMELBLAU": (-6, 6),
             "LEVY_MONTALVO": (-10, 10), "MOD_LANGERMAN": (0, 10), "ROSENBROCK": (-2.048, 2.048),
             "SIX_HUMP_CAMEL": (-3, 3), "SHEKEL5": (0, 10), "SHEKEL7": (0, 10), "SHEKEL10": (0, 10),
             "SHEKEL_FOXHOLES": (-5, 15)}
    for fam in _abi.FAMILIES:
        n = dims[fam]
        lo, hi = boxes[fam]
        pts = rng.uniform(lo, hi, size=(16, n))
        pts[0] = 0.5 * (lo + hi)  # box centre
        prob = Problem(fam, n, lo, hi)
        rec = {"family": fam, "dim": n, "lo": lo, "hi": hi, "x": [[hx(v) for v in row] for row in pts]}
        for prec, key in ((0, "f64"), (1, "f32")):
            o = np.zeros(len(pts))
            assert lib.ref_evaluate(C.byref(prob.c), prec, pts.ctypes.data_as(C.POINTER(C.c_double)), len(pts),
                                    o.ctypes.data_as(C.POINTER(C.c_double))) == 0
            rec[key] = [hx(v) for v in o]
        evals.append(rec)
    out["evaluate"] = evals

    runs = {}
    for name, engine, fam, dim, lo, hi, chains, sch, seed, prec, sm in RUNS + C1_RUNS:
        prob = Problem(fam, dim, lo, hi, ident=name)
        cfg = Config(chains, sch, seed, prec, sm, workers=0)
        rec = {"engine": engine, "family": fam, "dim": dim, "lo": lo, "hi": hi, "chains": chains,
               "schedule": list(sch), "seed": seed, "precision": prec, "start_mode": sm}
        rec.update(run_ref(engine, prob, cfg))
        runs[name] = rec
        print(name, rec["best_f"], rec["winning_chain"], flush=True)
    out["runs"] = runs

    # Nelder-Mead and hybrid (nelder_mead.cpp), default NelderMeadConfig
    nm_default = (1.0, 2.0, 0.5, 0.5, 1e-12, 1e-10, 0)
    nms = {}
    for name, fam, dim, lo, hi, x0, iters in [
            ("nm_sphere4", "SPHERE", 4, -2.048, 2.048, [1, 1, 1, 1], 0),
            ("nm_rosenbrock4", "ROSENBROCK", 4, -2.048, 2.048, [0.5, 0.3, 0.1, 0.0], 0),
            ("nm_shekel5", "SHEKEL5", 4, 0, 10, [4, 4, 4, 4], 0),
            ("nm_schwefel8", "SCHWEFEL", 8, -512, 512, [400.0, 430.0, 415.0, 425.0, 410.0, 421.0, 419.0, 423.0], 0),
            ("nm_griewank20", "GRIEWANK", 20, -600, 600, [3.0 * (k % 5 - 2) for k in range(20)], 2000),
            ("nm_schwefel64_capped", "SCHWEFEL", 64, -512, 512, [420.0 + (k % 7) for k in range(64)], 3000)]:
        prob = Problem(fam, dim, lo, hi)
        x0a = np.array(x0, dtype=np.float64)
        nmc = _abi.psa_nm_config(*nm_default[:6], iters, 0)
        xb = np.zeros(dim)
        r = _abi.psa_nm_result(xb.ctypes.data_as(C.POINTER(C.c_double)), 0, 0, 0, 0)
        assert lib.ref_nelder_mead(C.byref(prob.c), x0a.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nmc), C.byref(r)) == 0
        nms[name] = {"family": fam, "dim": dim, "lo": lo, "hi": hi, "x0": [hx(v) for v in x0a], "max_iters": iters,
                     "x_best": [hx(v) for v in xb], "f_best": hx(r.f_best), "iterations": r.iterations,
                     "evaluations": r.evaluations}
        print(name, r.f_best, r.iterations, flush=True)
    out["nelder_mead"] = nms
    hyb = {}
    for name, fam, dim, lo, hi, chains, sch, trunc, seed in [
            ("hybrid_rosenbrock4", "ROSENBROCK", 4, -2.048, 2.048, 64, (10, 1, 0.8, 10), (10, 0.5, 0.8, 10), 0),
            ("hybrid_schwefel32", "SCHWEFEL", 32, -512, 512, 512, (100, 1, 0.9, 20), (100.0, 1.0, 0.9, 20), 1),
            ("hybrid_griewank10", "GRIEWANK", 10, -600, 600, 256, (1000, 1, 0.9, 20), (1000.0, 1.0, 0.9, 20), 2)]:
        prob = Problem(fam, dim, lo, hi)
        cfg = Config(chains, sch, seed, 0, 0, workers=0)
        ts = _abi.psa_schedule(*trunc, 0)
        nmc = _abi.psa_nm_config(*nm_default[:6], 0, 0)
        L = levels_of_cfg(Config(chains, trunc))
        res = Result(dim, L + 2)
        assert lib.ref_hybrid_run(C.byref(prob.c), C.byref(cfg.c), C.byref(ts), C.byref(nmc), C.byref(res.c)) == 0
        d = res.as_dict()
        hyb[name] = {"family": fam, "dim": dim, "lo": lo, "hi": hi, "chains": chains, "schedule": list(sch),
                     "truncated": list(trunc), "seed": seed, "best_x": [hx(v) for v in d["best_x"]],
                     "best_f": hx(d["best_f"]), "evaluations": d["evaluations"], "winning_chain": d["winning_chain"],
                     "rng_draws": d["rng_draws"], "trace": [[a, b, hx(c)] for a, b, c in d["trace"]],
                     "sa_evaluations": d["sa_evaluations"], "refine_evaluations": d["refine_evaluations"],
                     "sa_best_f": hx(d["sa_best_f"])}
        print(name, d["best_f"], d["refine_evaluations"], flush=True)
    out["hybrid"] = hyb

    with open(os.path.join(HERE, "reference_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
