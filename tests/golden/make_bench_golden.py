"""Goldens at the benchmark configurations of BASELINE.json, from the
UNMODIFIED reference (oracle/_ref, the reference's own sources compiled with
its Release flags; all host threads — results do not depend on the worker
count, test_engines.cpp:145-158).

  C2  run_synchronous, normalized Schwefel n=100, 2^20 chains, the paper
      ladder truncated to its first 2 levels (1000, 989.01, 0.99, 100) —
      the exact chain count and kernel the bench times (engines.cpp:131-207)
  C3  run_asynchronous and run_synchronous at full size: 16384 chains x the
      full paper ladder (1000, 0.01, 0.99, 100) = 1146 levels, n=30, for
      Schwefel, Ackley and Rastrigin (engines.cpp:66-123, 131-207)
  C4  hybrid_run at Table-8 scale: 16384 chains, n=500, truncated schedule
      (1000, 32, 0.9, 100) = 33 levels, then Nelder-Mead capped at 20000
      iterations (nelder_mead.cpp:117-136)

Each record holds best_x, best_f, winning_chain, evaluations, rng_draws and
the trace (float.hex), plus the reference's wall time.

    make -C oracle && python tests/golden/make_bench_golden.py [c2|c3|c4 ...]

Writes tests/golden/bench_golden.json (merging with what is there).
"""
import ctypes as C
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Config, Problem, Result, levels_of, ref  # noqa: E402

from paper_2408_00018_b200 import _abi  # noqa: E402

OUT = os.path.join(HERE, "bench_golden.json")
PAPER = (1000.0, 0.01, 0.99, 100)
C2_SCHED = (1000.0, 989.01, 0.99, 100)
C4_SCHED = (1000.0, 32.0, 0.9, 100)
SUITE = {"SCHWEFEL": (-512.0, 512.0, "F0_a"), "ACKLEY": (-30.0, 30.0, "F1"), "RASTRIGIN": (-5.12, 5.12, "F13")}


def record(d, wall):
    return {"best_x": [float(v).hex() for v in d["best_x"]], "best_f": float(d["best_f"]).hex(),
            "winning_chain": d["winning_chain"], "evaluations": d["evaluations"], "rng_draws": d["rng_draws"],
            "trace": [[a, b, float(c).hex()] for a, b, c in d["trace"]], "ref_wall_s": wall,
            "sa_evaluations": d.get("sa_evaluations", 0), "refine_evaluations": d.get("refine_evaluations", 0),
            "sa_best_f": float(d.get("sa_best_f", 0.0)).hex()}


def run(engine, family, dim, chains, sched, prec, seed=0):
    lo, hi, ident = SUITE[family]
    prob = Problem(family, dim, lo, hi, ident=ident)
    cfg = Config(chains, sched, seed, prec, 0, workers=0)
    res = Result(dim, levels_of(sched) + 1)
    t0 = time.time()
    rc = ref().ref_run(engine, C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
    assert rc == 0, ref().ref_last_error()
    return record(res.as_dict(), time.time() - t0)


def hybrid(dim, chains, sched, prec, nm_iters, seed=0):
    lo, hi, ident = SUITE["SCHWEFEL"]
    prob = Problem("SCHWEFEL", dim, lo, hi, ident=ident)
    cfg = Config(chains, PAPER, seed, prec, 0, workers=0)
    ts = _abi.psa_schedule(*sched, 0)
    nm = _abi.psa_nm_config(1.0, 2.0, 0.5, 0.5, 1e-12, 1e-10, nm_iters, 0)
    res = Result(dim, levels_of(sched) + 2)
    t0 = time.time()
    rc = ref().ref_hybrid_run(C.byref(prob.c), C.byref(cfg.c), C.byref(ts), C.byref(nm), C.byref(res.c))
    assert rc == 0, ref().ref_last_error()
    return record(res.as_dict(), time.time() - t0)


def main(which):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["generator"] = "tests/golden/make_bench_golden.py"
    data["threads"] = int(ref().ref_max_threads())
    if "c2" in which:
        for prec, key in ((1, "f32"), (0, "f64")):
            data[f"c2_{key}"] = dict(run(2, "SCHWEFEL", 100, 1 << 20, C2_SCHED, prec),
                                     family="SCHWEFEL", dim=100, chains=1 << 20, schedule=C2_SCHED, engine=2)
            print("c2", key, data[f"c2_{key}"]["ref_wall_s"], flush=True)
            json.dump(data, open(OUT, "w"))
    if "c3" in which:
        for fam in SUITE:
            for engine in (1, 2):
                for prec, key in ((1, "f32"), (0, "f64")):
                    name = f"c3_{fam.lower()}_v{engine}_{key}"
                    if name in data:
                        continue
                    data[name] = dict(run(engine, fam, 30, 16384, PAPER, prec), family=fam, dim=30, chains=16384,
                                      schedule=PAPER, engine=engine)
                    print(name, data[name]["ref_wall_s"], flush=True)
                    json.dump(data, open(OUT, "w"))
    if "c4" in which:
        for prec, key in ((0, "f64"), (1, "f32")):
            data[f"c4_{key}"] = dict(hybrid(500, 16384, C4_SCHED, prec, 20000), family="SCHWEFEL", dim=500,
                                     chains=16384, schedule=PAPER, truncated=C4_SCHED, nm_max_iters=20000)
            print("c4", key, data[f"c4_{key}"]["ref_wall_s"], flush=True)
            json.dump(data, open(OUT, "w"))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
