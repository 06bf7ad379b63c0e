"""Config C4 of BASELINE.json: hybrid SA + Nelder–Mead on normalized
Schwefel n=500.

The SA phase is the paper's truncated schedule that reproduces Table 8's
budget shape (T0=1000, Tmin=32, rho=0.9, N=100 -> 33 levels); the polish is
the device Nelder–Mead, capped at --nm-iters iterations (the reference's
default cap is 50000*n = 25M iterations; its CPU implementation takes
~644 us per iteration at n=500 — SURVEY.md §3.3).  Prints one JSON line.

    python scripts/hybrid_c4.py --chains 1048576 --nm-iters 20000
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2408_00018_b200 as psa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500)
    ap.add_argument("--chains", type=int, default=1 << 20)
    ap.add_argument("--nm-iters", type=int, default=20000)
    ap.add_argument("--precision", default="f64")
    a = ap.parse_args()
    f = psa.registry_get("F0_g").with_dim(a.n)
    prec = psa.Precision.f32 if a.precision == "f32" else psa.Precision.f64
    cfg = psa.EngineConfig(n_chains=a.chains, precision=prec, seed=0)
    trunc = psa.AnnealSchedule(1000.0, 32.0, 0.9, 100)
    nm = psa.NelderMeadConfig(max_iters=a.nm_iters)
    # SA phase alone (device time through the plan API)
    t0 = time.perf_counter()
    sa = psa.run_synchronous(f, psa.EngineConfig(n_chains=a.chains, precision=prec, seed=0, schedule=trunc))
    t_sa = time.perf_counter() - t0
    t1 = time.perf_counter()
    r = psa.nelder_mead_minimize(f, sa.best_x, nm)
    t_nm = time.perf_counter() - t1
    t2 = time.perf_counter()
    h = psa.hybrid_run(f, cfg, trunc, nm)
    t_h = time.perf_counter() - t2
    print(json.dumps({
        "config": "C4 hybrid, Schwefel n=%d, %d chains, SA (1000, 32, 0.9, 100) + NM cap %d" % (a.n, a.chains, a.nm_iters),
        "precision": a.precision,
        "sa_levels": len(sa.trace), "sa_evaluations": sa.evaluations, "sa_seconds": t_sa,
        "sa_evals_per_s": sa.evaluations / t_sa, "sa_best_f": sa.best_f,
        "nm_iterations": r.iterations, "nm_evaluations": r.evaluations, "nm_seconds": t_nm,
        "nm_us_per_iteration": 1e6 * t_nm / max(1, r.iterations), "nm_f_best": r.f_best,
        "hybrid_seconds": t_h, "hybrid_best_f": h.best_f,
        "hybrid_abs_error": abs(h.best_f - f.reference.f_star),
        "hybrid_refine_evaluations": h.phases.refine_evaluations if h.phases else None,
    }))


if __name__ == "__main__":
    main()
