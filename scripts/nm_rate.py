"""Nelder-Mead rate on configs[3] at growing iteration caps: SA phase once,
then NM from its best point with max_iters = each cap; prints iterations,
evaluations (a shrink costs n of them), seconds and us per iteration."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_00018_b200 as psa  # noqa: E402

caps = [int(a) for a in sys.argv[1:]] or [20000, 100000, 300000]
f = psa.registry_get("F0_g").with_dim(500)
sa = psa.run_synchronous(f, psa.EngineConfig(n_chains=1 << 20, precision=psa.Precision.f64, seed=0,
                                             schedule=psa.AnnealSchedule(1000.0, 32.0, 0.9, 100)))
for cap in caps:
    t0 = time.perf_counter()
    r = psa.nelder_mead_minimize(f, sa.best_x, psa.NelderMeadConfig(max_iters=cap))
    dt = time.perf_counter() - t0
    print(json.dumps({"cap": cap, "iterations": r.iterations, "evaluations": r.evaluations, "seconds": dt,
                      "us_per_iteration": 1e6 * dt / max(1, r.iterations), "f_best": r.f_best}), flush=True)
