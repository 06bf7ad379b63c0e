"""configs[3] of BASELINE.json end to end: hybrid SA + Nelder-Mead on
normalized Schwefel n=500 with 2^20 chains, the truncated schedule
(1000, 32, 0.9, 100) and the reference's default NelderMeadConfig
(max_iters 0 => 50000 * n = 25M), through psa_hybrid_run.  One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_00018_b200 as psa  # noqa: E402

f = psa.registry_get("F0_g").with_dim(500)
cfg = psa.EngineConfig(n_chains=1 << 20, precision=psa.Precision.f64, seed=0)
t0 = time.perf_counter()
h = psa.hybrid_run(f, cfg, psa.AnnealSchedule(1000.0, 32.0, 0.9, 100), psa.NelderMeadConfig())
wall = time.perf_counter() - t0
print(json.dumps({"config": "configs[3]: hybrid, Schwefel n=500, 2^20 chains, SA (1000, 32, 0.9, 100) + default NM",
                  "wall_s": wall, "best_f": h.best_f, "abs_error": abs(h.best_f - f.reference.f_star),
                  "sa_evaluations": h.phases.sa_evaluations, "sa_best_f": h.phases.sa_best_f,
                  "nm_evaluations": h.phases.refine_evaluations, "evaluations": h.evaluations,
                  "trace_rows": len(h.trace)}))
