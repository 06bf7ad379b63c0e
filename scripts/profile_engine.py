"""One engine launch for profiling under ncu (one GPU, small level count).

    ncu --set full ... python scripts/profile_engine.py --levels 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2408_00018_b200 as psa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--chains", type=int, default=1 << 20)
    ap.add_argument("--t0", type=float, default=1000.0)
    ap.add_argument("--tmin", type=float, default=989.0)  # 1000, 990 -> 2 levels
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--engine", type=int, default=2)
    ap.add_argument("--launches", type=int, default=2)
    a = ap.parse_args()
    f = psa.registry_get("F0_a").with_dim(a.n)
    cfg = psa.EngineConfig(n_chains=a.chains, schedule=psa.AnnealSchedule(a.t0, a.tmin, 0.99, 100),
                           precision=psa.Precision.f32 if a.precision == "f32" else psa.Precision.f64)
    with psa.Plan(f, cfg, engine=a.engine) as p:
        for _ in range(a.launches):
            p.launch()
            r = p.fetch()
    print("levels", p.levels, "best_f", r.best_f, "evals", r.evaluations)


if __name__ == "__main__":
    main()
