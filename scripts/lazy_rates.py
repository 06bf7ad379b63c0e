"""Deferred fold vs fold-every-trial across the paper ladder's temperature
range (C2 shape: Schwefel n=100, 2^20 chains): evals/s per 10-level window
and the fraction of trials settled by exact folds.

    python scripts/lazy_rates.py [--precision f32|f64] [--chains N]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_00018_b200 as psa  # noqa: E402


def run(f, cfg, reps=3):
    s = torch.cuda.current_stream()
    with psa.Plan(f, cfg) as p:
        p.launch(s.cuda_stream)
        r = p.fetch(s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            p.launch(s.cuda_stream)
        e1.record(s)
        r = p.fetch(s.cuda_stream)
        ms = e0.elapsed_time(e1) / reps
        return p.description, r, ms, p.exact_settles()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--chains", type=int, default=1 << 20)
    ap.add_argument("--n", type=int, default=100)
    a = ap.parse_args()
    f = psa.registry_get("F0_a").with_dim(a.n)
    prec = psa.Precision.f32 if a.precision == "f32" else psa.Precision.f64
    for t0 in (1000.0, 100.0, 10.0, 1.0, 0.1, 0.0125):
        sched = psa.AnnealSchedule(t0, t0 * 0.99 ** 10 * 0.999, 0.99, 100)
        cfg = psa.EngineConfig(n_chains=a.chains, schedule=sched, precision=prec, seed=1)
        out = {"t0": t0, "n": a.n, "chains": a.chains, "dtype": a.precision}
        for key, env in (("lazy", "1"), ("fold", "0")):
            os.environ["PSA_LAZY"] = env
            desc, r, ms, settles = run(f, cfg)
            out[key] = {"kernel": desc.split(" (")[0], "evals_per_s": r.evaluations / (ms * 1e-3),
                        "ms": ms, "exact_settle_frac": settles / r.evaluations, "best_f": r.best_f}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
