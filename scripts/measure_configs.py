"""Device throughput of every BASELINE.json configuration (one JSON line each).

  C1  synchronous, Schwefel n=10, 1024 chains, paper ladder (1146 levels)
  C2  synchronous, Schwefel n=100, 2^20 chains (f32 and f64; --levels to truncate)
  C3  asynchronous vs synchronous, n=30 suite (Schwefel, Ackley, Rastrigin),
      16384 chains (the paper's 256x64), paper ladder
  C4  the SA phase of the hybrid: Schwefel n=500, 2^20 chains, (1000, 32, 0.9, 100)

Device time comes from CUDA events around psa_plan_launch on the launch
stream; results are fetched and sanity-checked (accounting).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_00018_b200 as psa  # noqa: E402


def timed(f, cfg, engine=2, reps=2):
    with psa.Plan(f, cfg, engine=engine) as p:
        s = torch.cuda.current_stream()
        p.launch(s.cuda_stream)  # warm-up
        p.fetch(s.cuda_stream)
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.launch(s.cuda_stream)
            e1.record(s)
            r = p.fetch(s.cuda_stream)
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return r, best


def line(name, f, cfg, engine=2, **extra):
    r, ms = timed(f, cfg, engine)
    assert r.evaluations == psa.expected_evaluations(cfg.schedule, cfg.n_chains)
    d = {"config": name, "engine": {1: "v1", 2: "v2"}[engine], "n": f.dim, "chains": cfg.n_chains,
         "precision": cfg.precision.name, "levels": len(r.trace), "evaluations": r.evaluations, "ms": ms,
         "evals_per_s": r.evaluations / (ms / 1e3), "best_f": r.best_f,
         "abs_error": abs(r.best_f - f.reference.f_star), "winning_chain": r.winning_chain}
    d.update(extra)
    print(json.dumps(d), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4")
    ap.add_argument("--c2-tmin", type=float, default=0.01)
    a = ap.parse_args()
    which = set(a.only.split(","))
    paper = psa.AnnealSchedule(1000.0, 0.01, 0.99, 100)
    schw = psa.registry_get("F0_a")
    if "C1" in which:
        for prec in (psa.Precision.f64, psa.Precision.f32):
            line("C1", schw.with_dim(10), psa.EngineConfig(n_chains=1024, schedule=paper, precision=prec))
    if "C2" in which:
        sched = psa.AnnealSchedule(1000.0, a.c2_tmin, 0.99, 100)
        for prec in (psa.Precision.f32, psa.Precision.f64):
            line("C2", schw.with_dim(100), psa.EngineConfig(n_chains=1 << 20, schedule=sched, precision=prec))
    if "C3" in which:
        for fid in ("F0_c", "F1_a", "F13_a"):
            f = psa.registry_get(fid)
            if f.dim != 30:
                f = f.with_dim(30)
            for engine in (1, 2):
                line("C3", f, psa.EngineConfig(n_chains=16384, schedule=paper, precision=psa.Precision.f32),
                     engine=engine, function=fid)
    if "C4" in which:
        trunc = psa.AnnealSchedule(1000.0, 32.0, 0.9, 100)
        for prec in (psa.Precision.f32, psa.Precision.f64):
            line("C4-SA", psa.registry_get("F0_g").with_dim(500),
                 psa.EngineConfig(n_chains=1 << 20, schedule=trunc, precision=prec))


if __name__ == "__main__":
    main()
