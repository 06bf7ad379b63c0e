"""One C1 run (Schwefel n=10, 1024 chains, the paper ladder) for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_00018_b200 as psa  # noqa: E402

f = psa.registry_get("F0_a").with_dim(10)
cfg = psa.EngineConfig(n_chains=1024, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100), precision=psa.Precision.f32)
with psa.Plan(f, cfg) as p:
    p.launch()
    r = p.fetch()
print(r.best_f, r.winning_chain)
