"""Per-level cost of the synchronous engine at small chain counts: time the
C1 workload (Schwefel n=10, 1024 chains, 1146 levels) at several sweep
lengths N; the intercept of ms-per-level against N is the level-end cost
(argmin, grid barrier, winner replay, level-start broadcast)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_00018_b200 as psa  # noqa: E402

for chains, n in ((1024, 10), (16384, 30)):
    f = psa.registry_get("F0_a").with_dim(n)
    for N in (25, 50, 100, 200):
        cfg = psa.EngineConfig(n_chains=chains, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, N),
                               precision=psa.Precision.f32)
        with psa.Plan(f, cfg) as p:
            s = torch.cuda.current_stream()
            p.launch(s.cuda_stream)
            p.fetch(s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.launch(s.cuda_stream)
            e1.record(s)
            p.fetch(s.cuda_stream)
            ms = e0.elapsed_time(e1)
            print(f"chains={chains} n={n} N={N} us_per_level={1e3 * ms / p.levels:.2f} {p.description}", flush=True)
