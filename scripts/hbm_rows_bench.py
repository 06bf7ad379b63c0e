"""Throughput of the HBM structure-of-arrays chain-row layout (large n).

Runs the synchronous engine on normalized Schwefel at n where rows no longer
fit in shared memory (or with PSA_FORCE_HBM_ROWS=1 at any n) and prints
evals/s plus the algorithmic HBM bandwidth of the fold (n * sizeof(R) bytes
read per trial).  One JSON line per (n, precision).

    python scripts/hbm_rows_bench.py --n 2000 --chains 262144 --levels 3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_00018_b200 as psa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[500, 2000])
    ap.add_argument("--chains", type=int, default=1 << 18)
    ap.add_argument("--levels", type=int, default=3)
    a = ap.parse_args()
    for n in a.n:
        for prec, rb in ((psa.Precision.f32, 4), (psa.Precision.f64, 8)):
            tmin = 1000.0 * 0.9 ** a.levels * 1.0001
            cfg = psa.EngineConfig(n_chains=a.chains, precision=prec,
                                   schedule=psa.AnnealSchedule(1000.0, tmin, 0.9, 100))
            f = psa.registry_get("F0_g").with_dim(n)
            with psa.Plan(f, cfg) as p:
                s = torch.cuda.current_stream()
                p.launch(s.cuda_stream)
                p.fetch(s.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                p.launch(s.cuda_stream)
                e1.record(s)
                r = p.fetch(s.cuda_stream)
                ms = e0.elapsed_time(e1)
                trials = a.chains * 100 * p.levels
                print(json.dumps({"n": n, "precision": "f32" if rb == 4 else "f64", "chains": a.chains,
                                  "levels": p.levels, "layout": p.description, "ms": ms,
                                  "evals_per_s": r.evaluations / (ms / 1e3),
                                  "fold_read_GBps": trials * n * rb / (ms / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
