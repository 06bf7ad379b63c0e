"""Small runs of every engine kernel for compute-sanitizer (racecheck,
synccheck, memcheck): the deferred-fold, one-chain, chain-pair and
producer/consumer V2 kernels, V1, the cluster Nelder-Mead and the two-rank
level exchange on one GPU.  Each run is checked against the single-plan /
oracle result so a tool-induced change would show too.

    compute-sanitizer --tool racecheck python scripts/sanitize_runs.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2408_00018_b200 as psa  # noqa: E402


def run(mode, engine=2, n=10, chains=2048, prec=psa.Precision.f32, start=psa.StartMode.random_per_chain):
    if mode:
        os.environ["PSA_V2_MODE"] = mode
    else:
        os.environ.pop("PSA_V2_MODE", None)
    f = psa.registry_get("F0_a").with_dim(n)
    cfg = psa.EngineConfig(n_chains=chains, schedule=psa.AnnealSchedule(50.0, 10.0, 0.5, 40), precision=prec,
                           seed=3, start_mode=start)
    with psa.Plan(f, cfg, engine=engine) as p:
        p.launch()
        r = p.fetch()
        print(mode or "default", engine, p.description.split(" (")[0], r.best_f, flush=True)
    return r


def main():
    base = run("single")
    for mode in ("lazy1", "pair", "pc", "lazypair"):
        r = run(mode)
        assert r.best_f == base.best_f and r.winning_chain == base.winning_chain, mode
    run("", engine=1)
    run("pc", engine=1)
    run("lazy1", n=100, chains=4096, prec=psa.Precision.f64, start=psa.StartMode.shared_point)
    # cluster Nelder-Mead (n = 64: 2 CTAs) and the batched form
    f = psa.registry_get("F0_a").with_dim(64)
    nm = psa.nelder_mead_minimize(f, [100.0] * 64, psa.NelderMeadConfig(max_iters=300))
    print("nm", nm.iterations, nm.f_best, flush=True)
    # two ranks sharing the GPU: the in-kernel level exchange
    import torch
    from paper_2408_00018_b200.dist import shard_range
    os.environ["PSA_V2_MODE"] = "lazy1"
    f = psa.registry_get("F0_a").with_dim(12)
    cfg = psa.EngineConfig(n_chains=4000, schedule=psa.AnnealSchedule(50.0, 10.0, 0.5, 20),
                           precision=psa.Precision.f32, seed=5)
    with psa.Plan(f, cfg) as single:
        single.launch()
        ref = single.fetch()
    plans = []
    for r in range(2):
        b, e = shard_range(4000, r, 2)
        plans.append(psa.Plan(f, cfg, chain_begin=b, chain_end=e, rank=r, world=2, max_blocks=16))
    boxes = [p.mailbox() for p in plans]
    for p in plans:
        p.set_peers(boxes)
    streams = [torch.cuda.Stream() for _ in range(2)]
    for p, s in zip(plans, streams):
        p.launch(s.cuda_stream)
    outs = [p.fetch(s.cuda_stream) for p, s in zip(plans, streams)]
    for o in outs:
        assert o.best_f == ref.best_f and o.winning_chain == ref.winning_chain
    print("two-rank exchange ok", ref.best_f, flush=True)
    for p in plans:
        p.close()


if __name__ == "__main__":
    main()
