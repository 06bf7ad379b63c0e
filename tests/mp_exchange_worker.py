"""One rank of a multi-process synchronous run (TEST HELPER, launched by
tests/test_gpu_parity.py::test_two_process_ipc_exchange).

Each process is one rank: torch.distributed over gloo is the control plane
(it all-gathers the CUDA IPC handles of the mailboxes once, in
dist.make_sharded_plan); the per-level minloc then crosses processes inside
the persistent kernels through the IPC-mapped mailboxes.  Both processes
share the one GPU of the box (the contexts time-slice), which is enough to
run the cross-process data path end to end.

usage: RANK=r WORLD_SIZE=w MASTER_ADDR=127.0.0.1 MASTER_PORT=p \
       python tests/mp_exchange_worker.py OUT.json PREC START DIM CHAINS T0 TMIN RHO N SEED
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out, prec, start, dim, chains, t0, tmin, rho, n, seed = sys.argv[1:11]
    import torch
    import torch.distributed as dist

    import paper_2408_00018_b200 as psa
    from paper_2408_00018_b200.dist import make_sharded_plan

    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    f = psa.registry_get("F0_a").with_dim(int(dim))
    cfg = psa.EngineConfig(n_chains=int(chains),
                           schedule=psa.AnnealSchedule(float(t0), float(tmin), float(rho), int(n)),
                           precision=psa.Precision.f32 if prec == "f32" else psa.Precision.f64,
                           seed=int(seed),
                           start_mode=psa.StartMode.random_per_chain if start == "random"
                           else psa.StartMode.shared_point)
    results = []
    with make_sharded_plan(f, cfg) as plan:
        for _ in range(2):  # two launches: the epoch tag keeps them apart
            plan.launch(0)
            r = plan.fetch(0)
            results.append({"best_x": [v.hex() for v in r.best_x], "best_f": r.best_f.hex(),
                            "winning_chain": r.winning_chain, "evaluations": r.evaluations,
                            "rng_draws": r.rng_draws,
                            "trace": [[t.level, t.cumulative_evals, t.best_f.hex()] for t in r.trace],
                            "description": plan.description})
    with open(f"{out}.rank{rank}", "w") as fh:
        json.dump(results, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
