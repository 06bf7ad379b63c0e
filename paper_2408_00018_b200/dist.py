"""Multi-GPU SA: one process per GPU, chains sharded by global index.

Synchronous engine (V2): the per-level minloc is exchanged inside the
persistent kernel through peer-mapped mailboxes (exchange_level).
Asynchronous engine (V1): the chains never interact, so each GPU runs its
shard to the end and the ranks combine one small record each (end-state
winner, per-level trace minima, counts) — run_asynchronous_sharded.

torch.distributed is only the control plane here: it exchanges the CUDA IPC
handles of the mailboxes once (all_gather_object) and provides barriers; no
collective runs on the data path.  Because streams are keyed by the global
chain index and the cross-GPU selection is the same total order as the
single-GPU argmin, a G-GPU run returns the single-GPU result bit for bit
(tests/test_gpu_parity.py: two ranks sharing one GPU).
"""
from __future__ import annotations

import math
from typing import Sequence

from .api import Candidate, EngineConfig, ObjectiveFunction, Plan, RunResult, TracePoint


def shard_range(n_chains: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of the global chain range; the first n % world ranks
    take one extra chain."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    base, extra = divmod(n_chains, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def select_record(records: Sequence[Candidate]) -> int:
    """Host statement of the cross-GPU selection (engine.cuh better()):
    chain 0 with a NaN value wins, other NaNs never win, then smaller value,
    then smaller global chain.  Returns the index of the winning record."""
    def key(c: Candidate):
        v = c.f_value
        if math.isnan(v):
            return (0, 0.0, c.chain_index) if c.chain_index == 0 else (2, 0.0, c.chain_index)
        return (1, v, c.chain_index)
    return min(range(len(records)), key=lambda i: key(records[i]))


def make_sharded_plan(f: ObjectiveFunction, cfg: EngineConfig, group=None, max_blocks: int = 0) -> Plan:
    """Create this rank's shard of a synchronous run and connect it to every
    other rank's mailbox (collective over `group`, default WORLD)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    begin, end = shard_range(cfg.n_chains, rank, world)
    plan = Plan(f, cfg, engine=2, chain_begin=begin, chain_end=end, rank=rank, world=world,
                max_blocks=max_blocks)
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, plan.mailbox_ipc_handle(), group=group)
        peers = [plan.mailbox() if r == rank else plan.open_ipc(handles[r]) for r in range(world)]
        plan.set_peers(peers)
        dist.barrier(group)
        plan._before_close = lambda: dist.barrier(group)
    return plan


def combine_async_shards(results: Sequence[RunResult]) -> RunResult:
    """Merge the shard results of one asynchronous run (engines.cpp:66-123)
    into the single-GPU result, bit for bit: the end-state winner by the
    engines' selection order (select_record), the per-level trace as the
    minimum over shards of each shard's minimum (the device trace skips NaN
    chains and reports +inf for a level without a finite value, so a plain
    min over shards is the min over all chains), evaluations and draws as
    sums; cumulative_evals already count the global chain range."""
    if not results:
        raise ValueError("combine_async_shards: no shard results")
    w = select_record([Candidate(r.best_x, r.best_f, r.winning_chain) for r in results])
    win = results[w]
    levels = len(win.trace)
    trace = []
    for l in range(levels):
        vals = [r.trace[l].best_f for r in results]
        trace.append(TracePoint(win.trace[l].level, win.trace[l].cumulative_evals, min(vals)))
    return RunResult(best_x=list(win.best_x), best_f=win.best_f,
                     evaluations=sum(r.evaluations for r in results),
                     wall_time_s=max(r.wall_time_s for r in results), trace=trace,
                     winning_chain=win.winning_chain, rng_draws=sum(r.rng_draws for r in results))


def run_asynchronous_sharded(f: ObjectiveFunction, cfg: EngineConfig, group=None, stream: int = 0) -> RunResult:
    """V1 over the ranks of `group` (one GPU each): this rank's shard on its
    device, then one all_gather of the shard results; every rank returns the
    identical, single-GPU-equal RunResult."""
    import time

    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    begin, end = shard_range(cfg.n_chains, rank, world)
    t0 = time.perf_counter()
    with Plan(f, cfg, engine=1, chain_begin=begin, chain_end=end) as plan:
        plan.launch(stream)
        mine = plan.fetch(stream)
    mine.wall_time_s = time.perf_counter() - t0
    shards = [None] * world
    dist.all_gather_object(shards, mine, group=group)
    return combine_async_shards(shards)
