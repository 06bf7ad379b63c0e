"""Multi-GPU synchronous SA: one process per GPU, chains sharded by global
index, the per-level minloc exchanged inside the persistent kernel through
peer-mapped mailboxes (engine.cu: exchange_level).

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

from .api import Candidate, EngineConfig, ObjectiveFunction, Plan


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
    return plan
