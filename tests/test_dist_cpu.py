"""Host side of the multi-GPU path on CPU (gloo, world_size 2): shard
ranges tile the global chain range, mailbox handles are exchanged through
torch.distributed exactly as make_sharded_plan does, and every rank selects
the same winner record."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_00018_b200.api import Candidate
from paper_2408_00018_b200.dist import select_record, shard_range


def test_shard_range_tiles():
    for n in (1, 7, 1024, 1 << 20, (1 << 23) + 3):
        for world in (1, 2, 3, 4, 8):
            if n < world:
                continue
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_select_record_semantics():
    nan = float("nan")
    assert select_record([Candidate([], 3.0, 5), Candidate([], 1.0, 9), Candidate([], 1.0, 2)]) == 2
    assert select_record([Candidate([], -0.0, 7), Candidate([], 0.0, 3)]) == 1  # -0 == +0 -> smaller chain
    assert select_record([Candidate([], 1.0, 4), Candidate([], nan, 0)]) == 1  # NaN at chain 0 sticks
    assert select_record([Candidate([], nan, 3), Candidate([], 5.0, 8)]) == 1  # other NaNs never win


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = (1 << 23) + 5
        begin, end = shard_range(n, rank, world)
        spans = [None] * world
        dist.all_gather_object(spans, (begin, end))
        handle = bytes([rank]) * 64  # stands in for a cudaIpcMemHandle_t
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        # every rank's local winner record; each rank must pick the same one
        local = Candidate([], [-5.0, -7.25, -7.25, 1.0][rank % 4], begin + 17)
        recs = [None] * world
        dist.all_gather_object(recs, (local.f_value, local.chain_index))
        pick = select_record([Candidate([], v, c) for v, c in recs])
        picks = [None] * world
        dist.all_gather_object(picks, pick)
        q.put((rank, spans, [h[0] for h in handles], picks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    spans = out[0][1]
    assert spans == [shard_range((1 << 23) + 5, r, world) for r in range(world)]
    for rank, sp, hs, picks in out:
        assert sp == spans and hs == list(range(world))
        assert len(set(picks)) == 1  # same winner everywhere


def test_combine_async_shards_semantics():
    from paper_2408_00018_b200.api import RunResult, TracePoint
    from paper_2408_00018_b200.dist import combine_async_shards
    inf = float("inf")
    a = RunResult(best_x=[1.0], best_f=-2.0, evaluations=10, trace=[TracePoint(0, 30, -1.0), TracePoint(1, 60, -2.0)],
                  winning_chain=4, rng_draws=27)
    b = RunResult(best_x=[2.0], best_f=-2.0, evaluations=10, trace=[TracePoint(0, 30, inf), TracePoint(1, 60, -3.0)],
                  winning_chain=1, rng_draws=27)
    c = combine_async_shards([a, b])
    assert c.winning_chain == 1 and c.best_x == [2.0]  # tie -> smaller global chain
    assert [t.best_f for t in c.trace] == [-1.0, -3.0]
    assert c.evaluations == 20 and c.rng_draws == 54
