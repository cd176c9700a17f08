"""N>1 host logic on CPU: world_size-2 gloo ranks each own a contiguous
walker slice of one batch (engine._slices) and merge with
engine.merge_across_ranks; the merged result must equal the single-process
reference merge (runner.py:251-256) of the whole batch.  Per-walk outputs of
the slices come from the oracle, so this exercises exactly the collective
logic the NCCL path runs on the GPU box."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path setup)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, L, W, master, batch, out_q):
    import oracle
    from paper_2210_15962_b200 import engine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        begin, cnt = engine._slices(W, world)[rank]
        d = (L + 1) // 2
        seeds = oracle.derive_walk_seeds(master, batch, cnt, walker_begin=begin)
        be, bw, st, _ = oracle.batch_outputs(L, 8 * d, seeds, threads=1)
        win = None
        if cnt:
            i = min(range(cnt), key=lambda j: (int(be[j]), j))
            win = engine.BatchResult(int(be[i]), begin + i, 0, bw[i])
        import torch

        res = engine.merge_across_ranks(win, int(st.sum()), (d + 63) // 64, None, torch.device("cpu"))
        out_q.put((rank, res.best_E, res.walker, res.steps_sum, [int(x) for x in res.best_words]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,W", [(27, 37), (101, 12), (129, 3)])
def test_two_rank_merge_equals_single_process(L, W):
    import oracle

    master, batch = 3, 1
    d = (L + 1) // 2
    seeds = oracle.derive_walk_seeds(master, batch, W)
    be, bw, st, _ = oracle.batch_outputs(L, 8 * d, seeds)
    best = None
    for w in range(W):  # runner.py:252-256
        if best is None or int(be[w]) < best[0]:
            best = (int(be[w]), w, [int(x) for x in bw[w]])

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, L, W, master, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e, walker, steps, words in results:
        assert (e, walker, words) == best, rank
        assert steps == int(st.sum())


def _rank_many(rank, world, port, L, W, masters, batch, out_q):
    """merge_many_across_ranks: R searches, each sharded over the ranks."""
    import oracle
    from paper_2210_15962_b200 import engine, runner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        begin, cnt = engine._slices(W, world)[rank]
        d = (L + 1) // 2
        wins, steps = [], []
        for m in masters:
            seeds = oracle.derive_walk_seeds(m, batch, cnt, walker_begin=begin)
            be, bw, st, _ = oracle.batch_outputs(L, 8 * d, seeds, threads=1)
            win = None
            if cnt:
                i = min(range(cnt), key=lambda j: (int(be[j]), j))
                win = engine.BatchResult(int(be[i]), begin + i, 0, bw[i])
            wins.append(win)
            steps.append(int(st.sum()))
        res = engine.merge_many_across_ranks(wins, steps, (d + 63) // 64, None, torch.device("cpu"))
        # every rank must take the same runtime-stop decision: _elapsed is the max over ranks
        el = runner._elapsed(runner.time.monotonic() - (5.0 if rank == 1 else 0.0), dist.group.WORLD)
        out_q.put((rank, [(r.best_E, r.walker, r.steps_sum, [int(x) for x in r.best_words]) for r in res], el))
    finally:
        dist.destroy_process_group()


def test_two_rank_multi_search_merge():
    import oracle

    L, W, batch = 45, 7, 2
    masters = [oracle.derive_repetition_seed(8, r) for r in range(5)]
    d = (L + 1) // 2
    want = []
    for m in masters:
        seeds = oracle.derive_walk_seeds(m, batch, W)
        be, bw, st, _ = oracle.batch_outputs(L, 8 * d, seeds)
        w = min(range(W), key=lambda j: (int(be[j]), j))
        want.append((int(be[w]), w, int(st.sum()), [int(x) for x in bw[w]]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_many, args=(r, 2, port, L, W, masters, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, el in results:
        assert got == want, rank
        assert el >= 5.0, rank  # rank 1's 5 s head start is every rank's elapsed time
