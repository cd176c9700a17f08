"""The multi-rank product path on the device (-m gpu): two processes share
cuda:0 over a gloo group and run solve(..., process_group=) and
target_campaign(..., process_group=); each rank's walks are its contiguous
walker slice (engine._slices) and the per-batch merge is the single
all_gather of engine.merge_many_across_ranks.  The records must equal the
single-process ones (runner.py:250-256: the global walker index keys both
the seeds and the tie-break, so the result is independent of the rank
count)."""

import json
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from conftest import ROOT  # noqa: E402,F401

CONFIGS = [
    dict(L=101, walkers=4096, master_seed=1, max_nses=4096 * 408 * 50 * 2),
    dict(L=201, walkers=1000, master_seed=2, max_nses=3 * 1000 * 808 * 100),
    dict(L=27, walkers=7, master_seed=5, target_E=37, max_nses=10**6),
    dict(L=449, walkers=301, master_seed=9, max_nses=1),
]
CAMPAIGN = dict(L=21, walkers=3, master_seed=4, target_E=26, max_nses=60_000)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_15962_b200.runner import RunConfig, solve, target_campaign

        recs = []
        for cfg in CONFIGS:
            r = solve(RunConfig(**cfg), process_group=dist.group.WORLD).to_json_dict()
            r.pop("wall_time_s")
            recs.append(r)
        camp = target_campaign(RunConfig(**CAMPAIGN), 6, process_group=dist.group.WORLD)
        out_q.put((rank, json.dumps(recs), camp.nses, camp.censored))
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_single_process():
    from paper_2210_15962_b200.runner import RunConfig, solve, target_campaign

    want = []
    for cfg in CONFIGS:
        r = solve(RunConfig(**cfg)).to_json_dict()
        r.pop("wall_time_s")
        want.append(r)
    camp = target_campaign(RunConfig(**CAMPAIGN), 6)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, recs, nses, cens in results:
        assert recs == json.dumps(want), rank
        assert (nses, cens) == (camp.nses, camp.censored), rank
