"""Concurrent repetitions on the device, the CLI search
commands and checkpoint/resume, against the reference's own outputs.

* sk_saw_multi summaries == sk_saw_batch summaries for the same
  (master, batch, walker range), search by search;
* runner.target_campaign (all repetitions concurrent on the device) ==
  the reference's sequential campaign (tests/golden/records.json) and the
  oracle's per-repetition solves;
* `solve` / `target` CLI outputs == the reference CLI's (tests/golden/host.json);
* a solve interrupted and resumed from its checkpoint == an uninterrupted one.
"""

import contextlib
import io
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from conftest import load_json  # noqa: E402

from paper_2210_15962_b200 import _lib, cli, engine  # noqa: E402
from paper_2210_15962_b200.runner import (  # noqa: E402
    RunConfig,
    derive_repetition_seed,
    solve,
    target_campaign,
)


def summary(L, n, master, batch, begin, W):
    s = torch.empty(engine.SUMMARY_WORDS, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().sk_saw_batch(L, n, None, master, batch, begin, W, None, None, None, None, s.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream))
    return s.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("L,W,R", [(27, 8, 13), (101, 37, 5), (201, 64, 3), (449, 16, 4)])
def test_multi_equals_single_searches(L, W, R):
    d = (L + 1) // 2
    n = 4 * d
    rng = np.random.default_rng(L)
    masters = rng.integers(0, 2**63, R, dtype=np.int64).view(np.uint64)
    batches = rng.integers(0, 50, R).astype(np.uint64)
    begin = 1000
    mb = torch.from_numpy(np.stack([masters, batches]).view(np.int64)).cuda()
    out = torch.empty((R, engine.SUMMARY_WORDS), dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().sk_saw_multi(L, n, mb[0].data_ptr(), mb[1].data_ptr(), R, begin, W, out.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream))
    got = out.cpu().numpy().view(np.uint64)
    for r in range(R):
        want = summary(L, n, int(masters[r]), int(batches[r]), begin, W)
        np.testing.assert_array_equal(got[r], want, err_msg=f"search {r}")


@pytest.mark.parametrize("layout", [_lib.VISITED_AUTO, _lib.VISITED_FINGERPRINT, _lib.VISITED_GLOBAL])
def test_run_multi_sharded_equals_run_batch(layout):
    # three shards on one device run on three streams, possibly concurrently:
    # their global visited-key scratch must be private per stream
    L, W = 101, 3 * 4096
    n = 8 * 51
    masters = [derive_repetition_seed(9, r) for r in range(6)]
    batches = [0, 3, 1, 7, 2, 2]
    _lib.set_visited_layout(layout)
    try:
        for devs in (None, [0, 0, 0]):
            eng = engine.BatchEngine(L, W, n, 0, devices=devs)
            res = eng.run_multi(masters, batches)
            for m, b, x in zip(masters, batches, res):
                y = engine.BatchEngine(L, W, n, m).run_batch(b)
                assert (x.best_E, x.walker, x.steps_sum) == (y.best_E, y.walker, y.steps_sum)
                np.testing.assert_array_equal(x.best_words, y.best_words)
    finally:
        _lib.set_visited_layout(_lib.VISITED_AUTO)


def test_campaign_matches_reference_golden(golden_records):
    want = golden_records["campaign_L15"]
    got = target_campaign(RunConfig(L=15, walkers=2, master_seed=4, target_E=15, max_nses=100_000), 5)
    assert got.nses == want["nses"] and got.censored == want["censored"]


@pytest.mark.parametrize("group", [1, 3, 1 << 20])
def test_campaign_equals_sequential_and_oracle(oracle, group):
    cfg = RunConfig(L=27, walkers=8, master_seed=5, target_E=37, max_nses=300_000)
    got = target_campaign(cfg, 9, max_walks_per_launch=group * cfg.walkers)
    for rep in range(9):
        m = derive_repetition_seed(cfg.master_seed, rep)
        rec = oracle.solve_record(27, 8, 8, m, cfg.max_nses, cfg.target_E)
        assert got.nses[rep] == rec["total_nses"], rep
        assert got.censored[rep] == (rec["stop_reason"] != "target_reached"), rep
        seq = solve(RunConfig(L=27, walkers=8, master_seed=m, target_E=37, max_nses=300_000))
        assert seq.total_nses == got.nses[rep]


def test_campaign_censoring_l45(oracle):
    # a target below the optimum (E=118): every repetition exhausts its budget
    cfg = RunConfig(L=45, walkers=4, master_seed=2, target_E=100, max_nses=20_000)
    got = target_campaign(cfg, 4)
    assert all(got.censored)
    for rep in range(4):
        m = derive_repetition_seed(2, rep)
        assert got.nses[rep] == oracle.solve_record(45, 4, 8, m, 20_000, 100)["total_nses"]


@pytest.mark.parametrize("idx", [i for i, c in enumerate(load_json("host.json")["cli"]["cases"])
                                 if c["argv"][0] in ("solve", "target") and c["code"] == 0])
def test_cli_search_commands_match_reference(idx):
    case = load_json("host.json")["cli"]["cases"][idx]
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(case["argv"])
    assert code == case["code"], err.getvalue()
    if case["argv"][0] == "solve":
        rec = json.loads(out.getvalue())
        assert rec.pop("wall_time_s") >= 0
        assert rec == case["stdout"]
    else:
        assert out.getvalue() == case["stdout"]


def test_checkpoint_resume_equals_uninterrupted(tmp_path, golden_records):
    item = next(x for x in golden_records["records"] if x["config"]["L"] == 101)
    cfg = RunConfig(**item["config"])
    want = item["record"]
    assert want["batches"] >= 2
    ck = str(tmp_path / "ck.json")
    # "interrupted" after one batch: same search, smaller budget
    first = cfg.max_nses // want["batches"] if cfg.max_nses else None
    part = solve(RunConfig(**{**item["config"], "max_nses": max(1, first or 1)}), checkpoint=ck)
    assert part.batches >= 1
    rec = solve(cfg, checkpoint=ck).to_json_dict()
    rec.pop("wall_time_s")
    assert rec == want
    # a checkpoint of another search is refused
    with pytest.raises(ValueError):
        solve(RunConfig(**{**item["config"], "master_seed": 12345}), checkpoint=ck)


def test_speculative_batches_change_nothing(oracle):
    # min_walks_per_launch=1 disables speculation; a large value runs up to 64
    # batches of every repetition per launch and discards those after its stop
    cfg = RunConfig(L=45, walkers=3, master_seed=13, target_E=118, max_nses=200_000)
    plain = target_campaign(cfg, 12, min_walks_per_launch=1)
    spec = target_campaign(cfg, 12, min_walks_per_launch=1 << 20)
    assert plain.nses == spec.nses and plain.censored == spec.censored
    assert plain.censored_count == 6  # both outcomes occur (oracle: 6 of 12 reach the optimum)
    for rep in range(12):
        rec = oracle.solve_record(45, 3, 8, derive_repetition_seed(13, rep), 200_000, 118)
        assert spec.nses[rep] == rec["total_nses"]
