"""BASELINE configs 1 and 2 as SURVEY §8(d) defines them, and the exhaustive
optima beyond L=41, on the device (-m gpu).

Fixtures are reference outputs (oracle/gen_golden_r2.py, run against
/root/reference in the build container):
  * config 2: traces of derive_walk_seed(1, 0, w), w < 64, at L=101
    (run_walk_traced, saw.py:139-148) and the RunRecord of
    RunConfig(L=101, walkers=4096, master_seed=1, max_nses=167,116,800)
    (runner.py:213-291), for every evaluator / visited-set layout;
  * config 1: RunConfig(L=27, walkers=8, master_seed=s, target_E=37,
    max_nses=10**6) for all s < 100, byte-equal RunRecords;
  * exhaustive_optimum(L) for L = 43..55 (saw.py:151-168), plus full-scan
    cross-checks of the device scan against the threaded CPU oracle at
    L = 55 and 57.
"""

import hashlib
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2210_15962_b200 import _kernels, _lib  # noqa: E402
from paper_2210_15962_b200.codec import encode  # noqa: E402
from paper_2210_15962_b200.runner import RunConfig, derive_walk_seed, solve  # noqa: E402
from paper_2210_15962_b200.saw import WalkConfig, exhaustive_optimum, run_walk_traced  # noqa: E402

SETUPS = [(_lib.VARIANT_SCALAR, _lib.VISITED_AUTO), (_lib.VARIANT_FAST, _lib.VISITED_AUTO),
          (_lib.VARIANT_FAST, _lib.VISITED_SMEM), (_lib.VARIANT_FAST, _lib.VISITED_FINGERPRINT),
          (_lib.VARIANT_FAST, _lib.VISITED_GLOBAL)]


@pytest.fixture(params=SETUPS, ids=["scalar", "fast", "fast_smem", "fast_fp", "fast_gk"])
def setup(request):
    ev, layout = request.param
    _lib.set_variant(ev)
    _lib.set_visited_layout(layout)
    yield request.param
    _lib.set_variant(_lib.VARIANT_AUTO)
    _lib.set_visited_layout(_lib.VISITED_AUTO)


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def test_config2_traces_64_walkers(setup, golden_config2_traces):
    g = golden_config2_traces
    for w in g["walks"]:
        seed = derive_walk_seed(g["master"], g["batch"], w["w"])
        res, tr = run_walk_traced(WalkConfig(L=g["L"], n=g["n"], seed=seed))
        assert (res.best_E, res.steps_taken, res.dead_end) == (w["best_E"], w["steps"], w["dead"]), w["w"]
        assert encode(res.best_half) == w["best_hex"], w["w"]
        assert tr.pivots.shape[0] == w["rows_pivots"] and tr.deltas.shape[0] == w["rows_deltas"]
        assert sha(tr.pivots.astype(np.int8)) == w["sha_pivots_i8"], w["w"]
        assert sha(tr.deltas.astype(np.int64)) == w["sha_deltas_i64"], w["w"]


def test_config2_run_record(setup, golden_config_records):
    item = golden_config_records["records"][0]
    assert item["config"]["walkers"] == 4096
    rec = solve(RunConfig(**item["config"])).to_json_dict()
    rec.pop("wall_time_s")
    assert json.dumps(rec) == json.dumps(item["record"])


def test_config1_records_all_100_seeds(setup, golden_config_records):
    items = [r for r in golden_config_records["records"] if r["config"]["L"] == 27]
    assert len(items) == 100
    for item in items:
        rec = solve(RunConfig(**item["config"])).to_json_dict()
        rec.pop("wall_time_s")
        assert json.dumps(rec) == json.dumps(item["record"]), item["config"]
        assert rec["best_E"] == 37


def test_optima_43_55_match_reference(golden_optima_43_55):
    for row in golden_optima_43_55["optima"]:
        rec, half = exhaustive_optimum(row["L"])
        assert rec.E == row["E"], row
        assert encode(half) == row["hex"], row


@pytest.mark.parametrize("L", [55, 57])
def test_full_scan_matches_threaded_oracle(oracle, L):
    # independent full enumeration on the host (all cores) vs the device scan
    assert tuple(int(x) for x in _kernels.exhaustive_scan(L)) == oracle.exhaustive_scan_threaded(L)
