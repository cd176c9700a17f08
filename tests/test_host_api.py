"""Host side of the drop-in API (no GPU): types, validation, codec, seeds,
record format, summary decoding -- checked against the reference's goldens
and its own test expectations (test_runner.py, test_saw.py, test_codec.py)."""

import json

import numpy as np
import pytest

from paper_2210_15962_b200 import _kernels, codec, core, engine
from paper_2210_15962_b200.runner import (
    RunConfig,
    RunRecord,
    SampleSet,
    derive_repetition_seed,
    derive_walk_seed,
)
from paper_2210_15962_b200.saw import WalkConfig, half_to_words, key, words_to_half

RECORD_KEYS = {
    "L", "walkers", "walk_factor", "master_seed", "max_nses", "max_runtime_s", "target_E",
    "best_E", "best_F", "best_hex", "total_nses", "batches", "wall_time_s", "stop_reason",
}


def test_run_config_validation():
    for kw in (dict(L=8, max_nses=10), dict(L=21), dict(L=21, walkers=0, max_nses=10),
               dict(L=21, walk_factor=0, max_nses=10), dict(L=21, max_nses=0),
               dict(L=21, max_runtime=0), dict(L=21, master_seed=-1, max_nses=5),
               dict(L=21, master_seed=2**64, max_nses=5)):
        with pytest.raises(ValueError):
            RunConfig(**kw)
    cfg = RunConfig(L=21, max_nses=10)
    assert cfg.walkers >= 1 and cfg.n == 88 and cfg.D == 11


def test_walk_config_validation():
    for kw in (dict(L=8, n=10, seed=0), dict(L=1, n=10, seed=0), dict(L=5, n=0, seed=0),
               dict(L=5, n=10, seed=-1), dict(L=5, n=10, seed=2**64)):
        with pytest.raises(ValueError):
            WalkConfig(**kw)


def test_seed_derivation_golden(golden_seeds_keys):
    for row in golden_seeds_keys["walk_seeds"]:
        assert derive_walk_seed(int(row["master"]), row["batch"], row["walker"]) == int(row["seed"])
    for row in golden_seeds_keys["rep_seeds"]:
        assert derive_repetition_seed(int(row["master"]), row["rep"]) == int(row["seed"])
    seen = {derive_walk_seed(1, b, w) for b in range(50) for w in range(50)}
    assert len(seen) == 2500


def test_key_golden(golden_seeds_keys):
    for row in golden_seeds_keys["keys"]:
        half = codec.unpack_half(int(row["hex"], 16), row["D"])
        assert key(half) == int(row["key"])


def test_codec_round_trip_and_examples():
    assert codec.encode([1, 1, 1]) == "0x0"
    assert codec.encode([-1, 1, 1]) == "0x4"
    rng = np.random.default_rng(3)
    for _ in range(50):
        d = int(rng.integers(1, 200))
        half = rng.choice([-1, 1], size=d)
        L = 2 * d - 1
        assert np.array_equal(codec.decode(codec.encode(half), L), half)
        w = half_to_words(half)
        assert np.array_equal(words_to_half(w, d), half)
        assert sum(int(x) << (64 * i) for i, x in enumerate(w)) == codec.pack_half(half)
    with pytest.raises(codec.DecodeError):
        codec.decode("0xFF", 5)
    with pytest.raises(codec.DecodeError):
        codec.decode("zz", 5)
    with pytest.raises(codec.DecodeError):
        codec.decode("0x1", 4)


def test_energy_of_published_rows():
    # PAPER Table 1 rows (skewsaw/published.py); pins host energy + decode
    rows = [(171, 1669, "0x07F018C27F3C01849035B3"), (193, 2040, "0x020C18D1A749035A04EFECC5A"),
            (247, 3259, "0x3FF9FE03FE31FDEC1870F23887276E5")]
    for L, E, hx in rows:
        assert core.energy(core.expand_skew(codec.decode(hx, L))).E == E


def test_mix64_and_key_host():
    assert _kernels.mix64(0) == 0
    assert int(_kernels.key_of_words(np.array([0], np.uint64))) == _kernels.mix64(_kernels.KEY_SEED)


def test_record_json_keys_and_float():
    cfg = RunConfig(L=21, walkers=4, master_seed=7, target_E=26, max_nses=10**6)
    rec = RunRecord(cfg, 26, core.merit_factor(21, 26), np.ones(11, np.int64), "0x356", 3520, 1, 0.5,
                    "target_reached")
    d = json.loads(rec.to_json())
    assert set(d) == RECORD_KEYS
    assert d["best_F"] == 21 * 21 / 52.0


def test_sample_set_csv():
    s = SampleSet(L=15, nses=[100, 250, 75], censored=[False, True, False])
    text = s.to_csv()
    assert text.splitlines()[0] == "L,repetition,nses,censored"
    assert text.splitlines()[2] == "15,1,250,1"
    back = SampleSet.from_csv(text)
    assert (back.L, back.nses, back.censored, back.uncensored) == (15, s.nses, s.censored, [100, 75])
    for bad, line in (("bogus,header\n", "line 1"), ("L,repetition,nses,censored\n15,0,10,0\n15,1,x,0\n", "line 3"),
                      ("L,repetition,nses,censored\n15,0,10,7\n", "line 2"), ("L,repetition,nses,censored\n", "line 2")):
        with pytest.raises(ValueError, match=line):
            SampleSet.from_csv(bad)


def test_decode_summary_and_slices():
    raw = np.zeros(10, np.uint64)
    raw[0] = (np.uint64(906) << np.uint64(32)) | np.uint64(17)
    raw[1] = 408 * 3
    raw[2] = 0xDEADBEEF
    r = engine.decode_summary(raw, 1)
    assert (r.best_E, r.walker, r.steps_sum, int(r.best_words[0])) == (906, 17, 1224, 0xDEADBEEF)
    raw[0] = np.uint64(2**64 - 1)
    assert engine.decode_summary(raw, 1) is None
    sl = engine._slices(10, 4)
    assert sl == [(0, 3), (3, 3), (6, 2), (8, 2)]
    assert sum(c for _, c in engine._slices(2**20, 8)) == 2**20
