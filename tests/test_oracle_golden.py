"""Pin the CPU oracle (oracle/sokol_oracle.c) to the real reference.

Every fixture under tests/golden/ is output of /root/reference's own code
(oracle/gen_golden.py).  Once these pass, the oracle may stand in for the
reference on the GPU box, where /root/reference does not exist.
"""

import hashlib

import numpy as np
import pytest


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def half_from_hex(hx, d):
    v = int(hx, 16)
    return np.array([-1 if (v >> (d - 1 - h)) & 1 else 1 for h in range(d)], dtype=np.int64)


def words_of_half(half):
    v = 0
    for s in half:
        v = (v << 1) | int(s < 0)
    nw = -(-len(half) // 64)
    return np.array([(v >> (64 * i)) & (2**64 - 1) for i in range(nw)], dtype=np.uint64)


def pivots_from_words(tw, d):
    return np.stack([half_from_hex(hex(sum(int(w) << (64 * i) for i, w in enumerate(row))), d) for row in tw])


def test_seeds(oracle, golden_seeds_keys):
    for row in golden_seeds_keys["walk_seeds"]:
        assert oracle.derive_walk_seed(int(row["master"]), row["batch"], row["walker"]) == int(row["seed"])
    for row in golden_seeds_keys["rep_seeds"]:
        assert oracle.derive_repetition_seed(int(row["master"]), row["rep"]) == int(row["seed"])


def test_keys(oracle, golden_seeds_keys):
    for row in golden_seeds_keys["keys"]:
        half = half_from_hex(row["hex"], row["D"])
        assert oracle.key_of_words(words_of_half(half)) == int(row["key"])


def test_neighbour_deltas(oracle, golden_deltas):
    for case in golden_deltas["cases"]:
        L = case["L"]
        half = half_from_hex(case["hex"], (L + 1) // 2)
        s, c, e = oracle.init_state(L, half)
        assert e == case["E"]
        assert oracle.all_neighbor_deltas(L, s, c).tolist() == case["deltas"]


def test_traces(oracle, golden_traces):
    meta, arrays = golden_traces
    for w in meta["walks"]:
        L, seed, n = w["L"], int(w["seed"]), w["n"]
        d = (L + 1) // 2
        be, st, dead, bw, tw, td = oracle.saw_walk(L, n, seed, record=True)
        assert (be, st, dead) == (w["best_E"], w["steps"], w["dead"]), (L, seed)
        assert "0x" + format(sum(int(x) << (64 * i) for i, x in enumerate(bw)), f"0{-(-d // 4)}X") == w["best_hex"]
        piv = pivots_from_words(tw[: st + 1], d).astype(np.int8)
        rows = st + (1 if dead else 0)
        deltas = td[:rows]
        key = f"L{L}_s{seed}_pivots"
        if key in arrays:
            np.testing.assert_array_equal(piv, arrays[key])
            np.testing.assert_array_equal(deltas, arrays[f"L{L}_s{seed}_deltas"].astype(np.int64))
        if "sha_pivots_i8" in w:
            assert sha(piv) == w["sha_pivots_i8"]
            assert sha(deltas.astype(np.int64)) == w["sha_deltas_i64"]


def test_batches(oracle, golden_batches):
    meta, arrays = golden_batches
    for b in meta["batches"]:
        seeds = oracle.derive_walk_seeds(b["master"], b["batch"], b["W"])
        be, bw, st, dd = oracle.batch_outputs(b["L"], b["n"], seeds)
        t = b["tag"]
        np.testing.assert_array_equal(be, arrays[t + "_best_e"])
        np.testing.assert_array_equal(bw, arrays[t + "_best_words"])
        np.testing.assert_array_equal(st, arrays[t + "_steps"])
        np.testing.assert_array_equal(dd, arrays[t + "_dead"])


def test_run_records(oracle, golden_records):
    for item in golden_records["records"]:
        cfg = dict(item["config"])
        got = oracle.solve_record(
            cfg["L"], cfg["walkers"], cfg.get("walk_factor", 8), cfg["master_seed"],
            cfg.get("max_nses"), cfg.get("target_E"),
        )
        assert got == item["record"], cfg


def test_exhaustive_optima(oracle, golden_optima):
    for row in golden_optima["optima"]:
        if row["L"] > 33:
            continue  # keep the CPU suite fast; larger rows are pinned on the GPU box
        e, bits = oracle.exhaustive_scan(row["L"])
        assert e == row["E"]


def test_thread_count_independence(oracle):
    seeds = oracle.derive_walk_seeds(5, 2, 64)
    a = oracle.batch_outputs(45, 8 * 23, seeds, threads=1)
    b = oracle.batch_outputs(45, 8 * 23, seeds, threads=0)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("L,seed", [(3, 5)])
def test_dead_end_tiny_space(oracle, L, seed):
    # test_saw.py:111-116: L=3 walk dies after 3 steps with best E = 1
    be, st, dead, *_ = oracle.saw_walk(L, 8 * 2, seed)
    assert (be, st, dead) == (1, 3, True)


def test_exhaustive_range_slices_compose(oracle):
    # the slice scan used as the device checker composes to the full scan
    for L in (9, 21, 27):
        D = (L + 1) // 2
        total = 1 << D
        e_all, bits = oracle.exhaustive_scan(L)
        cuts = [0, 1, total // 3, total // 2 + 5, total]
        parts = [oracle.exhaustive_range(L, a, b - a) for a, b in zip(cuts, cuts[1:])]
        e, g = min(parts)
        assert e == e_all and g ^ (g >> 1) == bits
        assert oracle.exhaustive_range(L, 0, total) == (e, g)


# ---- BASELINE configs 1 and 2 (fixtures: oracle/gen_golden_r2.py) ----------
def test_config2_traces(oracle, golden_config2_traces):
    # run_walk_traced for derive_walk_seed(1, 0, w), w < 64, at L=101
    g = golden_config2_traces
    L, n = g["L"], g["n"]
    d = (L + 1) // 2
    assert len(g["walks"]) == 64
    for w in g["walks"]:
        seed = oracle.derive_walk_seed(g["master"], g["batch"], w["w"])
        assert seed == int(w["seed"])
        be, st, dead, bw, tw, td = oracle.saw_walk(L, n, seed, record=True)
        assert (be, st, dead) == (w["best_E"], w["steps"], w["dead"]), w["w"]
        piv = pivots_from_words(tw[: st + 1], d).astype(np.int8)
        deltas = td[: st + (1 if dead else 0)]
        assert sha(piv) == w["sha_pivots_i8"], w["w"]
        assert sha(deltas.astype(np.int64)) == w["sha_deltas_i64"], w["w"]


def test_config_records(oracle, golden_config_records):
    # config 2's RunRecord (L=101, 4096 walkers, 2 batches) and config 1's
    # records for all 100 master seeds at L=27 (target 37)
    recs = golden_config_records["records"]
    assert sum(1 for r in recs if r["config"]["L"] == 27) == 100
    for item in recs:
        cfg = item["config"]
        got = oracle.solve_record(cfg["L"], cfg["walkers"], 8, cfg["master_seed"], cfg.get("max_nses"),
                                  cfg.get("target_E"))
        assert got == item["record"], cfg
        if cfg["L"] == 27:
            assert got["best_E"] == 37 and got["stop_reason"] == "target_reached"


def test_optima_43_55_small_rows(oracle, golden_optima_43_55):
    # the reference's exhaustive optima L=43..55; the CPU suite scans the two
    # smallest rows, the GPU suite checks all of them (device + threaded oracle)
    rows = {r["L"]: r for r in golden_optima_43_55["optima"]}
    assert sorted(rows) == list(range(43, 56, 2))
    for L in (43, 45):
        e, bits = oracle.exhaustive_scan(L)
        assert e == rows[L]["E"]
        d = (L + 1) // 2
        code = sum(1 << (d - 1 - h) for h in range(d) if (bits >> h) & 1)  # codec bit order
        assert "0x" + format(code, f"0{-(-d // 4)}X") == rows[L]["hex"]


def test_threaded_scan_equals_full_scan(oracle):
    # the threaded slice scan the GPU suite uses as the L=55/59 checker
    for L in (21, 31, 33):
        assert oracle.exhaustive_scan_threaded(L, threads=4, slices=13) == oracle.exhaustive_scan(L), L
