"""Bit-exact parity of the CUDA walk engine with the reference (-m gpu).

Three anchors, strongest first:
  1. golden fixtures produced by the reference itself (tests/golden/);
  2. the CPU oracle (oracle/sokol_oracle.c, pinned to 1 by
     test_oracle_golden.py) on fresh seeded inputs at many lengths;
  3. size-independent properties at BASELINE sizes (L=201, 2^16+ walks):
     summary == min over per-walk outputs, best energies re-derived from
     the returned sequences, device-derived seeds == host-derived seeds.
Both evaluators (SK_VARIANT_SCALAR, SK_VARIANT_FAST) must agree with all.
"""

import hashlib
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2210_15962_b200 import _kernels, _lib, core, engine  # noqa: E402
from paper_2210_15962_b200.runner import RunConfig, derive_walk_seed, solve  # noqa: E402
from paper_2210_15962_b200.saw import WalkConfig, run_walk, run_walk_traced, words_to_half  # noqa: E402

VARIANTS = [_lib.VARIANT_SCALAR, _lib.VARIANT_FAST]


# (evaluator, visited-set layout): both evaluators, and the production
# evaluator with each global-key layout forced (AUTO picks shared-memory keys
# for most lengths)
SETUPS = [(_lib.VARIANT_SCALAR, _lib.VISITED_AUTO), (_lib.VARIANT_FAST, _lib.VISITED_AUTO),
          (_lib.VARIANT_FAST, _lib.VISITED_FINGERPRINT), (_lib.VARIANT_FAST, _lib.VISITED_GLOBAL)]


@pytest.fixture(params=SETUPS, ids=["scalar", "fast", "fast_fp", "fast_gk"])
def variant(request):
    old = _lib.get_variant()
    ev, layout = request.param
    _lib.set_variant(ev)
    _lib.set_visited_layout(layout)
    yield ev
    _lib.set_variant(old)
    _lib.set_visited_layout(_lib.VISITED_AUTO)


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def gpu_batch(L, n, seeds):
    d = (L + 1) // 2
    nw = (d + 63) // 64
    W = len(seeds)
    be = np.empty(W, np.int64)
    bw = np.empty((W, nw), np.uint64)
    st = np.empty(W, np.int64)
    dd = np.empty(W, np.uint8)
    _kernels.saw_batch(L, n, np.asarray(seeds, np.uint64), be, bw, st, dd)
    return be, bw, st, dd


# --------------------------------------------------------------- goldens --
def test_traces_match_reference_goldens(variant, golden_traces):
    meta, arrays = golden_traces
    for w in meta["walks"]:
        L, seed, n = w["L"], int(w["seed"]), w["n"]
        res, tr = run_walk_traced(WalkConfig(L=L, n=n, seed=seed))
        assert (res.best_E, res.steps_taken, res.dead_end) == (w["best_E"], w["steps"], w["dead"]), (L, seed)
        assert core.energy(core.expand_skew(res.best_half)).E == res.best_E
        from paper_2210_15962_b200.codec import encode

        assert encode(res.best_half) == w["best_hex"]
        piv = tr.pivots.astype(np.int8)
        key = f"L{L}_s{seed}_pivots"
        if key in arrays:
            np.testing.assert_array_equal(piv, arrays[key])
            np.testing.assert_array_equal(tr.deltas, arrays[f"L{L}_s{seed}_deltas"].astype(np.int64))
        if "sha_pivots_i8" in w:
            assert sha(piv) == w["sha_pivots_i8"], (L, seed)
            assert sha(tr.deltas.astype(np.int64)) == w["sha_deltas_i64"], (L, seed)


def test_batches_match_reference_goldens(variant, golden_batches):
    meta, arrays = golden_batches
    for b in meta["batches"]:
        seeds = [derive_walk_seed(b["master"], b["batch"], w) for w in range(b["W"])]
        be, bw, st, dd = gpu_batch(b["L"], b["n"], seeds)
        t = b["tag"]
        np.testing.assert_array_equal(be, arrays[t + "_best_e"], err_msg=t)
        np.testing.assert_array_equal(bw, arrays[t + "_best_words"], err_msg=t)
        np.testing.assert_array_equal(st, arrays[t + "_steps"], err_msg=t)
        np.testing.assert_array_equal(dd, arrays[t + "_dead"], err_msg=t)


def test_run_records_match_reference_goldens(variant, golden_records):
    for item in golden_records["records"]:
        rec = solve(RunConfig(**item["config"])).to_json_dict()
        rec.pop("wall_time_s")
        assert json.dumps(rec) == json.dumps(item["record"]), item["config"]


# ---------------------------------------------------------------- oracle --
@pytest.mark.parametrize("L", [3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31, 33, 35, 37, 39, 41,
                               45, 53, 61, 63, 65, 67, 75, 99, 101, 127, 129, 131, 161, 201])
def test_batch_matches_oracle(variant, oracle, L):
    d = (L + 1) // 2
    W = 96 if L < 150 else 32
    n = 8 * d
    seeds = oracle.derive_walk_seeds(1000 + L, 3, W)
    got = gpu_batch(L, n, seeds)
    want = oracle.batch_outputs(L, n, seeds)
    for g, x, name in zip(got, want, ("best_e", "best_words", "steps", "dead")):
        np.testing.assert_array_equal(g, x, err_msg=f"L={L} {name}")


@pytest.mark.parametrize("L,factor", [(21, 1), (21, 40), (27, 3), (101, 2), (301, 1), (449, 1), (511, 1), (1023, 1)])
def test_walk_factors_and_large_lengths_match_oracle(variant, oracle, L, factor):
    d = (L + 1) // 2
    n = factor * d
    W = 8 if L > 300 else 48
    seeds = oracle.derive_walk_seeds(77, L, W)
    got = gpu_batch(L, n, seeds)
    want = oracle.batch_outputs(L, n, seeds)
    for g, x in zip(got, want):
        np.testing.assert_array_equal(g, x, err_msg=f"L={L} n={n}")


@pytest.mark.parametrize("L", [223, 253, 255, 257, 259, 383, 385, 511, 513, 769])
def test_tile_and_word_boundaries_match_oracle(variant, oracle, L):
    # D = 128 / 129 (one -> two 8-column tiles), nw = 2 / 3 / 4 / 5 / 7 words,
    # at the production walk factor 8
    d = (L + 1) // 2
    n = 8 * d
    W = 8 if L > 500 else 16
    seeds = oracle.derive_walk_seeds(4242, L, W)
    got = gpu_batch(L, n, seeds)
    want = oracle.batch_outputs(L, n, seeds)
    for g, x, name in zip(got, want, ("best_e", "best_words", "steps", "dead")):
        np.testing.assert_array_equal(g, x, err_msg=f"L={L} {name}")


@pytest.mark.parametrize("L", [5, 9, 15, 21, 31, 47, 101, 149, 201])
def test_traces_match_oracle(variant, oracle, L):
    d = (L + 1) // 2
    for s in range(4):
        seed = derive_walk_seed(9, L, s)
        be, st, dead, bw, tw, td = oracle.saw_walk(L, 8 * d, seed, record=True)
        res, tr = run_walk_traced(WalkConfig(L=L, n=8 * d, seed=seed))
        assert (res.best_E, res.steps_taken, res.dead_end) == (be, st, dead)
        np.testing.assert_array_equal(tr.deltas, td[: st + (1 if dead else 0)])
        np.testing.assert_array_equal(tr.pivots, np.stack([words_to_half(r, d) for r in tw[: st + 1]]))


def test_dead_end_tiny_space(variant):
    res, tr = run_walk_traced(WalkConfig(L=3, n=16, seed=5))
    assert res.dead_end and res.steps_taken == 3 and res.best_E == 1
    assert tr.deltas.shape == (4, 2)


def test_scalar_and_fast_traces_identical():
    L, d = 201, 101
    out = {}
    for v in VARIANTS:
        _lib.set_variant(v)
        out[v] = [run_walk_traced(WalkConfig(L=L, n=8 * d, seed=derive_walk_seed(4, 0, w))) for w in range(3)]
    _lib.set_variant(_lib.VARIANT_AUTO)
    for (ra, ta), (rb, tb) in zip(out[VARIANTS[0]], out[VARIANTS[1]]):
        assert ra.best_E == rb.best_E
        np.testing.assert_array_equal(ta.deltas, tb.deltas)
        np.testing.assert_array_equal(ta.pivots, tb.pivots)


# --------------------------------------------------- full-size properties --
def device_batch(L, n, master, batch, W, begin=0):
    d = (L + 1) // 2
    nw = (d + 63) // 64
    dev = torch.device("cuda")
    be = torch.empty(W, dtype=torch.int64, device=dev)
    bw = torch.empty((W, nw), dtype=torch.int64, device=dev)
    st = torch.empty(W, dtype=torch.int64, device=dev)
    dd = torch.empty(W, dtype=torch.uint8, device=dev)
    summ = torch.empty(engine.SUMMARY_WORDS, dtype=torch.int64, device=dev)
    lib = _lib.load()
    _lib.check(lib.sk_saw_batch(L, n, None, master, batch, begin, W, be.data_ptr(), bw.data_ptr(), st.data_ptr(),
                                dd.data_ptr(), summ.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return (be.cpu().numpy(), bw.cpu().numpy().view(np.uint64), st.cpu().numpy(), dd.cpu().numpy(),
            engine.decode_summary(summ.cpu().numpy().view(np.uint64), nw))


def test_device_seeds_equal_host_seeds(variant):
    L, W = 101, 300
    n = 8 * 51
    a = device_batch(L, n, 5, 2, W, begin=1000)
    seeds = [derive_walk_seed(5, 2, 1000 + w) for w in range(W)]
    b = gpu_batch(L, n, seeds)
    for x, y in zip(a[:4], b):
        np.testing.assert_array_equal(x, y)


def test_summary_is_min_over_walks_at_full_size(variant):
    L, W = 201, 1 << 16
    d = 101
    be, bw, st, dd, summ = device_batch(L, 8 * d, 1, 0, W)
    w = int(np.lexsort((np.arange(W), be))[0])
    assert (summ.best_E, summ.walker) == (int(be[w]), w)
    np.testing.assert_array_equal(summ.best_words, bw[w])
    assert summ.steps_sum == int(st.sum())
    assert np.all(st[dd == 0] == 8 * d)
    # the returned best sequences have the returned energies (naive O(L^2) check)
    rng = np.random.default_rng(0)
    for i in rng.choice(W, size=64, replace=False):
        half = words_to_half(bw[i], d)
        assert core.energy(core.expand_skew(half)).E == be[i]


def test_sharded_batch_equals_whole_batch(variant):
    L, W = 129, 4096
    n = 8 * 65
    whole = device_batch(L, n, 8, 1, W)
    parts = [device_batch(L, n, 8, 1, c, begin=b) for b, c in engine._slices(W, 3)]
    for k in range(4):
        np.testing.assert_array_equal(whole[k], np.concatenate([p[k] for p in parts]))
    best = min((p[4] for p in parts), key=lambda r: (r.best_E, r.walker))
    assert (best.best_E, best.walker) == (whole[4].best_E, whole[4].walker)


def test_l27_recovery_config1(variant):
    # BASELINE config 1: RunConfig(L=27, W=8, m=s, target_E=37, max_nses=1e6), s < 100
    for s in range(100):
        rec = solve(RunConfig(L=27, walkers=8, master_seed=s, target_E=37, max_nses=10**6))
        assert rec.best_E == 37 and rec.stop_reason == "target_reached", s


def test_never_below_exhaustive_optimum(variant, golden_optima):
    for row in golden_optima["optima"]:
        L = row["L"]
        if L < 9:
            continue
        d = (L + 1) // 2
        be, *_ = gpu_batch(L, 8 * d, [derive_walk_seed(2, 0, w) for w in range(256)])
        assert be.min() >= row["E"]


def test_unsupported_length_raises():
    with pytest.raises(_lib.SokolError):
        run_walk(WalkConfig(L=1025, n=10, seed=1))
