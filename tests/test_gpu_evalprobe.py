"""The walk kernels' evaluator at its exactness bounds (-m gpu).

Random walks keep |C_k| small (|C| <= ~55 at L=201), so walk-based parity
tests never drive the production evaluator near the limits its exactness
argument rests on (f16 holds |C_k| <= L-2 exactly, the f32
accumulation of the correlation stays below 2^24).  sk_eval_states runs the
same evaluator instantiation the batch kernel uses for L on caller-given
states -- all +1, all -1, alternating, short periods, the published Table-1
optima and random halves -- and on the chain of states produced by applying
moves (centre, ends, repeats), and each delta vector is compared with the
CPU oracle's all_neighbor_deltas / apply_neighbor (_kernels.py:85-165).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2210_15962_b200 import _kernels, _lib  # noqa: E402
from paper_2210_15962_b200.codec import decode  # noqa: E402
from paper_2210_15962_b200.published import BEST_KNOWN  # noqa: E402

LENGTHS = [3, 5, 27, 63, 65, 101, 129, 171, 201, 223, 247, 253, 255, 257, 301, 385, 449, 511, 513, 769, 1021, 1023]


@pytest.fixture(params=[_lib.VARIANT_FAST, _lib.VARIANT_SCALAR], ids=["fast", "scalar"])
def variant(request):
    _lib.set_variant(request.param)
    yield request.param
    _lib.set_variant(_lib.VARIANT_AUTO)


def extreme_halves(L, rng):
    d = (L + 1) // 2
    i = np.arange(d)
    pats = [np.ones(d), -np.ones(d), np.where(i % 2 == 0, 1, -1), np.where(i % 3 == 2, -1, 1),
            np.where((i // 2) % 2 == 0, 1, -1), np.where(i % 4 == 3, -1, 1), np.where(i < d // 2, 1, -1)]
    # skew expansion of the all-ones half alternates the tail; these make the
    # FULL sequence (anti)periodic instead, which maximises many |C_k|
    pats.append(np.where((i + (d - 1)) % 2 == 0, 1, -1))
    for row in BEST_KNOWN:
        if row.L == L:
            pats.append(decode(row.hex, L))
    for _ in range(4):
        pats.append(rng.choice([-1, 1], size=d))
    return np.array(pats, dtype=np.int8)


def moves_for(L, S, M, rng):
    d = (L + 1) // 2
    base = [d - 1, 0, d - 1, d - 2 if d > 1 else 0, 0, 1 % d, (d - 1) // 2]
    out = np.empty((S, M), np.int32)
    for s in range(S):
        seq = list(base) + list(rng.integers(0, d, size=M - len(base)))
        out[s] = np.array(seq[:M]) % d
    return out


def oracle_rows(oracle, L, half, moves):
    s, c, _ = oracle.init_state(L, half.astype(np.int64))
    rows = [oracle.all_neighbor_deltas(L, s, c)]
    for h in moves:
        oracle.apply_neighbor(L, s, c, int(h))
        rows.append(oracle.all_neighbor_deltas(L, s, c))
    return np.stack(rows)


@pytest.mark.parametrize("L", LENGTHS)
def test_extreme_states_and_move_chains(variant, oracle, L):
    rng = np.random.default_rng(L)
    halves = extreme_halves(L, rng)
    M = 16
    moves = moves_for(L, halves.shape[0], M, rng)
    got = _kernels.eval_states(L, halves, moves)
    assert got.shape == (halves.shape[0], M + 1, (L + 1) // 2)
    for i in range(halves.shape[0]):
        want = oracle_rows(oracle, L, halves[i], moves[i])
        np.testing.assert_array_equal(got[i], want, err_msg=f"L={L} state {i}")


def test_bounds_are_exercised(oracle):
    # the probe's states reach |C_k| >= L - 3 and |delta| > 2^16, the regime
    # the walk tests never see
    L = 1023
    halves = extreme_halves(L, np.random.default_rng(0))
    cmax = dmax = 0
    for h in halves:
        s, c, _ = oracle.init_state(L, h.astype(np.int64))
        cmax = max(cmax, int(np.abs(c[1:]).max()))
        dmax = max(dmax, int(np.abs(oracle.all_neighbor_deltas(L, s, c)).max()))
    assert cmax >= L - 3
    assert dmax > 1 << 16


def test_many_states_one_launch(oracle):
    # more states than resident warps: the persistent loop
    L = 201
    rng = np.random.default_rng(5)
    S = 3000
    halves = rng.choice([-1, 1], size=(S, 101)).astype(np.int8)
    moves = rng.integers(0, 101, size=(S, 3)).astype(np.int32)
    got = _kernels.eval_states(L, halves, moves)
    for i in rng.choice(S, size=40, replace=False):
        np.testing.assert_array_equal(got[i], oracle_rows(oracle, L, halves[i], moves[i]))


def test_probe_rejects_bad_input():
    with pytest.raises(ValueError):
        _kernels.eval_states(27, np.zeros((2, 14), np.int8))
    with pytest.raises(ValueError):
        _kernels.eval_states(27, np.ones((2, 14), np.int8), np.full((2, 1), 14))
    with pytest.raises(_lib.SokolError):
        _kernels.eval_states(1025, np.ones((1, 513), np.int8))
