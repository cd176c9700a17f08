"""Batched device neighbourhood API against the
reference: golden compute_deltas cases and compute_deltas/apply_flip chains
produced by the reference itself, the CPU oracle on large random batches
(including non-skew +-1 inputs, which the reference's arithmetic accepts),
and the acceptance criterion-2 identity E + delta_j == E(flip j) at scale."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from conftest import load_json  # noqa: E402

from paper_2210_15962_b200 import _kernels  # noqa: E402
from paper_2210_15962_b200.codec import decode  # noqa: E402
from paper_2210_15962_b200.core import autocorrelations, energy, expand_skew  # noqa: E402
from paper_2210_15962_b200.neighborhood import (  # noqa: E402
    NeighborhoodBatch,
    apply_flip,
    compute_deltas,
    flip,
    naive_oracle,
)


def test_golden_delta_cases(golden_deltas):
    for case in golden_deltas["cases"]:
        st = naive_oracle(decode(case["hex"], case["L"]))
        assert st.E == case["E"]
        np.testing.assert_array_equal(compute_deltas(st), np.array(case["deltas"], np.int64))


def test_golden_chains():
    for ch in load_json("host.json")["neighborhood"]:
        st = naive_oracle(np.array(ch["half"], np.int64))
        assert st.E == ch["E0"]
        for j, dl, e in zip(ch["flips"], ch["deltas"], ch["E"]):
            d = compute_deltas(st)
            np.testing.assert_array_equal(d, np.array(dl, np.int64))
            st = apply_flip(st, j, d)
            assert st.E == e
        np.testing.assert_array_equal(st.sidelobes, np.array(ch["sidelobes_final"], np.int64))


def test_validation():
    st = naive_oracle(np.ones(5, np.int64))
    with pytest.raises(ValueError):
        apply_flip(st, 5, compute_deltas(st))
    with pytest.raises(ValueError):
        flip(st.half, -1)


@pytest.mark.parametrize("L,S", [(3, 64), (27, 1000), (101, 4096), (201, 2048), (449, 512), (1023, 64)])
def test_batch_matches_oracle(oracle, L, S):
    rng = np.random.default_rng(L)
    D = (L + 1) // 2
    halves = np.where(rng.random((S, D)) < 0.5, -1, 1).astype(np.int64)
    nb = NeighborhoodBatch(halves)
    ref = [oracle.init_state(L, h) for h in halves]
    check = rng.choice(S, size=min(S, 48), replace=False)
    for step in range(6):
        got = nb.deltas().cpu().numpy()
        hs = rng.integers(0, D, S)
        for i in check:
            s, c, e = ref[i]
            np.testing.assert_array_equal(got[i], oracle.all_neighbor_deltas(L, s, c))
            ref[i] = (s, c, e + int(got[i][hs[i]]))
            oracle.apply_neighbor(L, s, c, int(hs[i]))
        nb.apply(hs)
    E = nb.E.cpu().numpy()
    full = nb.full.cpu().numpy()
    c_dev = nb.c.cpu().numpy()
    for i in check:
        s, c, e = ref[i]
        np.testing.assert_array_equal(full[i], s)
        np.testing.assert_array_equal(c_dev[i], c)
        assert E[i] == e == energy(s).E


def test_non_skew_inputs_follow_reference_arithmetic(oracle):
    rng = np.random.default_rng(3)
    for L in (5, 31, 99):
        S = 16
        s = np.where(rng.random((S, L)) < 0.5, -1, 1).astype(np.int64)
        c = np.stack([autocorrelations(x) for x in s])
        out = np.empty((S, (L + 1) // 2), np.int64)
        _kernels.all_neighbor_deltas(s, c, out)
        for i in range(S):
            np.testing.assert_array_equal(out[i], oracle.all_neighbor_deltas(L, s[i], c[i]))
        s2, c2 = s.copy(), c.copy()
        hs = rng.integers(0, (L + 1) // 2, S)
        _kernels.apply_neighbor(s2, c2, hs)
        for i in range(S):
            a, b = s[i].copy(), c[i].copy()
            oracle.apply_neighbor(L, a, b, int(hs[i]))
            np.testing.assert_array_equal(s2[i], a)
            np.testing.assert_array_equal(c2[i], b)


def test_criterion2_identity_at_scale():
    # every delta of every state equals the naive energy difference
    rng = np.random.default_rng(2025)
    for L in (21, 63, 125):
        D = (L + 1) // 2
        S = 256
        halves = np.where(rng.random((S, D)) < 0.5, -1, 1).astype(np.int64)
        nb = NeighborhoodBatch(halves)
        d = nb.deltas().cpu().numpy()
        E = nb.E.cpu().numpy()
        for i in range(0, S, 16):
            for j in range(D):
                assert E[i] + d[i, j] == energy(expand_skew(flip(halves[i], j))).E
