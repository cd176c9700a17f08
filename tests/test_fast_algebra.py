"""CPU model of the tensor-core evaluator's algebra (eval_fast.cuh), checked
against the oracle's reference-formula deltas along real walks.

The model reproduces the kernel's decomposition exactly: the block-Toeplitz
product Y = sum_m A_m B_m with A_m[b][d] = G(16m + d - b) and
B_m[d][n] = S_pi(n)[16(a(n)+m) + d] (in float32, like the MMA's f32
accumulator), the per-neighbour corrections, and the O(1) incremental update
of R_h after every move.  If this passes, a GPU mismatch is a fragment /
addressing bug, not an algebra bug.
"""

import numpy as np
import pytest


def geom(L):
    D = (L + 1) // 2
    hmax = (D - 1) >> 1
    NB = hmax // 16 + 1
    NI = (D + 15) // 16
    NT = (2 * NB + 7) // 8
    return D, NB, NI, NT


def correlations(L, s, ce):
    """X[h] for all h via the kernel's block-Toeplitz formulation (float32)."""
    D, NB, NI, NT = geom(L)
    K = D - 1
    Gx = {}

    def G(d):
        d = abs(d)
        return 0 if d == 0 or d > K else ce[d]

    S = [np.zeros(16 * (NI + 2 * NB + 2), np.float32) for _ in range(2)]
    pad = 16 * NB
    for i in range(D):
        S[0][pad + i] = s[2 * i]
        if i < D - 1:
            S[1][pad + i] = s[2 * i + 1]
    Y = np.zeros((16, 8 * NT), np.float32)
    for m in range(-(NB - 1), NI):
        A = np.array([[G(16 * m + d - b) for d in range(16)] for b in range(16)], np.float32)
        B = np.zeros((16, 8 * NT), np.float32)
        for n in range(8 * NT):
            pi, a = divmod(n, NB)
            if pi < 2:
                for d in range(16):
                    B[d, n] = S[pi][pad + 16 * (a + m) + d]
        Y += A @ B
    X = {}
    for n in range(2 * NB):
        pi, a = divmod(n, NB)
        for b in range(16):
            h = 2 * (16 * a + b) + pi
            if h < D:
                X[h] = int(Y[b, n])
    return X


def deltas_model(L, s, ce, R):
    D = (L + 1) // 2
    K = D - 1
    X = correlations(L, s, ce)
    out = np.zeros(D, np.int64)
    for h in range(D):
        sp = s[h]
        if h == K:
            out[h] = 16 * (h >> 1) - 4 * sp * X[h]
            continue
        sq = -sp if (D - 1 - h) & 1 else sp
        assert sq == s[L - 1 - h]
        sx = s[3 * h - 2 * K] if 3 * h - 2 * K >= 0 else 0
        v2 = (K - 1 - (h & 1)) + 2 * R[h] - 2 * sx * sq
        out[h] = 16 * v2 - 8 * sp * (X[h] - sq * ce[K - h])
    return out


def r_init(L, s):
    D = (L + 1) // 2
    R = np.zeros(D, np.int64)
    for h in range(D - 1):
        R[h] = sum(s[h - 2 * j] * s[h + 2 * j] for j in range(1, (h >> 1) + 1))
    return R


def r_update(L, s, R, p):
    """Kernel's O(1)-per-neighbour update, s = sequence BEFORE the flip."""
    D = (L + 1) // 2
    K = D - 1
    q = L - 1 - p
    for h in range(K):
        if (h ^ p) & 1:
            continue
        if p != h and 2 * h - p >= 0:
            R[h] -= 2 * s[p] * s[2 * h - p]
        if p != q and 2 * h - q >= 0:
            R[h] -= 2 * s[q] * s[2 * h - q]


@pytest.mark.parametrize("L", [3, 5, 7, 9, 13, 21, 27, 31, 63, 65, 101, 129, 201, 257, 301])
def test_model_matches_oracle_along_walk(oracle, L):
    D = (L + 1) // 2
    steps = 12 if L > 200 else 40
    seed = 12345 + L
    be, st, dead, bw, tw, td = oracle.saw_walk(L, steps, seed, record=True)
    for t in range(st + (1 if dead else 0)):
        v = sum(int(w) << (64 * i) for i, w in enumerate(tw[t]))
        half = np.array([-1 if (v >> (D - 1 - h)) & 1 else 1 for h in range(D)], np.int64)
        s, c, _ = oracle.init_state(L, half)
        ce = {j: int(c[2 * j]) for j in range(1, D)}
        if t == 0:
            R = r_init(L, s)
        else:
            np.testing.assert_array_equal(R, r_init(L, s))  # incremental == from scratch
        got = deltas_model(L, s, ce, R)
        np.testing.assert_array_equal(got, td[t], err_msg=f"L={L} step {t}")
        if t < st:
            v2 = sum(int(w) << (64 * i) for i, w in enumerate(tw[t + 1]))
            hs = [h for h in range(D) if ((v ^ v2) >> (D - 1 - h)) & 1]
            assert len(hs) == 1
            r_update(L, s, R, hs[0])


def test_delta_is_multiple_of_8_and_fits_key(oracle):
    # packing contract of sokol_common.cuh: delta = 8 * (integer), |delta/8| < 2^20
    rng = np.random.default_rng(1)
    for L in (3, 11, 101, 449, 1023):
        D = (L + 1) // 2
        K = D - 1
        for _ in range(3):
            half = rng.choice([-1, 1], size=D)
            s, c, _ = oracle.init_state(L, half)
            d = oracle.all_neighbor_deltas(L, s, c)
            assert np.all(d % 8 == 0)
            assert np.abs(d // 8).max() <= 8 * K + 2 * K * K < 2**20


def test_packed_key_identity():
    # the epilogue accumulates 64*dE + 2^29 + h directly; it must equal the
    # packed selection key ((dE/8 + 2^20) << 9) | h for every reachable dE
    # (multiples of 8, |dE/8| < 2^20) and h < 512, and order (dE, h) pairs
    import random

    rng = random.Random(5)
    keys = []
    for _ in range(20000):
        d8 = rng.randint(-(1 << 20) + 1, (1 << 20) - 1)
        h = rng.randint(0, 511)
        dE = 8 * d8
        a = (64 * dE + (1 << 29) + h) & 0xFFFFFFFF
        b = ((d8 + (1 << 20)) << 9) | h
        assert a == b
        keys.append((a, dE, h))
    keys.sort()
    assert [(k[1], k[2]) for k in keys] == sorted((k[1], k[2]) for k in keys)
