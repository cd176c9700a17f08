"""Host emulation of EvalTC's shared-memory layout and fragment algebra.

Mirrors paper_2210_15962_b200/csrc/eval_tc.cuh byte for byte: the Q records,
the two G copies, the parity-split f16 spin copies, S2 and the int8 sequence
live in one bytearray per walk; every lane's MMA fragments are gathered from
it with the kernel's own address arithmetic and multiplied out, the keys are
formed exactly as the epilogue does, and moves go through the same scattered
stores.  Used to check the layout (and by tests/test_tc_layout.py) without a
GPU; the device is checked against the oracle by the -m gpu suite.
"""

from __future__ import annotations

import numpy as np

H = np.float16


class Geom:
    def __init__(self, L):
        self.L = L
        self.D = (L + 1) // 2
        self.K = self.D - 1
        self.NI = (self.D + 15) // 16
        self.MT = (self.NI + 7) // 8
        o = 0
        self.q_off = o
        o += 16 * (8 * self.NI + 56)
        self.ge_off = o + (4 if ((self.K - 3) & 3) == 2 else 0)
        o += 2 * (128 * self.MT + 16) + 16
        o = (o + 15) & ~15
        self.go_off = o + (4 if ((self.K - 3) & 3) == 1 else 0)
        o += 2 * (128 * self.MT + 20) + 16
        o = (o + 15) & ~15
        self.NG = (self.NI + 3) // 4
        ng = (self.NI + 3) // 4
        self.TOFF = max(self.K + 8, 64 * ng + 2)
        self.TOFF += self.TOFF & 1
        self.NT = max(3 * self.K + 20, self.TOFF + self.K // 2 + 64 * ng + 4)
        self.NT += self.NT & 1
        if self.NT % 64 < 8:  # adjacent spin rows on different banks
            self.NT += 8 - self.NT % 64
        elif self.NT % 64 > 56:
            self.NT += 72 - self.NT % 64
        assert 16 <= (2 * self.NT) % 128 <= 112
        self.t_off = o
        o += 8 * self.NT
        self.s2_off = o
        o += 128 * self.MT + 16
        self.bytes = (o + 31) & ~31
        self.span_lo = (L + 8 + 3) & ~3
        self.span_hi = L + 16


def amax(NI, tau):
    return min(8 * tau + 7, NI - 1)


def mlo(NI, tau):
    return -((amax(NI, tau) + 1) >> 1)


def mhi(NI, tau):
    return NI - 4 * tau - 1


HOFF = (0, 2, 1, 3)
VIRTUAL_RK = 0xC0000000 - (1 << 32)  # int32 of 3 * 2^30: padding slots' Rk
KEY_LIMIT = 1 << 30


class Emu:
    """One walk's evaluator state (all 32 lanes)."""

    def __init__(self, L, half):
        g = self.g = Geom(L)
        self.ext = bytearray(g.bytes)
        self.s8 = bytearray(g.span_lo + g.span_hi + 1)
        D, K = g.D, g.K
        s = np.zeros(L, np.int64)
        s[:D] = half
        for i in range(1, D):
            s[D - 1 + i] = (-1) ** i * s[D - 1 - i]
        for x in range(L):
            self.s8[g.span_lo + x] = int(s[x]) & 0xFF
        C = [int(np.dot(s[: L - 2 * j], s[2 * j:])) for j in range(K + 1)]
        for j in range(1, K + 1):
            self.st16(g.ge_off + 16 + 2 * j, H(C[j]))
            self.st16(g.go_off + 18 + 2 * j, H(C[j]))
        for h in range(D):
            self.ext[g.s2_off + h] = (int(s[h]) if h == K else 2 * int(s[h])) & 0xFF
        for x in range(L):
            v = H(s[x])
            pi, i = x & 1, x >> 1
            self.st16(g.t_off + 2 * (2 * pi * g.NT + g.TOFF + i), v)
            self.st16(g.t_off + 2 * ((2 * pi + 1) * g.NT + g.TOFF + 1 + i), v)
            qo = 2 * pi + (i & 1)
            self.st16(g.q_off + 2 * (8 * 32 + 8 * (i >> 1) + qo), v)
            self.st16(g.q_off + 2 * (8 * 32 + 8 * ((i >> 1) - 4) + 4 + qo), v)
        sigma = -1 if (D - 1) & 1 else 1
        self.xq = (512 * sigma, -512 * sigma)
        # per-lane registers
        self.Rk = {}
        self.inv = {}
        for lane in range(32):
            gg, t = lane >> 2, lane & 3
            for tau in range(g.MT):
                h0 = 128 * tau + 16 * gg + 4 * t
                for f in range(4):
                    h = h0 + HOFF[f]
                    live, centre = h < D, h == K
                    r = 0
                    if live and not centre:
                        r = sum(int(s[h - 2 * j]) * int(s[h + 2 * j]) for j in range(1, h // 2 + 1)
                                if h + 2 * j < L)
                    c0 = 16 * ((h >> 1) if centre else (K - 1 - (h & 1)))
                    self.Rk[lane, tau, f] = ((64 * c0 + 2048 * r + (1 << 29) + h
                                              + (2 * self.xq[f >= 2] if centre else 0)) if live else VIRTUAL_RK)
                    self.inv[lane, tau, f] = not live
        self.cq = {}
        for lane in range(32):
            for r in range(g.NG):
                for u in range(2):
                    j = 64 * r + 2 * lane + u
                    self.cq[lane, r, u] = H(C[j] if 1 <= j <= K else 0)

    # byte-level access ------------------------------------------------------
    def st16(self, off, v):
        self.ext[off:off + 2] = np.array([v], H).tobytes()

    def ld16(self, off):
        return np.frombuffer(bytes(self.ext[off:off + 2]), H)[0]

    def s8v(self, pos):
        b = self.s8[self.g.span_lo + pos]
        return b - 256 if b > 127 else b

    def s2v(self, h):
        b = self.ext[self.g.s2_off + h]
        return b - 256 if b > 127 else b

    # G copies, addressed like the kernel (G(0) at ge_off + 16 / go_off + 18)
    def gpair(self, x, copy):
        base = self.g.ge_off + 16 if copy == 0 else self.g.go_off + 18
        off = base + 2 * x
        assert off % 4 == 0, (x, copy)
        return float(self.ld16(off)), float(self.ld16(off + 2))

    def evaluate(self):
        return self.mma_full()

    def mma_full(self):
        """Gather the full 16x16 A and 16x8 B tiles from the 32 lanes' fragments,
        multiply, and scatter D back to the lanes (the mma.sync semantics)."""
        g = self.g
        D = g.D
        out = np.zeros(D, np.int64)
        keys = {}
        for tau in range(g.MT):
            Y = np.zeros((2, 16, 8))  # two accumulator chains
            for m in range(-(g.NI >> 1), g.NI):
                if not (mlo(g.NI, tau) <= m <= mhi(g.NI, tau)):
                    continue
                A = np.zeros((16, 16))
                B = np.zeros((16, 8))
                for lane in range(32):
                    gg, t = lane >> 2, lane & 3
                    rec = g.q_off + 16 * (32 + 32 * tau + 4 * gg + 8 * m + t)
                    a = [float(self.ld16(rec + 2 * k)) for k in range(8)]
                    A[gg, 2 * t], A[gg, 2 * t + 1] = a[0], a[1]
                    A[gg + 8, 2 * t], A[gg + 8, 2 * t + 1] = a[2], a[3]
                    A[gg, 2 * t + 8], A[gg, 2 * t + 9] = a[4], a[5]
                    A[gg + 8, 2 * t + 8], A[gg + 8, 2 * t + 9] = a[6], a[7]
                    x0 = 2 * t - gg
                    own, oth = (1 if gg & 1 else 0), (0 if gg & 1 else 1)
                    x = 16 * m + x0
                    if x >= 0:
                        b0 = self.gpair(x, own)
                    else:
                        p = self.gpair(-x - 1, oth)
                        b0 = (p[1], p[0])
                    if x + 8 >= 0:
                        b1 = self.gpair(x + 8, own)
                    else:
                        p = self.gpair(-x - 9, oth)
                        b1 = (p[1], p[0])
                    B[2 * t, gg], B[2 * t + 1, gg] = b0
                    B[2 * t + 8, gg], B[2 * t + 9, gg] = b1
                Y[(m + (g.NI >> 1)) & 1] += A @ B
            for lane in range(32):
                gg, t = lane >> 2, lane & 3
                h0 = 128 * tau + 16 * gg + 4 * t
                padl = h0 > g.K
                h0a = (g.K & ~3) if padl else h0
                frag = [(gg, 2 * t), (gg, 2 * t + 1), (gg + 8, 2 * t), (gg + 8, 2 * t + 1)]
                copy = 1 if (g.K + 1) & 1 else 0
                y0 = (-8 + ((g.K - 3) & 3)) if padl else g.K - h0a - 3  # padding lanes: zero cells
                assert ((g.go_off + 18 if copy else g.ge_off + 16) + 2 * y0) % 8 == 0  # one LDS.64
                p1 = self.gpair(y0, copy)
                p2 = self.gpair(y0 + 2, copy)
                cx = [int(p2[1]), int(p1[1]), int(p2[0]), int(p1[0])]
                for f in range(4):
                    r, c = frag[f]
                    X = int(Y[0, r, c] + Y[1, r, c])
                    ho = HOFF[f]
                    sx = self.s8v(3 * (h0a + ho) - 2 * g.K)
                    sh = self.s2v(h0 + ho)  # padding lanes: zero cells h >= D
                    xq = self.xq[f >= 2]
                    k = self.Rk[lane, tau, f] + xq * cx[f] + sh * (-256 * X + (-2 * xq) * sx)
                    if not self.inv[lane, tau, f]:
                        out[h0 + ho] = (k - (1 << 29) - (h0 + ho)) >> 6
                        assert 0 < k < KEY_LIMIT
                    else:  # a padding slot's key is exactly its Rk, never a candidate
                        assert k == self.Rk[lane, tau, f] and (k & 0xFFFFFFFF) >= KEY_LIMIT
                    keys[lane, tau, f] = k
        return out

    def apply(self, hs):
        g = self.g
        L, K = g.L, g.K
        p, q = hs, L - 1 - hs
        centre = p == q
        sp, sq = self.s8v(p), self.s8v(q)
        # zero pass
        for x in {p, q}:
            self.s8[g.span_lo + x] = 0
            pi, i = x & 1, x >> 1
            self.st16(g.t_off + 2 * (2 * pi * g.NT + g.TOFF + i), H(0))
            self.st16(g.t_off + 2 * ((2 * pi + 1) * g.NT + g.TOFF + 1 + i), H(0))
        P1, pi, par = p >> 1, p & 1, (p >> 1) & 1
        scale = H(-2 * sp if centre else -4 * sp)
        ua = g.t_off + 2 * (g.NT * (2 * pi + par) + P1 + g.TOFF + par)
        ub = g.t_off + 2 * (g.NT * (2 * pi + 1 - par) + P1 - 1 + g.TOFF + 1 - par)
        for lane in range(32):
            for r in range(g.NG):
                j0 = 64 * r + 2 * lane  # every lane, unpredicated: past K the pair stays 0
                aa, ab = ua + 2 * j0, ub - 2 * j0
                assert aa % 4 == 0 and ab % 4 == 0
                for a in (aa, ab):  # inside the row
                    row = (a - g.t_off) // (2 * g.NT)
                    assert 0 <= row < 4 and (a + 2 - g.t_off) // (2 * g.NT) == row
                A = (self.ld16(aa), self.ld16(aa + 2))
                B = (self.ld16(ab), self.ld16(ab + 2))
                v = [A[0] + B[1], A[1] + B[0]]
                for u in range(2):
                    self.cq[lane, r, u] = H(float(v[u]) * float(scale) + float(self.cq[lane, r, u]))
                    assert j0 + u <= K or float(self.cq[lane, r, u]) == 0.0
                assert (g.ge_off + 16 + 2 * j0) % 4 == 0 and (g.go_off + 18 + 2 * j0) % 4 == 2
                for u in range(2):
                    self.st16(g.ge_off + 16 + 2 * (j0 + u), self.cq[lane, r, u])
                    self.st16(g.go_off + 18 + 2 * (j0 + u), self.cq[lane, r, u])
        wp, wq = -4096 * sp, (0 if centre else -4096 * sq)
        for lane in range(32):
            gg, t = lane >> 2, lane & 3
            for tau in range(g.MT):
                h0 = 128 * tau + 16 * gg + 4 * t
                h0a = h0 if h0 <= K else (K & ~3)
                base = 2 * h0a + 2 * pi
                vp0, vp1 = self.s8v(base - p), self.s8v(base + 4 - p)
                vq0, vq1 = self.s8v(base - q), self.s8v(base + 4 - q)
                f0 = 0 if pi == 0 else 2
                self.Rk[lane, tau, f0] += wp * vp0 + wq * vq0
                self.Rk[lane, tau, f0 + 1] += wp * vp1 + wq * vq1
        # final pass
        for x, sxo in ((p, sp), (q, sq)):
            self.s8[g.span_lo + x] = (-sxo) & 0xFF
            v = H(-sxo)
            pi2, i = x & 1, x >> 1
            self.st16(g.t_off + 2 * (2 * pi2 * g.NT + g.TOFF + i), v)
            self.st16(g.t_off + 2 * ((2 * pi2 + 1) * g.NT + g.TOFF + 1 + i), v)
            qo = 2 * pi2 + (i & 1)
            self.st16(g.q_off + 2 * (8 * 32 + 8 * (i >> 1) + qo), v)
            self.st16(g.q_off + 2 * (8 * 32 + 8 * ((i >> 1) - 4) + 4 + qo), v)
        self.ext[g.s2_off + p] = (-sp if centre else -2 * sp) & 0xFF


def check_geometry(L):
    """The layout properties EvalTC relies on, for every lane, tile, lag pair and
    move at length L (vectorised; the emulator above exercises them on data):
    disjoint regions, the epilogue's C_{q-p} quad one aligned 8-byte load, the
    move's unclamped spin reads inside their row and past K on zero cells, the
    C stores inside the G copies, adjacent spin rows on different banks."""
    g = Geom(L)
    K, NG, MT, NT, TOFF = g.K, g.NG, g.MT, g.NT, g.TOFF
    regions = [(g.q_off, 16 * (8 * g.NI + 56)), (g.ge_off, 2 * (128 * MT + 16)), (g.go_off, 2 * (128 * MT + 20)),
               (g.t_off, 8 * NT), (g.s2_off, 128 * MT + 16)]
    for (a, n), (b, _) in zip(regions, regions[1:]):
        assert a + n <= b, (L, a, n, b)
    assert regions[-1][0] + regions[-1][1] <= g.bytes
    assert 16 <= (2 * NT) % 128 <= 112, (L, NT)  # adjacent spin rows start on different banks
    # epilogue: G(K - 3 - h0 .. K - h0) (zero cells y0 in [-8, -5] for padding lanes), one aligned LDS.64
    h0 = (128 * np.arange(MT)[:, None] + 16 * (np.arange(32) >> 2) + 4 * (np.arange(32) & 3)).ravel()
    y0 = np.where(h0 > K, -8 + ((K - 3) & 3), K - h0 - 3)
    base = g.go_off + 18 if (K + 1) & 1 else g.ge_off + 16
    assert np.all((base + 2 * y0) % 8 == 0), L
    # the move: lag pair j = 64 r + 2 lane, every lane, unpredicated
    p = np.arange(K + 1)[:, None, None]
    lane = np.arange(32)[None, :, None]
    r = np.arange(NG)[None, None, :]
    j = 64 * r + 2 * lane
    P1, pi = p >> 1, p & 1
    par = P1 & 1
    ia = P1 + TOFF + par + j  # row 2 pi + par: (T[ia], T[ia + 1])
    ib = P1 - 1 + TOFF + 1 - par - j  # row 2 pi + 1 - par: (T[ib], T[ib + 1])
    for idx, row_par in ((ia, par), (ib, 1 - par)):
        assert idx.min() >= 0 and idx.max() + 1 < NT, (L, idx.min(), idx.max(), NT)
        # position held by row (pi, shift) at index I: x = 2 (I - TOFF - shift) + pi
        for off in (0, 1):
            x = 2 * (idx + off - TOFF - row_par) + pi
            far = (j + off > K) if idx is ia else (j + 1 - off > K)
            inside = (x >= 0) & (x < L)
            assert not np.any(far & inside), L
    # the C stores: G(j), G(j + 1) in both copies, inside their regions
    jmax = 64 * NG - 1
    assert g.ge_off + 16 + 2 * jmax + 2 <= g.ge_off + 2 * (128 * MT + 16)
    assert g.go_off + 18 + 2 * jmax + 2 <= g.go_off + 2 * (128 * MT + 20)
    return g
