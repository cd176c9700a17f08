// eval_fast.cuh -- production neighbourhood evaluator (SK_VARIANT_FAST).
//
// The reference evaluates each neighbour h with an O(L) loop over even lags
// (neighbor_delta, _kernels.py:85-123).  Using skew symmetry the four
// products of each lag collapse to v_k(h) = s_p (s_{p-k} + s_{p+k}[k != q-p])
// and  dE(h) = 16 * sum_k v_k^2 - 8 * sum_k v_k C_k  (exact).
//
// * sum_k v_k C_k = s_p (X_h - s_q C_{q-p}) with X_h = sum_i S_pi[i] G(i-h'),
//   a correlation of the parity-split signal S_pi[i] = s_{2i+pi} with
//   G(d) = C_{2|d|} (G(0) = 0), pi = h&1, h' = h>>1.  All D correlations of a
//   step are one block-Toeplitz matrix product done on the tensor cores with
//   mma.sync.m16n8k16 (f16 x f16 -> f32):  A_m[b][d] = G(16m + d - b) is a
//   16x16 Toeplitz block of G, B_m[d][n] = S_pi(n)[16(a(n)+m) + d] holds the
//   signal, column n = (parity, output block a), row b = offset in the block;
//   Y[b][n] = sum_m A_m B_m = X_{h}, h' = 16a + b.  Every value is a small
//   integer (|C| <= L-2 < 2048, sums < 2^24), so f16 inputs and the f32
//   accumulation are exact -- bit-identical to the int64 reference.
// * sum_k v_k^2 = (K - 1 - pi) + 2 R_h - 2 s_{3h-2K} s_q, with
//   R_h = sum_j s_{h-2j} s_{h+2j} kept per neighbour and updated in O(1) per
//   move (only terms touching the two flipped positions change sign).
// * a move updates C_k -= 4 v_k(h*) for all even k (apply_neighbor,
//   _kernels.py:126-158), rewrites the Toeplitz source G in shared memory and
//   flips two signal entries.
//
// Fragment bookkeeping (PTX ISA m16n8k16 layouts, g = lane>>2, t = lane&3):
//   A regs {a0,a1,a2,a3} = G pairs at x, x-8, x+8, x  with x = 16m + 2t - g,
//   so consecutive m share one pair (2 new LDS.32 per MMA); G is stored twice
//   (shifted by one half) so every pair is a 4-byte aligned load.
//   B regs {b0,b1} = signal pairs at 16(a+m) + 2t + {0, 8}, stored adjacently
//   (sig_perm) so that both come from one LDS.64.
//   D regs {c0..c3} = rows g, g+8 x columns 2t, 2t+1 of each 8-column tile.
#pragma once
#include <cuda_fp16.h>

#include "walk_engine.cuh"

// Blocks per SM the L <= 255 kernels are register-capped for (4 x 128 threads:
// 128 registers; 5: 102).  Chosen by measurement; overridable
// at build time for experiments.
#ifndef SK_MT1_MIN_BLOCKS
#define SK_MT1_MIN_BLOCKS 4
#endif
#ifndef SK_MT2_MIN_BLOCKS
#define SK_MT2_MIN_BLOCKS 3
#endif

namespace sk {

struct FastGeom {
  int NB;    // 16-row output blocks per parity
  int NI;    // 16-wide input blocks
  int NT;    // 8-column MMA tiles (2*NB columns)
  int MLO, MHI;
  int GOFF, GLEN;  // Toeplitz source: index GOFF + d holds G(d); halves per copy
  int SPAD, SLEN;  // signal arrays: index SPAD + i holds S[i]
  uint32_t ext_halves;
};

// The signal arrays start 32-byte aligned (after both G copies), so that each
// 16-element block is one aligned 32-byte unit.
__host__ __device__ inline int sig_off(const FastGeom& g) { return (2 * g.GLEN + 2 + 15) / 16 * 16; }

// Within a 16-element signal block, element u is stored at sig_perm(u): the
// B-fragment elements of lane t (u = 2t, 2t+1, 2t+8, 2t+9) become the four
// consecutive halves 4t..4t+3, loaded with one LDS.64.
__host__ __device__ inline int sig_perm(int u) { return 4 * ((u & 7) >> 1) + 2 * (u >> 3) + (u & 1); }
__host__ __device__ inline int sig_index(int i) { return (i & ~15) + sig_perm(i & 15); }

__host__ __device__ inline FastGeom fast_geom(int L) {
  FastGeom g;
  const int D = (L + 1) / 2;
  const int hmax = (D - 1) >> 1;
  g.NB = hmax / 16 + 1;
  g.NI = (D + 15) / 16;
  g.NT = (2 * g.NB + 7) / 8;
  g.MLO = -(g.NB - 1);
  g.MHI = g.NI - 1;
  g.GOFF = 16 * (g.NB - 1) + 32;
  g.GLEN = g.GOFF + 16 * g.NI + 32;
  g.GLEN = (g.GLEN + 31) / 64 * 64 + 32;  // copy 2 sits 16 banks away from copy 1
  g.SPAD = 16 * (g.NB - 1) + 16;
  g.SLEN = g.SPAD + 16 * (g.NI + g.NB) + 32;
  // S_1 starts 32 bytes (mod 128) after S_0: a half-warp of a B load reads
  // S_0 blocks a, a+2 and S_1 blocks a, a+2 (column map below), which then
  // fall on disjoint banks
  g.SLEN = (g.SLEN + 63) / 64 * 64 + 16;
  // ... + ces (int16 C copy, D entries) + flip table (2 x D uint16 byte offsets)
  g.ext_halves = uint32_t(sig_off(g) + 2 * g.SLEN + ((D + 1) & ~1) + 2 * D);
  return g;
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// MT  : compile-time max number of 8-column tiles (ceil(NW/2) covers every L)
// NMC : compile-time MMA count per step (even), 0 = runtime (G.nm)
template <int MT, int NMC = 0>
struct EvalFast {
  static constexpr int CPL = 4 * MT;  // lags per lane: K <= 128*MT - 1
  FastGeom G;
  __half* ga;           // G copy 1 (pairs at even x aligned)
  __half* gb;           // G copy 2, shifted by one half (pairs at odd x aligned)
  __half* sp0;
  __half* sp1;
  int16_t* ces;         // int16 copy of C_{2j}, read by the epilogue (C_{q-p})
  uint16_t* flipoff;    // [2][D]: byte offset (from sp0) of the signal cell of p = h / q = L-1-h
  uint32_t a_addr;      // shared byte address of this lane's A pair at x0 = 2t - g, m = MLO
  uint32_t b_addr[MT];  // shared byte address of this lane's B pair, m = MLO
  // per accumulator slot (nt, o): neighbour h (clamped to >= 0) and its constants
  // The selection key ((dE/8 + 2^20) << 9) | h equals 64 dE + 2^29 + h, so the
  // epilogue accumulates the key directly (every term pre-scaled by 64):
  //   key = Rk - sx * sq2k - xsp64 * X + xq64 * C_{q-p}
  int hc[MT][4];
  uint32_t inv[MT][4];  // 0 for a live slot, ~0 for padding
  int32_t Rk[MT][4];    // 64*c0 + 2048*R_h + 2^29 + h;  R_h = sum_j s_{h-2j} s_{h+2j},
                        // c0 = 16 (K - 1 - pi)  (16 (h >> 1) at the centre)
  int32_t xsp64[MT][4]; // 64 * xm * s_h  (xm = 8, 4 at the centre, 0 for padding)
  int32_t sq2k[MT][4];  // 2048 * s_{L-1-h} (0 at the centre / padding)
  int32_t xq64[MT][4];  // 64 * xm * s_q s_p (= +-512; 0 at the centre / padding)
  int ridx[MT][4];      // 2h for live non-centre slots; -1 otherwise (R-update reads land in zero padding)
  int lpar;             // parity of every slot of this lane (column map: pi = t & 1)
  uint32_t key[MT][4];
  int32_t ce[CPL];      // C_{2j}, j = 1 + lane + 32 r (lag-owned)

  static uint32_t ext_bytes(int L, int) { return fast_geom(L).ext_halves * 2u; }
  static bool supports(int L) { return L >= 3 && L <= SK_MAX_L; }
  static constexpr bool kNeedsDl = false;
  static constexpr bool kSmemKeysVariant = (MT <= 2);  // L <= 511: built per visited-set layout (compile-time probes)
  static constexpr bool kCeAliasKeys = true;  // C lives in registers + ces16 after init
  static constexpr int kMinBlocks = MT == 1 ? SK_MT1_MIN_BLOCKS : (MT == 2 ? SK_MT2_MIN_BLOCKS : 2);  // register caps chosen by measurement
  // Spin-array margins.  The C update reads s_{p -+ 2j} for every lag slot
  // j <= 32 CPL (idle slots j > K must read zeros, so they need no test), the
  // R update reads down to -1 - q, the epilogue up to p + 2K.  CPL follows L
  // (the tile count of the evaluator the launcher picks for it).
  static int cpl_for(int D) { return 4 * ((((D + 63) / 64) + 1) / 2); }
  static int span_hi(int L, int D) { return L - 1 + max(D - 1, 64 * cpl_for(D)); }
  static int span_lo(int L, int D) { return max(L + 1, 64 * cpl_for(D)); }
  static uint32_t block_bytes(int) { return 0; }  // no per-block table
  __device__ static void block_init(const WalkParams&, char*, int, int) {}
  __device__ __forceinline__ void prefetch(const WalkParams&, int, int) {}  // nothing to prefetch
  __device__ __forceinline__ void renormalize(const WalkParams&, int) {}     // no drifting state

  __device__ __forceinline__ void init(const WalkParams& P, WarpSmem& sm, int8_t* s, int lane) {
    G = fast_geom(P.L);
    const int D = P.D, K = P.K;
    __half* base = reinterpret_cast<__half*>(sm.ext);
    ga = base;
    gb = ga + G.GLEN;
    sp0 = base + sig_off(G);
    sp1 = sp0 + G.SLEN;
    ces = reinterpret_cast<int16_t*>(sp1 + G.SLEN);
    flipoff = reinterpret_cast<uint16_t*>(ces + ((D + 1) & ~1));
    const __half z = __ushort_as_half(0);
    for (uint32_t i = lane; i < G.ext_halves; i += 32) base[i] = z;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < CPL; r++) {
      const int j = 1 + lane + 32 * r;
      ce[r] = j <= K ? sm.ce[j] : 0;
      if (j <= K) {
        write_g(j, ce[r]);
        ces[j] = int16_t(ce[r]);
      }
    }
    for (int i = lane; i < D; i += 32) {
      sp0[sig_index(G.SPAD + i)] = __int2half_rn(s[2 * i]);                     // S_0[i] = s_{2i}
      if (i < D - 1) sp1[sig_index(G.SPAD + i)] = __int2half_rn(s[2 * i + 1]);  // S_1[i] = s_{2i+1}
    }
    for (int i = lane; i < 2 * D; i += 32) {  // position x -> its signal cell, for the flips of a move
      const int h = i < D ? i : i - D;
      const int x = i < D ? h : P.L - 1 - h;
      flipoff[i] = uint16_t(2 * ((x & 1) * G.SLEN + sig_index(G.SPAD + (x >> 1))));
    }
    const int g = lane >> 2, t = lane & 3;
    const int x0 = 2 * t - g + 16 * G.MLO;
    a_addr = uint32_t(__cvta_generic_to_shared((g & 1) ? gb + G.GOFF + 1 + x0 : ga + G.GOFF + x0));
    // Column map: column c of tile nt holds parity pi = (c >> 1) & 1 and
    // output block a = 4 nt + ((c & 7) >> 2) + 2 (c & 1).  A lane's
    // accumulator columns 2t, 2t+1 then share the parity t & 1, so the R
    // update needs no per-slot parity test; and the lanes with t >> 1 = 0, 1
    // sit one block (16 neighbours) apart, so the epilogue's and the R
    // update's scattered spin / C loads avoid bank conflicts.
    lpar = t & 1;
#pragma unroll
    for (int nt = 0; nt < MT; nt++) {
      const int c = 8 * nt + g;
      const int pi = (c >> 1) & 1, a = 4 * nt + ((c & 7) >> 2) + 2 * (c & 1);
      const __half* sb = pi == 1 ? sp1 : sp0;  // columns with a >= NB are padding: any signal will do
      b_addr[nt] = uint32_t(__cvta_generic_to_shared(sb + G.SPAD + (a < G.NB ? 16 * (a + G.MLO) : 0) + 4 * t));
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int cc = 8 * nt + 2 * t + (o & 1);
        const int ppi = (cc >> 1) & 1, aa = 4 * nt + ((cc & 7) >> 2) + 2 * (cc & 1);
        const int hp = 16 * aa + g + 8 * (o >> 1);
        const int h = 2 * hp + ppi;
        const bool ok = nt < G.NT && aa < G.NB && h < D;
        const bool centre = ok && h == K;
        hc[nt][o] = ok ? h : 0;
        inv[nt][o] = ok ? 0u : ~0u;
        int32_t r = 0;
        if (ok && !centre)
          for (int j = 1; j <= hp; j++) r += int32_t(s[h - 2 * j]) * int32_t(s[h + 2 * j]);
        const int32_t sp = ok ? int32_t(s[h]) : 0;
        const int32_t qs = ((D - 1 - h) & 1) ? -1 : 1;  // s_{L-1-h} = qs * s_h (skew symmetry)
        const int32_t c0 = ok ? 16 * (centre ? (h >> 1) : (K - 1 - (h & 1))) : 0;
        Rk[nt][o] = 64 * c0 + 2048 * r + (1 << 29) + (ok ? h : 0);
        xsp64[nt][o] = 64 * (centre ? 4 : 8) * sp;
        sq2k[nt][o] = centre ? 0 : 2048 * qs * sp;
        xq64[nt][o] = (ok && !centre) ? 512 * qs : 0;
        ridx[nt][o] = (ok && !centre) ? 2 * h : -1;
      }
    }
    __syncwarp();
  }

  // G(+j) and G(-j) in both copies.
  __device__ __forceinline__ void write_g(int j, int32_t c) {
    const __half v = __int2half_rn(c);
    ga[G.GOFF + j] = v;
    gb[G.GOFF + 1 + j] = v;
    if (j <= G.GOFF - 2) {
      ga[G.GOFF - j] = v;
      gb[G.GOFF + 1 - j] = v;
    }
  }

  __device__ __forceinline__ void mma_pair(float (&acc)[MT][4], uint32_t aa, const uint32_t (&bb)[MT], uint32_t& pm) {
    const uint32_t p0 = lds32(aa), p1 = lds32(aa + 16u);
#pragma unroll
    for (int nt = 0; nt < MT; nt++)
      if (nt == 0 || nt < G.NT) {
        const uint2 b = lds64(bb[nt]);
        mma16816(acc[nt], p0, pm, p1, p0, b.x, b.y);
      }
    pm = p1;
  }

  __device__ __forceinline__ void evaluate(const WalkParams& P, WarpSmem&, const int8_t* s, int,
                                           int64_t* trace_row) {
    float accA[MT][4], accB[MT][4];
#pragma unroll
    for (int nt = 0; nt < MT; nt++)
#pragma unroll
      for (int o = 0; o < 4; o++) accA[nt][o] = accB[nt][o] = 0.f;

    // Y = sum_m A_m B_m; A pairs roll along m (pair x-8 of step m is pair x+8 of m-1).
    // The MMA count is padded to even; the extra block reads zero signal.
    uint32_t aa = a_addr, bb[MT];
#pragma unroll
    for (int nt = 0; nt < MT; nt++) bb[nt] = b_addr[nt];
    uint32_t pm = lds32(aa - 16u);
    if (NMC > 0) {
#pragma unroll
      for (int i = 0; i < NMC; i += 2) {
        mma_pair(accA, aa, bb, pm);
#pragma unroll
        for (int nt = 0; nt < MT; nt++) bb[nt] += 32u;
        mma_pair(accB, aa + 32u, bb, pm);
        aa += 64u;
#pragma unroll
        for (int nt = 0; nt < MT; nt++) bb[nt] += 32u;
      }
    } else {
      const int nm = G.MHI - G.MLO + 1;
      for (int i = 0; i < nm; i += 2) {
        mma_pair(accA, aa, bb, pm);
#pragma unroll
        for (int nt = 0; nt < MT; nt++) bb[nt] += 32u;
        mma_pair(accB, aa + 32u, bb, pm);
        aa += 64u;
#pragma unroll
        for (int nt = 0; nt < MT; nt++) bb[nt] += 32u;
      }
    }

    // dE(h) = 16 (c0 + 2R - 2 s_x s_q) - xm s_p (X - s_q C_{q-p})   (see header),
    // accumulated as key = 64 dE + 2^29 + h
    const int K = P.K;
    const int8_t* sx0 = s - 2 * K;   // sx0[3h] = s_{3h-2K} = s_{p-(q-p)} (zero padded)
    const int16_t* cx0 = ces + K;    // cx0[-h] = C_{q-p}
#pragma unroll
    for (int nt = 0; nt < MT; nt++) {
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int h = hc[nt][o];
        const int32_t X = __float2int_rn(accA[nt][o] + accB[nt][o]);
        const int32_t cx = cx0[-h];
        const int32_t sx = sx0[3 * h];
        const int32_t k = Rk[nt][o] - sx * sq2k[nt][o] - xsp64[nt][o] * X + xq64[nt][o] * cx;
        if (trace_row && !inv[nt][o]) trace_row[h] = (k - (1 << 29) - h) >> 6;
        key[nt][o] = uint32_t(k) | inv[nt][o];
      }
    }
  }

  __device__ __forceinline__ uint32_t local_min() const {
    uint32_t m = kNoCand;
#pragma unroll
    for (int nt = 0; nt < MT; nt++)
#pragma unroll
      for (int o = 0; o < 4; o++) m = min(m, key[nt][o]);
    return m;
  }

  __device__ __forceinline__ void exclude(int h, int) {
#pragma unroll
    for (int nt = 0; nt < MT; nt++)
#pragma unroll
      for (int o = 0; o < 4; o++)
        if (hc[nt][o] == h) key[nt][o] = kNoCand;
  }

  __device__ __forceinline__ void apply(const WalkParams& P, WarpSmem&, int8_t* s, int hs, int lane) {
    const int L = P.L, K = P.K;
    const int p = hs, q = L - 1 - hs;
    const bool centre = (p == q);
    const int32_t sp = s[p];
    const int32_t sq = s[q];
    const int csh = centre ? 1 : 0;      // centre: s_{p+k} = s_{p-k}, so v = (sum) / 2
    const int32_t nsp4 = -4 * sp;
    // s_p and s_q are zeroed for the duration of the update (they are
    // overwritten with -s_p, -s_q below).  Then the lag k = q - p, whose
    // s_{p+k} = s_q term is excluded, needs no test, and neither does the R
    // update's own-slot term s_p s_{2h-p} at h = p.
    __syncwarp();
    if (lane < 2) s[lane ? q : p] = 0;
    __syncwarp();
    // C_k -= 4 v_k(h*) for every even lag (apply_neighbor, _kernels.py:126-158);
    // lags with v_k = 0 leave C_k and its copies untouched
#pragma unroll
    for (int r = 0; r < CPL; r++) {
      const int j = 1 + lane + 32 * r;
      const int k = 2 * j;  // idle slots (j > K) read the zero margins: v = 0
      const int32_t a = s[p - k];
      const int32_t b = s[p + k];
      const int32_t v = (a + b) >> csh;
      if constexpr (MT >= 2) {
        // unconditional: a lag with v = 0 rewrites its unchanged value (no
        // branch); measured faster for two tiles, slower for one
        ce[r] += nsp4 * v;
        if (j <= K) {
          ces[j] = int16_t(ce[r]);
          write_g(j, ce[r]);
        }
      } else if (v != 0) {
        ce[r] += nsp4 * v;
        ces[j] = int16_t(ce[r]);
        write_g(j, ce[r]);
      }
    }
    // R_h: the terms s_x s_{2h-x} with x in {p, q} change sign (same-parity,
    // live, non-centre slots).  Out-of-range partners read the zero padding,
    // the own-slot pair (x = h = p) reads the zeroed s_p, and a centre move
    // flips only x = p.  A flip of h itself negates s_h and s_{L-1-h}.
    // Centre and padding slots have ridx = -1, so both reads hit the zero
    // padding below position 0; other-parity lanes get zero weights.
    const bool same = (lpar == (p & 1));
    const int32_t sp4k = same ? 4096 * sp : 0, sq4k = (same && !centre) ? 4096 * sq : 0;
#pragma unroll
    for (int nt = 0; nt < MT; nt++) {
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int h = hc[nt][o];
        const bool own = (h == p);  // padding slots have xsp64 = sq2k = 0: negating them is harmless
        const int32_t v1 = s[ridx[nt][o] - p];
        const int32_t v2 = s[ridx[nt][o] - q];
        Rk[nt][o] -= sp4k * v1 + sq4k * v2;
        xsp64[nt][o] = own ? -xsp64[nt][o] : xsp64[nt][o];
        sq2k[nt][o] = own ? -sq2k[nt][o] : sq2k[nt][o];
      }
    }
    __syncwarp();
    if (lane < (centre ? 1 : 2)) {  // lane 0 flips p, lane 1 flips q
      const int x = lane ? q : p;
      const int32_t sx = lane ? sq : sp;
      s[x] = int8_t(-sx);
      const uint16_t half_bits = sx > 0 ? 0xBC00u : 0x3C00u;  // f16 of -sx
      if constexpr (MT == 1) {  // table lookup (measured faster for MT = 1, slower for MT = 2)
        *reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(sp0) + flipoff[lane * P.D + p]) = half_bits;
      } else {
        reinterpret_cast<uint16_t*>((x & 1) ? sp1 : sp0)[sig_index(G.SPAD + (x >> 1))] = half_bits;
      }
    }
    __syncwarp();
  }
};

}  // namespace sk
