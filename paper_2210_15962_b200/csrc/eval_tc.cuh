// eval_tc.cuh -- production neighbourhood evaluator (SK_VARIANT_FAST), every L <= SK_MAX_L.
//
// Same exact arithmetic as the reference's neighbor_delta / apply_neighbor
// (_kernels.py:85-158), restated for one warp per walk:
//
//   dE(h) = 16 (c0 + 2 R_h - 2 s_x s_q) - xm s_p (X_h - s_q C_{q-p}),
//   X_h   = sum_i T_pi[i] G(i - h'),   T_pi[i] = s_{2i+pi},  G(d) = C_{2|d|},
//   p = h, q = L-1-h, pi = h & 1, h' = h >> 1, x = 3h - 2K, xm = 8 (4 at the centre).
//
// The correlation X_h of all D neighbours is one block-Toeplitz product on the
// tensor cores (mma.sync.m16n8k16, f16 x f16 -> f32, exact: every operand is
// a small integer, |C| <= L - 2 < 2048 and every partial sum < 2^24), laid out
// so that each MMA costs four instructions:
//
//   A (16 x 16, the SIGNAL): row g <-> (pi = 0, block a = 8 tau + g),
//     row g + 8 <-> (pi = 1, same a); A_m[row][k] = T_pi[8a + 16m + k].
//     The four A registers of lane (g, t) are one 16-byte "Q record"
//     {T0[e], T0[e+1], T1[e], T1[e+1], T0[e+8], T0[e+9], T1[e+8], T1[e+9]},
//     e = 8a + 16m + 2t: ONE LDS.128, no register moves.
//   B (16 x 8, the TOEPLITZ source): B_m[k][c] = G(16m + k - c), i.e. the
//     pairs (G(x), G(x+1)) and (G(x+8), G(x+9)), x = 16m + 2t - g: two LDS.32
//     from one of two copies of G (even- / odd-aligned pairs); x < 0 reads the
//     mirrored pair and swaps its halves (G(-d) = G(d)).
//   D: lane (g, t) holds the four CONSECUTIVE neighbours h0 + {0, 2, 1, 3},
//     h0 = 128 tau + 16 g + 4 t, so the epilogue's per-neighbour operands
//     (C_{q-p}, s_x, s_h) come from a few vector loads.
//
// A move (apply_neighbor, _kernels.py:126-158): every lane owns two
// consecutive lags per 64 (j0 = 64 r + 2 l): C_{2j} -= 4 s_p v_j(h*) with
// v_j = s_{p-2j} + s_{p+2j} (the flipped positions p, q read as zero, which
// removes the excluded lag q - p and the own lag j = 0), computed as one
// HADD2 + one HFMA2 on a half2 register from parity-split f16 spin arrays
// (two shifted copies, so every spin pair is one aligned LDS.32), then
// stored to both G copies.  Consecutive lanes touch consecutive 4-byte words,
// so none of these accesses has a bank conflict (a quad per lane, 8-byte
// lane stride, costs two wavefronts per 4-byte access).
// R_h (sum_j s_{h-2j} s_{h+2j}) changes in O(1) per neighbour.  Then 11 scattered cells (int8 sequence, f16 spin copies,
// Q records, S2) take the flipped spins: two predicated stores.
//
// Padding slots (h >= D) have no mask: their operands read zero cells, so
// their key is their Rk (kVirtualRk, kept above every real key; see below).
#pragma once
#include <cuda_fp16.h>

#include "walk_engine.cuh"

// Blocks per SM (4 warps each) the one- / two- / three-or-four-tile kernels
// are register-capped for (__maxnreg__, walk_engine.cuh); measured
// (DESIGN.md §4), overridable at build time for experiments.
#ifndef SK_TC_MIN_BLOCKS1
#define SK_TC_MIN_BLOCKS1 5
#endif
#ifndef SK_TC_MIN_BLOCKS2
#define SK_TC_MIN_BLOCKS2 4
#endif
#ifndef SK_TC_MIN_BLOCKS4
#define SK_TC_MIN_BLOCKS4 2
#endif
// Independent HMMA accumulator chains per tile (2: alternate k-blocks and add
// at the end; 1: one dependent chain, no FADD).
#ifndef SK_TC_CHAINS
#define SK_TC_CHAINS 2
#endif

namespace sk {

#ifndef SK_TC_MAX_L
#define SK_TC_MAX_L 1023
#endif
// Rk of a padding slot (h >= D).  Its S2 and C_{q-p} read zero cells, so its
// key is its Rk, which the R update moves by at most 8192 per step: from
// 3 * 2^30 it stays in [2^30, 2^32) for kRenormSteps = 2^16 steps, i.e. above
// every real key (< kKeyLimit = 2^30), and renormalize() resets it.
constexpr int32_t kVirtualRk = int32_t(0xC0000000u);
constexpr int kTcMaxL = SK_TC_MAX_L;  // = SK_MAX_L: D <= 512, up to four 128-neighbour tiles

// Byte offsets inside the evaluator's shared-memory area (host and device).
struct TcGeom {
  int D, K, NI, MT;
  int NT, TOFF;       // f16 spin arrays: NT halves each, index i at TOFF + i (+1 in the odd-aligned copy);
                      // cells outside the sequence are zero
  uint32_t q_off;     // Q records: record r in [-32, 8 NI + 24) at q_off + 16 (r + 32)
  uint32_t ge_off;    // G(y), y in [-8, 128 MT + 8): even-aligned copy at ge_off + 2 (y + 8)
  uint32_t go_off;    //                               odd-aligned copy at go_off + 2 (y + 9)
                      // (each 4 bytes past a 16-byte boundary where that makes the epilogue's
                      // C_{q-p} quad, G(K - 3 - h0 .. K - h0), 8-byte aligned)
  uint32_t t_off;     // [TA_0 | TB_0 | TA_1 | TB_1]: TA_pi[i] at +2 (i + TOFF), TB_pi[i] at +2 (i + TOFF + 1)
  uint32_t s2_off;    // int8 S2[h] = 2 s_h (s_h at the centre h = K), h < D; 0 beyond
  uint32_t bytes;
};

__host__ __device__ inline TcGeom tc_geom(int L) {
  TcGeom g;
  g.D = (L + 1) / 2;
  g.K = g.D - 1;
  g.NI = (g.D + 15) / 16;
  g.MT = (g.NI + 7) / 8;
  uint32_t o = 0;
  g.q_off = o;
  o += 16u * uint32_t(8 * g.NI + 56);
  g.ge_off = o + (((g.K - 3) & 3) == 2 ? 4u : 0u);
  o += 2u * uint32_t(128 * g.MT + 16) + 16u;
  o = (o + 15u) & ~15u;
  g.go_off = o + (((g.K - 3) & 3) == 1 ? 4u : 0u);
  o += 2u * uint32_t(128 * g.MT + 20) + 16u;
  o = (o + 15u) & ~15u;
  // the move's lag pairs j < 64 NG (NG = ceil(NI / 4)) read T_pi at P1 +- j
  // without clamping: past K they read zero cells, so v_j = 0 there
  const int ng = (g.NI + 3) / 4;
  g.TOFF = g.K + 8 > 64 * ng + 2 ? g.K + 8 : 64 * ng + 2;
  g.TOFF += g.TOFF & 1;
  g.NT = 3 * g.K + 20 > g.TOFF + g.K / 2 + 64 * ng + 4 ? 3 * g.K + 20 : g.TOFF + g.K / 2 + 64 * ng + 4;
  g.NT += g.NT & 1;
  // rows 2 NT bytes apart must not land on the same bank: the move's flip
  // stores write TA_pi[i] and TB_pi[i] (adjacent rows) in one instruction
  if ((g.NT & 63) < 8) g.NT += 8 - (g.NT & 63);
  else if ((g.NT & 63) > 56) g.NT += 72 - (g.NT & 63);
  g.t_off = o;
  o += 8u * uint32_t(g.NT);
  g.s2_off = o;
  o += 128u * uint32_t(g.MT) + 16u;
  g.bytes = (o + 31u) & ~31u;
  return g;
}

// Shared-memory accesses by address (the layout is computed, not typed).  The
// "memory" clobbers order them against the C++ stores of init() and of the
// walk engine: an asm without one may be scheduled across ordinary stores.
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld64s(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld32s(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int32_t lds8(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
// Predicated stores (one ISETP + @P STS, no divergent branch).
__device__ __forceinline__ void sts8_if(bool c, uint32_t a, int32_t v) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p st.shared.s8 [%0], %1; }" ::"r"(a), "r"(v), "r"(int(c))
               : "memory");
}
__device__ __forceinline__ void sts16_if(bool c, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p st.shared.b16 [%0], %1; }" ::"r"(a), "h"(uint16_t(v)),
               "r"(int(c))
               : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(uint16_t(v)) : "memory");
}
__device__ __forceinline__ void sts32_if(bool c, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p st.shared.b32 [%0], %1; }" ::"r"(a), "r"(v), "r"(int(c))
               : "memory");
}
// v if a != b else ~0 (a SEL; a plain ternary on an unrolled constant b can
// become a jump table)
__device__ __forceinline__ uint32_t mask_if_eq(uint32_t v, int a, int b) {
  uint32_t r;
  asm("{ .reg .pred p; setp.eq.s32 p, %1, %2; selp.b32 %0, -1, %3, p; }" : "=r"(r) : "r"(a), "r"(b), "r"(v));
  return r;
}
__device__ __forceinline__ void mma_tc(float (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
// Makes a value opaque to the compiler: per-walk constants set up once in
// init() stay in registers instead of being recomputed inside the step loop.
__device__ __forceinline__ void pin(uint32_t& v) { asm volatile("" : "+r"(v)); }
__device__ __forceinline__ void pin(int32_t& v) { asm volatile("" : "+r"(v)); }
// Byte B of x, sign-extended (one PRMT: the selector's bit 3 replicates the
// sign; __byte_perm masks that bit off, so this is inline PTX).
__device__ __forceinline__ int32_t sext_byte(uint32_t x, int b) {
  int32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"(b | ((b | 8) << 4) | ((b | 8) << 8) | ((b | 8) << 12)));
  return r;
}
__device__ __forceinline__ uint32_t h2u(__half2 v) { return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ __half2 u2h(uint32_t v) { return *reinterpret_cast<__half2*>(&v); }

// NI = ceil(D / 16), compile time: every loop bound and MMA count below is a
// constant (one instantiation per 16 lengths).
template <int NI>
struct EvalTC {
  static constexpr int MT = (NI + 7) / 8;  // 128-neighbour tiles
  static constexpr int NG = (NI + 3) / 4;  // lag pairs per lane (K < 64 NG)
  static constexpr int M_LO = -(NI >> 1);  // k-blocks of the product
  static constexpr int M_HI = NI - 1;
  __host__ __device__ static constexpr int amax(int tau) { return (8 * tau + 7 < NI - 1) ? 8 * tau + 7 : NI - 1; }
  __host__ __device__ static constexpr int mlo(int tau) { return -((amax(tau) + 1) >> 1); }
  __host__ __device__ static constexpr int mhi(int tau) { return NI - 4 * tau - 1; }
  // D-fragment register f <-> neighbour h0 + hoff(f)
  __host__ __device__ static constexpr int hoff(int f) { return f == 1 ? 2 : (f == 2 ? 1 : f); }

  // per-lane state
  uint32_t qbase;           // this lane's Q record for tau = 0, m = 0
  uint32_t b_pos, b_neg;    // B pair addresses at x0 = 2t - g (own-parity copy) / at -x0-1 (other copy)
  uint32_t b_m0;            // m = 0 pair: b_pos if x0 >= 0 else b_neg (then swapped)
  uint32_t sel_m0;          // byte_perm selector for it
  uint32_t cxb[MT], sxb[MT], shb[MT], r2b[MT];  // epilogue / R-update bases per tile
  int32_t Rk[MT][4];
  uint32_t key[MT][4];
  int32_t h0[MT];
  int32_t xq_e, xq_o;       // 512 qs for the even / odd neighbours of a lane (qs = (-1)^(D-1-h))
  int32_t m2xq_e, m2xq_o;   // -2 xq
  __half2 cq[NG];           // C_{2j}, j = j0, j0 + 1, j0 = 64 r + 2 lane (lag-owned)
  // move-role constants (lanes 0..10): address = fb + f4 (x>>2) + 2 ((x>>1)&1) + f1 (x&1)
  uint32_t fb, f4, f1;
  uint32_t t_base, s8_a;    // shared addresses
  uint32_t ge_l, go_l;      // G(2 lane) in the even / odd copy

  static uint32_t ext_bytes(int L, int) { return tc_geom(L).bytes; }
  // No per-block table and no prefetch: both were measured (a table of the
  // per-move window offsets and flip-cell offsets, loaded before the probe):
  // +2% at L=301, -1.4% at L=201, so the addresses are computed.
  static uint32_t block_bytes(int) { return 0; }
  __device__ static void block_init(const WalkParams&, char*, int, int) {}
  __device__ __forceinline__ void prefetch(const WalkParams&, int, int) {}
  static bool supports(int L) { return L >= 3 && L <= kTcMaxL; }
  static constexpr bool kNeedsDl = false;
  static constexpr bool kSmemKeysVariant = MT <= 2;  // per-layout kernels only where they pay (L <= 511)
  static constexpr bool kCeAliasKeys = true;
  static constexpr int kMinBlocks = MT == 1 ? SK_TC_MIN_BLOCKS1 : (MT == 2 ? SK_TC_MIN_BLOCKS2 : SK_TC_MIN_BLOCKS4);
  // s8 reads: R update 2h - x in [-(L-1), 2K + 12], s_{3h-2K} in [-2K, K + 18],
  // position 0 kept 4-byte aligned (the s_h quad is one LDS.32)
  static int span_lo(int L, int) { return (L + 8 + 3) & ~3; }
  static int span_hi(int L, int) { return L + 16; }

  __device__ __forceinline__ void init(const WalkParams& P, WarpSmem& sm, int8_t* s, int lane) {
    const TcGeom G = tc_geom(P.L);
    const int D = P.D, K = P.K;
    char* ext = reinterpret_cast<char*>(sm.ext);
    const uint32_t ext_a = uint32_t(__cvta_generic_to_shared(ext));
    for (uint32_t i = lane; i < G.bytes / 16u; i += 32) reinterpret_cast<uint4*>(ext)[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    __half* ge = reinterpret_cast<__half*>(ext + G.ge_off) + 8;
    __half* go = reinterpret_cast<__half*>(ext + G.go_off) + 9;
    for (int j = 1 + lane; j <= K; j += 32) {
      const __half v = __int2half_rn(sm.ce[j]);
      ge[j] = v;
      go[j] = v;
    }
    __half* ta = reinterpret_cast<__half*>(ext + G.t_off);
    __half* q = reinterpret_cast<__half*>(ext + G.q_off) + 8 * 32;
    int8_t* s2 = reinterpret_cast<int8_t*>(ext + G.s2_off);
    for (int h = lane; h < D; h += 32) s2[h] = int8_t(h == K ? s[h] : 2 * s[h]);
    for (int x = lane; x < P.L; x += 32) {
      const __half v = __int2half_rn(s[x]);
      const int pi = x & 1, i = x >> 1;
      ta[2 * pi * G.NT + G.TOFF + i] = v;
      ta[(2 * pi + 1) * G.NT + G.TOFF + 1 + i] = v;
      const int qo = 2 * pi + (i & 1);
      q[8 * (i >> 1) + qo] = v;
      q[8 * ((i >> 1) - 4) + 4 + qo] = v;
    }
    t_base = ext_a + G.t_off;
    const uint32_t ge_a = ext_a + G.ge_off + 16u;  // address of G(0) in the even copy
    const uint32_t go_a = ext_a + G.go_off + 18u;  // ... in the odd copy
    ge_l = ge_a + 4u * uint32_t(lane);
    go_l = go_a + 4u * uint32_t(lane);
    s8_a = uint32_t(__cvta_generic_to_shared(s));
    const int g = lane >> 2, t = lane & 3;
    qbase = ext_a + G.q_off + 16u * uint32_t(32 + 4 * g + t);
    const int x0 = 2 * t - g;
    const uint32_t own = (g & 1) ? go_a : ge_a, oth = (g & 1) ? ge_a : go_a;
    b_pos = own + uint32_t(2 * x0);
    b_neg = oth + uint32_t(2 * (-x0 - 1));
    b_m0 = x0 >= 0 ? b_pos : b_neg;
    sel_m0 = x0 >= 0 ? 0x3210u : 0x1032u;
    const int sigma = ((D - 1) & 1) ? -1 : 1;
    xq_e = 512 * sigma;
    xq_o = -512 * sigma;
    m2xq_e = -2 * xq_e;
    m2xq_o = -2 * xq_o;
    const uint32_t s2_a = ext_a + G.s2_off;
    const uint32_t cxcopy = ((K + 1) & 1) ? go_a : ge_a;  // parity of y0 = K - h0 - 3
#pragma unroll
    for (int tau = 0; tau < MT; tau++) {
      h0[tau] = 128 * tau + 16 * g + 4 * t;
      // padding lanes (h0 > K) read in-range cells, with S2 and C_{q-p} from
      // zero cells so that their keys are exactly their Rk (see kVirtualRk)
      const bool padl = h0[tau] > K;
      const int h0a = padl ? (K & ~3) : h0[tau];
      cxb[tau] = cxcopy + uint32_t(2 * (padl ? -8 + ((K - 3) & 3) : K - h0a - 3));  // 8-byte aligned
      sxb[tau] = s8_a + uint32_t(3 * h0a - 2 * K);
      shb[tau] = s2_a + uint32_t(h0[tau]);  // zero cells beyond D, in the same 128-byte row
      r2b[tau] = s8_a + uint32_t(2 * h0a);
#pragma unroll
      for (int f = 0; f < 4; f++) {
        const int h = h0[tau] + hoff(f);
        const bool live = h < D, centre = h == K;
        const int pi = h & 1;
        int32_t r = 0;
        if (live && !centre)
          for (int j = 1; 2 * j <= h; j++) r += int32_t(s[h - 2 * j]) * int32_t(s[h + 2 * j]);
        const int32_t c0 = 16 * (centre ? (h >> 1) : (K - 1 - pi));
        // the centre's s_x term is the constant S2[K] m2xq s_K = -2 xq (s_x = s_K): cancelled here
        Rk[tau][f] = live ? 64 * c0 + 2048 * r + (1 << 29) + h + (centre ? 2 * (f < 2 ? xq_e : xq_o) : 0)
                          : kVirtualRk;
      }
    }
#pragma unroll
    for (int r = 0; r < NG; r++) {
      const int j = 64 * r + 2 * lane;
      const int c0 = (j >= 1 && j <= K) ? sm.ce[j] : 0, c1 = (j + 1 <= K) ? sm.ce[j + 1] : 0;
      cq[r] = __halves2half2(__int2half_rn(c0), __int2half_rn(c1));
    }
    // move roles: 0,1 int8 sequence; 2,3 / 4,5 even- / odd-aligned f16 spin
    // copies; 6,7 / 8,9 the two Q records holding the spin (even lane: p, odd: q)
    // and lane 10 the S2 cell of p
    const int role = lane >> 1;
    fb = role == 0 ? s8_a
                   : role == 1 ? t_base + 2u * G.TOFF
                   : role == 2 ? t_base + 2u * G.NT + 2u * G.TOFF + 2u
                   : role == 3 ? ext_a + G.q_off + 512u
                   : role == 4 ? ext_a + G.q_off + 512u - 56u
                               : s2_a;
    f4 = (role == 0 || role >= 5) ? 4u : role <= 2 ? 4u : 16u;
    f1 = (role == 0 || role >= 5) ? 1u : role <= 2 ? 4u * G.NT : 4u;
    pin(qbase), pin(b_pos), pin(b_neg), pin(b_m0), pin(sel_m0), pin(xq_e), pin(xq_o), pin(m2xq_e), pin(m2xq_o);
    pin(fb), pin(f4), pin(f1), pin(t_base), pin(ge_l), pin(go_l), pin(s8_a);
#pragma unroll
    for (int tau = 0; tau < MT; tau++) {
      pin(cxb[tau]), pin(sxb[tau]), pin(shb[tau]), pin(r2b[tau]), pin(h0[tau]);
    }
    __syncwarp();
  }

  __device__ __forceinline__ void evaluate(const WalkParams& P, WarpSmem&, const int8_t*, int, int64_t* trace_row) {
    float acc[MT][2][4];
#pragma unroll
    for (int tau = 0; tau < MT; tau++)
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int o = 0; o < 4; o++) acc[tau][u][o] = 0.f;
    // Y = sum_m A_m B_m over k-blocks m (B shared by the tiles)
#pragma unroll
    for (int m = M_LO; m <= M_HI; m++) {
      uint32_t b0, b1;
      if (m < 0) {  // both pairs mirrored: (G(x), G(x+1)) = swap(G(-x-1), G(-x))
        b0 = __byte_perm(ld32s(b_neg - 32 * m), 0, 0x1032);
        b1 = __byte_perm(ld32s(b_neg - 32 * m - 16), 0, 0x1032);
      } else if (m == 0) {
        b0 = __byte_perm(ld32s(b_m0), 0, sel_m0);
        b1 = ld32s(b_pos + 16);
      } else {
        b0 = ld32s(b_pos + 32 * m);
        b1 = ld32s(b_pos + 32 * m + 16);
      }
#pragma unroll
      for (int tau = 0; tau < MT; tau++)
        if (m >= mlo(tau) && m <= mhi(tau)) {
          const uint4 a = lds128(qbase + 512u * tau + 128 * m);
          mma_tc(acc[tau][SK_TC_CHAINS == 2 ? ((m - M_LO) & 1) : 0], a, b0, b1);
        }
    }
    // key(h) = 64 dE + 2^29 + h = Rk + 512 qs C_{q-p} - s_h (xm 64 X + 2048 qs s_x)   (see header)
#pragma unroll
    for (int tau = 0; tau < MT; tau++) {
      const uint2 cpq = ld64s(cxb[tau]);
      const uint32_t cp1 = cpq.x;                 // (C_{q-p} of h0+3, of h0+2)
      const uint32_t cp2 = cpq.y;                 // (h0+1, h0)
      const uint32_t shq = ld32s(shb[tau]);       // S2[h0 .. h0+3]
      const __half2 c12 = u2h(cp1), c34 = u2h(cp2);
      const int32_t cx[4] = {__half2int_rz(__high2half(c34)), __half2int_rz(__high2half(c12)),
                             __half2int_rz(__low2half(c34)), __half2int_rz(__low2half(c12))};
#pragma unroll
      for (int f = 0; f < 4; f++) {
        const int ho = hoff(f);
        const int32_t X = __float2int_rz(SK_TC_CHAINS == 2 ? acc[tau][0][f] + acc[tau][1][f] : acc[tau][0][f]);
        const int32_t sx = lds8(sxb[tau] + 3 * ho);
        const int32_t sh = sext_byte(shq, ho);
        // S2 = 2 s_h: sh (-256 X - 2 xq s_x) = s_h (-512 X - 2048 qs s_x); at the
        // centre S2 = s_K gives -256 s_K X and the constant cancelled in Rk
        const int32_t k = Rk[tau][f] + (f < 2 ? xq_e : xq_o) * cx[f] + sh * (-256 * X + (f < 2 ? m2xq_e : m2xq_o) * sx);
        if (trace_row && h0[tau] + ho < P.D) trace_row[h0[tau] + ho] = (k - (1 << 29) - (h0[tau] + ho)) >> 6;
        key[tau][f] = uint32_t(k);  // padding slots: exactly their Rk, >= kKeyLimit
      }
    }
  }

  __device__ __forceinline__ void renormalize(const WalkParams& P, int) {
#pragma unroll
    for (int tau = 0; tau < MT; tau++)
#pragma unroll
      for (int f = 0; f < 4; f++)
        if (h0[tau] + hoff(f) >= P.D) Rk[tau][f] = kVirtualRk;
  }

  __device__ __forceinline__ uint32_t local_min() const {
    uint32_t m = kNoCand;
#pragma unroll
    for (int tau = 0; tau < MT; tau++)
#pragma unroll
      for (int f = 0; f < 4; f++) m = min(m, key[tau][f]);
    return m;
  }

  __device__ __forceinline__ void exclude(int h, int) {
#pragma unroll
    for (int tau = 0; tau < MT; tau++) {
      const int d = h - h0[tau];
#pragma unroll
      for (int f = 0; f < 4; f++)
        key[tau][f] = mask_if_eq(key[tau][f], d, hoff(f));
    }
  }

  __device__ __forceinline__ void apply(const WalkParams& P, WarpSmem&, int8_t*, int hs, int lane) {
    const int K = P.K;
    const int p = hs, q = P.L - 1 - hs;
    const bool centre = (p == q);
    const int32_t sp = lds8(s8_a + p), sq = lds8(s8_a + q);
    // this lane's scattered cell (lanes 0..9): position x of the move
    const int x = (lane & 1) ? q : p;
    const int32_t sxo = (lane & 1) ? sq : sp;
    const uint32_t fa = fb + f4 * uint32_t(x >> 2) + 2u * uint32_t((x >> 1) & 1) + f1 * uint32_t(x & 1);
    __syncwarp();
    // the flipped spins read as 0 while C and R are updated
    sts8_if(lane < 2, fa, 0);
    sts16_if(lane >= 2 && lane < 6, fa, 0);
    __syncwarp();
    // C_{2j} += scale * v_j, v_j = s_{p-2j} + s_{p+2j} (apply_neighbor, _kernels.py:126-158)
    {
      const int P1 = p >> 1, pi = p & 1, par = P1 & 1;
      const __half2 scale = __half2half2(__int2half_rn(centre ? -2 * sp : -4 * sp));
      const TcGeom G = tc_geom(P.L);
      const uint32_t ua = t_base + 2u * uint32_t(G.NT * (2 * pi + par) + P1 + G.TOFF + par);
      const uint32_t ub = t_base + 2u * uint32_t(G.NT * (2 * pi + 1 - par) + P1 - 1 + G.TOFF + 1 - par);
      const uint32_t al = ua + 4u * uint32_t(lane), bl = ub - 4u * uint32_t(lane);
#pragma unroll
      for (int r = 0; r < NG; r++) {
        // lag pair (j, j + 1), j = 64 r + 2 lane: 32 lanes x 4 consecutive bytes
        // per access, no bank conflict.  Past K, v_j reads zero cells, so those
        // C stay 0 and the unpredicated stores write the zeros the cells hold.
        const __half2 A = u2h(ld32s(al + 128u * r)), B = u2h(ld32s(bl - 128u * r));
        cq[r] = __hfma2(__hadd2(A, __lowhigh2highlow(B)), scale, cq[r]);
        const uint32_t c = h2u(cq[r]);
        sts32(ge_l + 128u * r, c);
        sts16(go_l + 128u * r, c);
        sts16(go_l + 128u * r + 2u, c >> 16);
      }
    }
    // R_h: the terms s_y s_{2h-y}, y in {p, q}, change sign (same-parity
    // neighbours; the zeroed cells drop the own term and, for a centre move,
    // the pair that flips together)
    {
      const int32_t wp = -4096 * sp, wq = centre ? 0 : -4096 * sq;
      const int pi = p & 1;
#pragma unroll
      for (int tau = 0; tau < MT; tau++) {
        const uint32_t bp = r2b[tau] + uint32_t(2 * pi - p), bq = r2b[tau] + uint32_t(2 * pi - q);
        const int32_t vp0 = lds8(bp), vp1 = lds8(bp + 4), vq0 = lds8(bq), vq1 = lds8(bq + 4);
        const int32_t d0 = wp * vp0 + wq * vq0, d1 = wp * vp1 + wq * vq1;
        if (pi == 0) {
          Rk[tau][0] += d0;
          Rk[tau][1] += d1;
        } else {
          Rk[tau][2] += d0;
          Rk[tau][3] += d1;
        }
      }
    }
    __syncwarp();
    // the flipped spins: int8 sequence, f16 spin copies, Q records
    sts8_if(lane < 2 || lane == 10, fa, lane == 10 ? (centre ? -sp : -2 * sp) : -sxo);
    sts16_if(lane >= 2 && lane < 10, fa, sxo > 0 ? 0xBC00u : 0x3C00u);
    __syncwarp();
  }
};

}  // namespace sk
