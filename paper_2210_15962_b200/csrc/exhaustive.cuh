// exhaustive.cuh -- Gray-code enumeration of the whole skew half-sequence
// space on the device.
//
// Reference: exhaustive_scan (_kernels.py:290-323), called by
// saw.exhaustive_optimum (saw.py:151-168).  The reference walks g = 1..2^D-1
// single-threaded, flipping half spin h = ctz(g) with neighbor_delta +
// apply_neighbor, and keeps the FIRST minimum (strict '<').  After step g the
// half is gray(g) = g ^ (g >> 1), so the reference's answer is
//   best_e = min_g E(gray(g)),  best_bits = gray(smallest g attaining it).
// Here the g range is cut into chunks, one thread per chunk: the thread
// rebuilds the state at its first g from scratch (O(L^2) with popcounts) and
// then runs the same Gray sequence, h = ctz(g) for every g (valid for any
// chunk start).  The result is the min over key = (E << 44) | g, i.e. the
// lexicographic (E, g) minimum -- exactly the reference's first-minimum rule.
//
// Per-thread state (D <= 44, so every parity class fits one uint64):
//   P0 / P1  bit i set iff s_{2i} / s_{2i+1} == -1 (full skew sequence)
//   c[j]     C_{2j}, j = 1..K, in registers (compile-time bound KMAX)
// A flip of half h negates positions p = h and q = L-1-h, which have the same
// parity, so only one class changes.  With v_j = s_p s_{p-2j}[2j <= p]
// + s_p s_{p+2j}[p < q, p+2j <= L-1, 2j != q-p] (the mirror-collapsed form,
// DESIGN.md §2), apply_neighbor is C_{2j} -= 4 v_j and E = sum_j C_{2j}^2.
#pragma once
#include "sokol_common.cuh"

namespace sk {

constexpr int kExhKeyShift = 44;  // key = (E << 44) | g; g < 2^D <= 2^44, E < 2^20 for L <= 87

template <int KMAX>
__device__ __forceinline__ uint64_t exh_chunk(int L, uint64_t g0, uint64_t g1) {
  const int D = (L + 1) >> 1, K = D - 1;
  // ---- state at g0: half = gray(g0), expanded (_kernels.py:62-67) --------
  const uint64_t x = g0 ^ (g0 >> 1);
  uint64_t P0 = 0, P1 = 0;
  for (int h = 0; h < D; h++) {
    const uint64_t nh = (x >> h) & 1ull;
    const uint64_t nq = nh ^ uint64_t((K - h) & 1);  // s_{L-1-h} = (-1)^{D-1-h} s_h
    uint64_t m = nh << (h >> 1);
    if (h != K) m |= nq << ((L - 1 - h) >> 1);
    if (h & 1) P1 |= m; else P0 |= m;
  }
  // ---- sidelobes of even lags (_kernels.py:70-82) -------------------------
  int32_t c[KMAX + 1];
  int32_t E = 0;
#pragma unroll
  for (int j = 1; j <= KMAX; j++) {
    int32_t cj = 0;
    if (j <= K) {
      const int n0 = D - j, n1 = D - 1 - j;  // pairs (i, i+j) inside each parity class
      cj = n0 - 2 * __popcll((P0 ^ (P0 >> j)) & ((1ull << n0) - 1ull));
      if (n1 > 0) cj += n1 - 2 * __popcll((P1 ^ (P1 >> j)) & ((1ull << n1) - 1ull));
    }
    c[j] = cj;
    E += cj * cj;
  }
  int32_t best_e = E;
  uint64_t best_g = g0;
  // ---- Gray steps (_kernels.py:313-322) ------------------------------------
  for (uint64_t g = g0 + 1; g < g1; g++) {
    const int h = __ffsll(int64_t(g)) - 1;
    const int par = h & 1, i0 = h >> 1;
    const bool centre = (h == K);
    const uint64_t P = par ? P1 : P0;
    const int imax = K - par;  // last index of this parity class
    const uint64_t spm = 0ull - ((P >> i0) & 1ull);  // all ones iff s_p == -1
    const uint64_t lo = i0 ? (__brevll(P) >> (64 - i0)) : 0ull;  // bit j-1 = s_{p-2j}
    const uint64_t hi = P >> (i0 + 1);                          // bit j-1 = s_{p+2j}
    const uint64_t vA = (1ull << i0) - 1ull;
    const uint64_t vB = centre ? 0ull : (((1ull << (imax - i0)) - 1ull) & ~(1ull << (K - h - 1)));
    const uint64_t nA = (lo ^ spm) & vA, nB = (hi ^ spm) & vB;  // products s_p s_x == -1
    const uint64_t pA = vA & ~nA, pB = vB & ~nB;                // products == +1
    E = 0;
#pragma unroll
    for (int j = 1; j <= KMAX; j++) {
      const int b = j - 1;
      const int32_t v = int32_t((pA >> b) & 1ull) + int32_t((pB >> b) & 1ull) - int32_t((nA >> b) & 1ull) -
                        int32_t((nB >> b) & 1ull);
      c[j] -= 4 * v;
      E += c[j] * c[j];
    }
    const uint64_t fm = (1ull << i0) | (centre ? 0ull : (1ull << ((L - 1 - h) >> 1)));
    if (par) P1 ^= fm; else P0 ^= fm;
    if (E < best_e) {
      best_e = E;
      best_g = g;
    }
  }
  return (uint64_t(uint32_t(best_e)) << kExhKeyShift) | best_g;
}

template <int KMAX>
__global__ void __launch_bounds__(256) exhaustive_kernel(int L, uint64_t g_begin, uint64_t g_end, int chunk_log2,
                                                         unsigned long long* min_key) {
  const uint64_t span = g_end - g_begin;
  const uint64_t nchunks = (span + (1ull << chunk_log2) - 1) >> chunk_log2;
  unsigned long long best = ~0ull;
  for (uint64_t ci = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; ci < nchunks;
       ci += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g0 = g_begin + (ci << chunk_log2);
    const uint64_t gs = g0 + (1ull << chunk_log2);
    const uint64_t g1 = gs < g_end ? gs : g_end;
    const unsigned long long k = exh_chunk<KMAX>(L, g0, g1);
    best = k < best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(kFull, best, o);
    best = other < best ? other : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(min_key, best);
}

}  // namespace sk
