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
// chunk start).  The result is the min over key = (E' << 47) | g with
// E' = min(E, 2^17 - 1), i.e. the lexicographic (E, g) minimum -- exactly the
// reference's first-minimum rule (the optimum lies far below the saturation).
//
// Per-thread state (D <= 47, so every parity class fits one uint64):
//   P0 / P1  bit i set iff s_{2i} / s_{2i+1} == -1 (full skew sequence)
//   cw[g]    C_{2j} + 128 as bytes, lags 4g+1..4g+4, in registers (G = ceil(K/4) groups)
// A flip of half h negates positions p = h and q = L-1-h, which have the same
// parity, so only one class changes.  With v_j = s_p s_{p-2j}[2j <= p]
// + s_p s_{p+2j}[p < q, p+2j <= L-1, 2j != q-p] (the mirror-collapsed form,
// DESIGN.md §2), apply_neighbor is C_{2j} -= 4 v_j and E = sum_j C_{2j}^2.
#pragma once
#include "sokol_common.cuh"

namespace sk {

constexpr int kExhKeyShift = 47;  // key = (E' << 47) | g; g < 2^D <= 2^47
constexpr int32_t kExhEMax = (1 << 17) - 1;  // E' = min(E, kExhEMax)

// Bits 4g..4g+3 of m, one per byte (bit i -> byte i): the four products
// x * (1 + 2^7 + 2^14 + 2^21) land in disjoint bit ranges, so no carries.
__device__ __forceinline__ uint32_t spread4(uint64_t m, int g) {
  const uint32_t x = uint32_t(m >> (4 * g)) & 0xFu;
  return (x * 0x00204081u) & 0x01010101u;
}

// One thread's chunk [g0, g1).  The even-lag correlations C_{2j} (|C| <= 91
// for L <= 93) live as offset-binary bytes C + 128, four lags per register,
// so a move updates four lags with one add (the per-byte changes 8 n - 4 v
// never carry or borrow across bytes) and E = sum C^2 is one signed
// IDP4A per four lags after flipping the offset bit (x ^ 0x80 = C as int8).
// Row stride of the per-move table (multiple of 4 words: LDS.128 reads).
template <int G>
__host__ __device__ constexpr int exh_row() { return (G + 3) / 4 * 4; }

// svt[h][g] = 4 * (number of valid partner terms of lag 4g+k+1, per byte):
// the part of a move's update that depends only on the flipped index h.
template <int G>
__device__ void exh_fill_table(int L, uint32_t* svt) {
  const int D = (L + 1) >> 1, K = D - 1;
  for (int i = threadIdx.x; i < D * exh_row<G>(); i += blockDim.x) {
    const int h = i / exh_row<G>(), gi = i % exh_row<G>();
    const int par = h & 1, i0 = h >> 1, imax = K - par;
    const uint64_t vA = (1ull << i0) - 1ull;
    const uint64_t vB = (h == K) ? 0ull : (((1ull << (imax - i0)) - 1ull) & ~(1ull << (K - h - 1)));
    svt[i] = gi < G ? 4u * (spread4(vA, gi) + spread4(vB, gi)) : 0u;
  }
}

template <int G>
__device__ __forceinline__ uint64_t exh_chunk(int L, uint64_t g0, uint64_t g1, const uint32_t* svt) {
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
  // ---- sidelobes of even lags (_kernels.py:70-82), packed -----------------
  uint32_t cw[G];
  int32_t E = 0;
#pragma unroll
  for (int gi = 0; gi < G; gi++) {
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int j = 4 * gi + k + 1;
      int32_t cj = 0;
      if (j <= K) {
        const int n0 = D - j, n1 = D - 1 - j;  // pairs (i, i+j) inside each parity class
        cj = n0 - 2 * __popcll((P0 ^ (P0 >> j)) & ((1ull << n0) - 1ull));
        if (n1 > 0) cj += n1 - 2 * __popcll((P1 ^ (P1 >> j)) & ((1ull << n1) - 1ull));
      }
      E += cj * cj;
      w |= uint32_t(cj + 128) << (8 * k);
    }
    cw[gi] = w;
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
    // C_{2j} -= 4 v_j,  v_j = [vA] + [vB] - 2 [nA] - 2 [nB]:  per byte + 8 (nA + nB) - 4 (vA + vB).
    // h is the same in every lane of a warp (aligned chunks: ctz(g) = ctz(g - g0)), so the
    // table row read below is a broadcast.
    const uint4* row = reinterpret_cast<const uint4*>(svt + h * exh_row<G>());
    uint32_t sv[exh_row<G>()];
#pragma unroll
    for (int q = 0; q < exh_row<G>() / 4; q++) {
      const uint4 v = row[q];
      sv[4 * q] = v.x; sv[4 * q + 1] = v.y; sv[4 * q + 2] = v.z; sv[4 * q + 3] = v.w;
    }
    E = 0;
#pragma unroll
    for (int gi = 0; gi < G; gi++) {
      const uint32_t sn = spread4(nA, gi) + spread4(nB, gi);
      cw[gi] = cw[gi] + (sn << 3) - sv[gi];
      const int32_t sc = int32_t(cw[gi] ^ 0x80808080u);
      E = __dp4a(sc, sc, E);
    }
    const uint64_t fm = (1ull << i0) | (centre ? 0ull : (1ull << ((L - 1 - h) >> 1)));
    if (par) P1 ^= fm; else P0 ^= fm;
    if (E < best_e) {
      best_e = E;
      best_g = g;
    }
  }
  return (uint64_t(uint32_t(min(best_e, kExhEMax))) << kExhKeyShift) | best_g;
}

template <int G>
__global__ void __launch_bounds__(256) exhaustive_kernel(int L, uint64_t g_begin, uint64_t g_end, int chunk_log2,
                                                         unsigned long long* min_key) {
  __shared__ __align__(16) uint32_t svt[SK_MAX_EXHAUSTIVE_D * exh_row<G>()];
  exh_fill_table<G>(L, svt);
  __syncthreads();
  const uint64_t span = g_end - g_begin;
  const uint64_t nchunks = (span + (1ull << chunk_log2) - 1) >> chunk_log2;
  unsigned long long best = ~0ull;
  for (uint64_t ci = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; ci < nchunks;
       ci += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g0 = g_begin + (ci << chunk_log2);
    const uint64_t gs = g0 + (1ull << chunk_log2);
    const uint64_t g1 = gs < g_end ? gs : g_end;
    const unsigned long long k = exh_chunk<G>(L, g0, g1, svt);
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
