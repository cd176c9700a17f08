// sokol_common.cuh -- device building blocks shared by the walk kernels.
//
// Semantics mirror /root/reference/pkg/src/skewsaw/_kernels.py; every helper
// cites the reference lines it reproduces.  Layout conventions:
//   * half index h in [0, D); full positions p = h, q = L-1-h (mirror pair).
//   * `words` = the reference's packed half (_kernels.py:5-7): little-endian
//     uint64 words, bit b = D-1-h set iff half spin h is -1.  Kept uniform in
//     every lane's registers because the visited-set key is a function of it.
//   * energies / deltas are int32 on device (|E| < 2^31 for L <= SK_MAX_L).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sokol.h"

namespace sk {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;   // _kernels.py:22
constexpr uint64_t kKeySeed = 0xA0761D6478BD642Full;  // _kernels.py:23
constexpr int kMaxWords = SK_MAX_WORDS;                // D <= 64*kMaxWords
constexpr unsigned kFull = 0xffffffffu;

// Packed selection key: ((delta/8 + kBias) << kHBits) | h.  delta is always a
// multiple of 8 (dE = 8*sum_k v_k(2v_k - C_k)) and
// |delta/8| <= 8K + 2K^2 < 2^20 for L <= 1023, so the key orders candidates
// lexicographically by (delta, h) -- the reference's tie rule
// (_kernels.py:244-258: strict '<' while scanning h ascending).
constexpr int kHBits = 9;
constexpr int32_t kBias = 1 << 20;
constexpr uint32_t kNoCand = 0xffffffffu;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // _kernels.py:32-37
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t derive_walk_seed(uint64_t master, uint64_t batch,
                                                     uint64_t walker) {  // runner.py:53-57
  uint64_t h = mix64(master ^ kGolden);
  h = mix64(h ^ batch);
  return mix64(h ^ walker);
}

template <int NW>
__device__ __forceinline__ uint64_t key_of_words(const uint64_t (&w)[NW]) {  // _kernels.py:46-53
  uint64_t h = kKeySeed;
#pragma unroll
  for (int i = 0; i < NW; i++) h = mix64(h ^ w[i]);
  return h;
}

// Key of `w` with half index h flipped (bit D-1-h toggled), _kernels.py:250-253.
template <int NW>
__device__ __forceinline__ uint64_t key_of_flipped(const uint64_t (&w)[NW], int D, int h) {
  const int b = D - 1 - h;
  uint64_t h64 = kKeySeed;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const uint64_t x = w[i] ^ ((b >> 6) == i ? (1ull << (b & 63)) : 0ull);
    h64 = mix64(h64 ^ x);
  }
  return h64;
}

template <int NW>
__device__ __forceinline__ void toggle_half_bit(uint64_t (&w)[NW], int D, int h) {
  const int b = D - 1 - h;
#pragma unroll
  for (int i = 0; i < NW; i++)
    if ((b >> 6) == i) w[i] ^= 1ull << (b & 63);
}

__device__ __forceinline__ uint32_t pack_cand(int32_t delta, int h) {
  return (uint32_t(delta / 8 + kBias) << kHBits) | uint32_t(h);
}
__device__ __forceinline__ int cand_h(uint32_t key) { return int(key & ((1u << kHBits) - 1)); }
__device__ __forceinline__ int32_t cand_delta(uint32_t key) { return (int32_t(key >> kHBits) - kBias) * 8; }

// ---------------------------------------------------------------------------
// Per-walk visited set (_kernels.py:168-186 semantics: exact membership of
// 64-bit keys).  Open addressing with linear probing, probed 32 slots at a
// time by the whole warp: lane i inspects slot (start + i) & mask, a ballot
// over the occupancy bitmap finds the end of the probe run, a second ballot
// finds a key match inside the run.  Membership -- the only thing the walk
// observes -- is identical to the reference's table whatever the capacity.
// Occupancy lives in a bitmap so that key 0 is a legal key (no sentinel).
// ---------------------------------------------------------------------------
struct VisitedSet {
  uint64_t* keys;  // [cap]
  uint32_t* occ;   // [cap/32] occupancy bits
  uint32_t mask;   // cap - 1, cap a power of two >= 32

  __device__ __forceinline__ void clear(int lane) {
    for (uint32_t i = lane; i <= (mask >> 5); i += 32) occ[i] = 0u;
  }

  // Warp-collective.  Returns true iff key present.  If absent and
  // `insert_if_absent`, lane 0 writes it into the first free slot.
  __device__ __forceinline__ bool probe(uint64_t key, int lane, bool insert_if_absent) {
    uint32_t start = uint32_t(key) & mask;
    for (;;) {
      const uint32_t slot = (start + lane) & mask;
      const bool used = (occ[slot >> 5] >> (slot & 31)) & 1u;
      const uint32_t empty_mask = __ballot_sync(kFull, !used);
      // lanes strictly before the first empty slot are the live probe run
      const uint32_t run = empty_mask ? ((empty_mask & (0u - empty_mask)) - 1u) : kFull;
      const bool hit = ((run >> lane) & 1u) && keys[slot] == key;
      if (__any_sync(kFull, hit)) return true;
      if (empty_mask) {
        if (insert_if_absent) {
          const int first = __ffs(empty_mask) - 1;
          if (lane == first) {
            keys[slot] = key;
            atomicOr(&occ[slot >> 5], 1u << (slot & 31));
          }
          __syncwarp();
        }
        return false;
      }
      start = (start + 32) & mask;
    }
  }
};

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) { return __reduce_min_sync(kFull, v); }
__device__ __forceinline__ int32_t warp_sum_i32(int32_t v) { return __reduce_add_sync(kFull, v); }

}  // namespace sk
