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
// Every real candidate key ((delta/8 + kBias) << kHBits | h) is below 2^30;
// a warp minimum at or above it means no unvisited neighbour is left.
constexpr uint32_t kKeyLimit = 1u << 30;

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

// Visited-set identity.  The reference keys a pivot by key = mix64(u) with
// u = h_{NW-1} ^ w_{NW-1}, h_0 = KEY_SEED, h_{i+1} = mix64(h_i ^ w_i)
// (key_of_words, _kernels.py:46-53).  mix64 is a bijection on 64-bit words
// (_kernels.py:32), so  key(x) == key(y)  <=>  u(x) == u(y): storing u instead
// of the key gives the identical membership (including the reference's
// cross-word collisions for D > 64) without the final mix64.  The prefixes
// h_i of the current pivot are cached, so a candidate whose flipped bit lies
// in word i costs (NW - 1 - i) mix64 calls -- zero for the last word.
template <int NW>
struct KeyState {
  uint64_t hp[NW];  // hp[i] = h_i of the current pivot

  __device__ __forceinline__ void init(const uint64_t (&w)[NW]) {
    hp[0] = kKeySeed;
#pragma unroll
    for (int i = 0; i + 1 < NW; i++) hp[i + 1] = mix64(hp[i] ^ w[i]);
  }
  __device__ __forceinline__ uint64_t u_of(const uint64_t (&w)[NW]) const { return hp[NW - 1] ^ w[NW - 1]; }

  // u of the pivot with half index h flipped; chain[] receives the candidate's
  // prefixes (valid from its flipped word on) for commit().
  // wi / bit receive the flipped word and bit (for toggle_word on acceptance).
  __device__ __forceinline__ uint64_t u_of_flip(const uint64_t (&w)[NW], int D, int h, uint64_t (&chain)[NW],
                                                int& wi, uint64_t& bit) const {
    const int b = D - 1 - h;
    wi = b >> 6;
    bit = 1ull << (b & 63);
    if constexpr (NW == 1) {
      return hp[0] ^ w[0] ^ bit;
    } else if constexpr (NW == 2) {
      // wi is warp-uniform: a branch, so only the needed path executes
      if (wi == 1) return hp[1] ^ w[1] ^ bit;
      chain[1] = mix64(hp[0] ^ w[0] ^ bit);
      return chain[1] ^ w[1];
    } else {
      uint64_t x = hp[0];
#pragma unroll
      for (int i = 0; i < NW; i++) {
        x = (i == wi) ? hp[i] : x;  // prefix unchanged up to the flipped word (selects: no local memory)
        chain[i] = x;
        if (i + 1 < NW && i >= wi) x = mix64(x ^ (w[i] ^ (i == wi ? bit : 0ull)));
      }
      return chain[NW - 1] ^ (w[NW - 1] ^ (wi == NW - 1 ? bit : 0ull));
    }
  }

  __device__ __forceinline__ void commit(int D, int h, const uint64_t (&chain)[NW]) {
    const int wi = (D - 1 - h) >> 6;
    if constexpr (NW == 2) {
      if (wi == 0) hp[1] = chain[1];
    } else {
#pragma unroll
      for (int i = 1; i < NW; i++) hp[i] = (i > wi) ? chain[i] : hp[i];
    }
  }
};

// words ^= bit in word wi (wi, bit from KeyState::u_of_flip); wi is warp-uniform
template <int NW>
__device__ __forceinline__ void toggle_word(uint64_t (&w)[NW], int wi, uint64_t bit) {
  if constexpr (NW == 1) {
    w[0] ^= bit;
  } else if constexpr (NW == 2) {
    if (wi) w[1] ^= bit; else w[0] ^= bit;  // warp-uniform: predicated XORs
  } else {
#pragma unroll
    for (int i = 0; i < NW; i++) w[i] ^= (wi == i) ? bit : 0ull;
  }
}

template <int NW>
__device__ __forceinline__ void toggle_half_bit(uint64_t (&w)[NW], int D, int h) {
  const int b = D - 1 - h;
  const uint64_t bit = 1ull << (b & 63);
  if constexpr (NW == 1) {
    w[0] ^= bit;
  } else if constexpr (NW == 2) {
    if (b >> 6) w[1] ^= bit; else w[0] ^= bit;  // warp-uniform
  } else {
    // selects, not a conditional store: a data-dependent index would push w[] to local memory
#pragma unroll
    for (int i = 0; i < NW; i++) w[i] ^= ((b >> 6) == i) ? bit : 0ull;
  }
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
// finds the end of the probe run, a second ballot finds a key match inside
// the run.  Membership -- the only thing the walk observes -- is identical to
// the reference's table whatever the capacity.  Two layouts:
//   * keys in shared memory (KS = 1) with an occupancy bitmap, so that key 0
//     is a legal key (no sentinel);
//   * fingerprints (KS = 2): a nonzero 32-bit fingerprint per slot in shared
//     memory (0 = empty) and the full keys in an L2-resident global scratch,
//     read only when a fingerprint matches.  Half the shared memory per walk;
//   * global keys (KS = 3): the occupancy bitmap in shared memory, the keys
//     in the global scratch (read for the slots of the probe run).
// KS = 0 decides at run time from the launch's layout (bind()).
// ---------------------------------------------------------------------------
struct VisitedSet {
  uint64_t* keys;  // [cap]  (stores u, see KeyState): smem, or global in fingerprint mode
  uint32_t* occ;   // smem: [cap/32] occupancy bits, or [cap] fingerprints (0 = empty)
  uint32_t mask;   // cap - 1, cap a power of two >= 32
  uint32_t shift;  // 32 - log2(cap)
  uint32_t keys_s = 0;  // shared-window address of keys when they live in shared memory
  bool keys_shared = false;    // KS = 0 only: the launch placed the keys in shared memory (layout 1)
  bool bitmap_global = false;  // KS = 0 only: global keys with a bitmap (layout 3) instead of fingerprints

  // The layout is the launch's explicit choice (WalkParams::visited_mode), not
  // inferred from the address, so a key array at shared offset 0 is fine.
  __device__ __forceinline__ void bind(int visited_mode) {
    keys_shared = visited_mode == SK_VISITED_SMEM;
    bitmap_global = visited_mode == SK_VISITED_GLOBAL;
    keys_s = keys_shared ? uint32_t(__cvta_generic_to_shared(keys)) : 0u;
  }
  template <int KS>
  __device__ __forceinline__ bool smem_keys() const { return KS == 1 || (KS == 0 && keys_shared); }

  __device__ __forceinline__ uint64_t lds_key(uint32_t slot) const {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(keys_s + slot * 8u));
    return v;
  }

  template <int KS = 0>
  __device__ __forceinline__ void clear(int lane) {
    const bool bitmap = smem_keys<KS>() || KS == 3 || (KS == 0 && bitmap_global);
    const uint32_t words = bitmap ? (mask >> 5) + 1u : mask + 1u;
    for (uint32_t i = lane; i < words; i += 32) occ[i] = 0u;
  }

  __device__ __forceinline__ static uint32_t home(uint64_t u, uint32_t shift) {
    // Fibonacci hash of the folded identity (u itself is not uniformly mixed
    // for D <= 64, where it is KEY_SEED ^ words)
    return ((uint32_t(u) ^ uint32_t(u >> 32)) * 0x9E3779B1u) >> shift;
  }
  __device__ __forceinline__ static uint32_t fingerprint(uint64_t u) {
    return ((uint32_t(u >> 32) * 0x85EBCA6Bu) ^ uint32_t(u)) | 1u;  // never 0 (= empty)
  }

  // Warp-collective.  Returns true iff u is present.  If absent and
  // `insert_if_absent`, the lane at the first free slot writes it.
  template <int KS = 0>
  __device__ __forceinline__ bool probe(uint64_t key, int lane, bool insert_if_absent) {
    uint32_t start = home(key, shift);
    if (smem_keys<KS>()) {
      for (;;) {
        const uint32_t slot = (start + lane) & mask;
        const uint32_t ow = occ[slot >> 5];
        // load the slot's key alongside its occupancy word (stale keys of
        // free slots are masked by `run` below)
        const uint64_t kv = lds_key(slot);
        const bool used = (ow >> (slot & 31)) & 1u;
        const uint32_t empty_mask = __ballot_sync(kFull, !used);
        // lanes strictly before the first empty slot are the live probe run
        const uint32_t run = empty_mask ? ((empty_mask & (0u - empty_mask)) - 1u) : kFull;
        const bool hit = ((run >> lane) & 1u) && kv == key;
        if (__any_sync(kFull, hit)) return true;
        if (empty_mask) {
          if (insert_if_absent) {
            const int first = __ffs(empty_mask) - 1;
            if (lane == first) {
              asm volatile("st.shared.u64 [%0], %1;" ::"r"(keys_s + slot * 8u), "l"(key) : "memory");
              atomicOr(&occ[slot >> 5], 1u << (slot & 31));
            }
            __syncwarp();
          }
          return false;
        }
        start = (start + 32) & mask;
      }
    }
    if (KS == 3 || (KS == 0 && bitmap_global)) {
      // keys in global memory, occupancy bitmap in shared memory
      for (;;) {
        const uint32_t slot = (start + lane) & mask;
        const bool used = (occ[slot >> 5] >> (slot & 31)) & 1u;
        const uint32_t empty_mask = __ballot_sync(kFull, !used);
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
    const uint32_t f = fingerprint(key);
    for (;;) {
      const uint32_t slot = (start + lane) & mask;
      const uint32_t x = occ[slot];
      const uint32_t empty_mask = __ballot_sync(kFull, x == 0u);
      const uint32_t run = empty_mask ? ((empty_mask & (0u - empty_mask)) - 1u) : kFull;
      // full keys are read (from L2) only where the fingerprint matches: a
      // rare, warp-uniform branch (a true hit, or a fingerprint collision)
      const bool fm = ((run >> lane) & 1u) && x == f;
      if (__ballot_sync(kFull, fm)) {
        if (__any_sync(kFull, fm && keys[slot] == key)) return true;
      }
      if (empty_mask) {
        if (insert_if_absent) {
          const int first = __ffs(empty_mask) - 1;
          if (lane == first) {
            keys[slot] = key;
            occ[slot] = f;
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
