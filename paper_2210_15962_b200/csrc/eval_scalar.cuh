// eval_scalar.cuh -- reference-formula neighbourhood evaluator (cross-check
// variant, SK_VARIANT_SCALAR).
//
// Lane-per-neighbour evaluation of exactly the arithmetic of neighbor_delta
// (_kernels.py:85-123) and apply_neighbor (_kernels.py:126-158), on int8
// spins in shared memory (zero padded, so the reference's range guards are
// implicit) and int32 even-lag correlations.  O(L) per neighbour; kept as an
// independent on-device implementation that the production evaluator is
// cross-checked against in tests (identical traces).
#pragma once
#include "walk_engine.cuh"

namespace sk {

__device__ __forceinline__ int32_t pair_products(const int8_t* s, int p, int q, int k) {
  // Sum of the (up to) four products of _kernels.py:112-121 at lag k; the
  // range guards are the zero padding, the p+k != q / q-k != p guards are the
  // single lag k == q - p.
  const int32_t sp = s[p], sq = s[q];
  const bool ex = (k == q - p);
  int32_t t = int32_t(s[p - k]) * sp + sq * int32_t(s[q + k]);
  if (!ex) t += sp * int32_t(s[p + k]) + int32_t(s[q - k]) * sq;
  return t;
}

__device__ __forceinline__ int32_t center_products(const int8_t* s, int p, int k) {
  const int32_t sp = s[p];  // _kernels.py:98-106
  return sp * int32_t(s[p + k]) + int32_t(s[p - k]) * sp;
}

struct EvalScalar {
  int32_t* dl = nullptr;
  int nd = 0;
  static constexpr uint32_t ext_bytes(int, int) { return 0; }
  static bool supports(int) { return true; }
  static constexpr bool kNeedsDl = true;
  static constexpr bool kSmemKeysVariant = false;
  static constexpr bool kCeAliasKeys = false;
  static constexpr int kMinBlocks = 1;
  static int span_hi(int L, int) { return 2 * L - 2; }  // q + k
  static int span_lo(int L, int) { return L - 1; }      // p - k
  static uint32_t block_bytes(int) { return 0; }  // no per-block table
  __device__ static void block_init(const WalkParams&, char*, int, int) {}
  __device__ __forceinline__ void prefetch(const WalkParams&, int, int) {}  // nothing to prefetch
  __device__ __forceinline__ void renormalize(const WalkParams&, int) {}     // no drifting state

  __device__ __forceinline__ void init(const WalkParams&, WarpSmem&, int8_t*, int) {}

  __device__ __forceinline__ void evaluate(const WalkParams& P, WarpSmem& sm, const int8_t* s, int lane,
                                           int64_t* trace_row) {
    const int L = P.L, D = P.D;
    dl = sm.dl;
    nd = D;
    for (int h = lane; h < D; h += 32) {
      const int p = h, q = L - 1 - h;
      int32_t acc = 0;
      if (p == q) {
        for (int k = 2; k < L; k += 2) {
          const int32_t d = -2 * center_products(s, p, k);
          acc += d * (2 * sm.ce[k >> 1] + d);
        }
      } else {
        for (int k = 2; k < L; k += 2) {
          const int32_t d = -2 * pair_products(s, p, q, k);
          acc += d * (2 * sm.ce[k >> 1] + d);
        }
      }
      sm.dl[h] = acc;
      if (trace_row) trace_row[h] = acc;
    }
    __syncwarp();
  }

  __device__ __forceinline__ uint32_t local_min() const {
    uint32_t local = kNoCand;
    for (int h = int(threadIdx.x & 31); h < nd; h += 32) {
      const int32_t d = dl[h];
      if (d != kExcluded) local = min(local, pack_cand(d, h));
    }
    return local;
  }

  __device__ __forceinline__ void exclude(int h, int lane) {
    if (lane == (h & 31)) dl[h] = kExcluded;
    __syncwarp();
  }

  __device__ __forceinline__ void apply(const WalkParams& P, WarpSmem& sm, int8_t* s, int hs, int lane) {
    const int L = P.L, K = P.K;
    const int p = hs, q = L - 1 - hs;
    for (int j = 1 + lane; j <= K; j += 32) {
      const int k = 2 * j;
      const int32_t d = (p == q) ? -center_products(s, p, k) : -pair_products(s, p, q, k);
      sm.ce[j] += 2 * d;
    }
    __syncwarp();
    if (lane == 0) {
      s[p] = int8_t(-s[p]);
      if (p != q) s[q] = int8_t(-s[q]);
    }
    __syncwarp();
  }
};

}  // namespace sk
