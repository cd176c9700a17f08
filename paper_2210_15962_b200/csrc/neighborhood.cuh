// neighborhood.cuh -- batched neighbourhood evaluation and moves on the
// device.
//
// Device versions of _kernels.all_neighbor_deltas (_kernels.py:162-165, via
// neighbor_delta, 85-123) and _kernels.apply_neighbor (126-158), the kernels
// behind neighborhood.compute_deltas / apply_flip (neighborhood.py:80-100),
// batched over S independent states.  Arrays keep the reference's layout
// and dtypes so a state moves between host and device unchanged:
//   s[S][L]  int64 full sequence (+-1),  c[S][L]  int64 with c[k] = C_k,
//   deltas[S][D] int64,  h[S] int64 half index of the move.
// The arithmetic is the reference's four-product form verbatim, in int64
// (these entry points accept any +-1 sequence and any sidelobe values, as
// the reference does; the walk engine's algebraic shortcuts assume skew
// symmetry and are not used here).  One warp per state; lanes own
// neighbours (deltas) or lags (apply).
#pragma once
#include "sokol_common.cuh"

namespace sk {

__device__ __forceinline__ int64_t nb_lag_d(const int64_t* s, int L, int p, int q, int k) {
  // d of one even lag k, before doubling (_kernels.py:98-121)
  const int64_t sp = s[p];
  int64_t d = 0;
  if (p == q) {
    if (p + k < L) d -= sp * s[p + k];
    if (p - k >= 0) d -= s[p - k] * sp;
    return d;
  }
  const int64_t sq = s[q];
  const int pk = p + k, qk = q - k;
  if (pk < L && pk != q) d -= sp * s[pk];
  if (p - k >= 0) d -= s[p - k] * sp;
  if (q + k < L) d -= sq * s[q + k];
  if (qk >= 0 && qk != p) d -= s[qk] * sq;
  return d;
}

__global__ void neighbor_deltas_kernel(int L, int64_t S, const int64_t* __restrict__ s_all,
                                       const int64_t* __restrict__ c_all, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int D = (L + 1) / 2;
  for (int64_t st = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; st < S;
       st += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t* s = s_all + st * L;
    const int64_t* c = c_all + st * L;
    for (int h = lane; h < D; h += 32) {
      const int p = h, q = L - 1 - h;
      int64_t acc = 0;
      for (int k = 2; k < L; k += 2) {
        int64_t d = nb_lag_d(s, L, p, q, k);
        d += d;
        acc += d * (2 * c[k] + d);
      }
      out[st * D + h] = acc;
    }
  }
}

__global__ void apply_neighbor_kernel(int L, int64_t S, int64_t* __restrict__ s_all, int64_t* __restrict__ c_all,
                                      const int64_t* __restrict__ h_all) {
  const int lane = threadIdx.x & 31;
  for (int64_t st = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; st < S;
       st += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    int64_t* s = s_all + st * L;
    int64_t* c = c_all + st * L;
    const int64_t hv = h_all[st];
    if (hv < 0 || hv >= (L + 1) / 2) continue;  // invalid move index: state left unchanged (host validates)
    const int p = int(hv), q = L - 1 - p;
    for (int k = 2 * (lane + 1); k < L; k += 64) c[k] += 2 * nb_lag_d(s, L, p, q, k);  // _kernels.py:133-155
    __syncwarp();
    if (lane == 0) {
      const int64_t sp = s[p], sq = s[q];
      s[p] = -sp;
      if (p != q) s[q] = -sq;
    }
    __syncwarp();
  }
}

}  // namespace sk
