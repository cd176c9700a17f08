// walk_engine.cuh -- warp-per-walk driver of the contiguous self-avoiding walk.
//
// One warp runs one walk at a time (persistent grid: warp g runs walks
// g, g + nwarps, ...).  The driver reproduces saw_walk (_kernels.py:189-275)
// step for step:
//   init   : first pivot from the splitmix64 stream (204-209), skew expansion
//            (62-67), O(L^2) sidelobes (70-82), packed words (214-218),
//            visited set seeded with key(P1) (220-226), best = P1 (228-233)
//   step   : all-D delta evaluation (239-243) -> lexicographic (delta, h)
//            argmin over unvisited neighbours (244-258) -> dead end (259-261)
//            or move (262-274: apply, e += delta, toggle bit, visited.add,
//            steps += 1, strict '<' best update)
// The neighbourhood evaluator is a policy class (Eval) so that the scalar
// reference-formula evaluator and the production evaluator share every other
// line of the walk.
#pragma once
#include "sokol_common.cuh"

namespace sk {

struct WalkParams {
  int L, n, D, K;
  uint32_t cap;             // visited-set capacity (power of two)
  const uint64_t* seeds;    // nullable -> derive on device
  uint64_t master, batch, walker_begin;
  int64_t W;
  int64_t* best_e;          // nullable
  uint64_t* best_words;     // nullable (then summary words come from scratch)
  int64_t* steps_out;       // nullable
  uint8_t* dead_out;        // nullable
  sk_batch_summary* summary;  // nullable
  uint64_t* trace_words;    // TRACE only: [W][n+1][nw]
  int64_t* trace_deltas;    // TRACE only: [W][n][D]
  uint64_t* gkeys;          // global visited keys [nwarps][cap] or null (keys in smem)
  int visited_mode;         // SK_VISITED_SMEM / _FINGERPRINT / _GLOBAL chosen by the launch
  // multi-search mode (sk_saw_multi): W = R * W_rep walks; walk w belongs to
  // search r = w / W_rep with its own master seed and batch index, and
  // reduces into summary[r].  masters == nullptr: a single search.
  const uint64_t* masters;
  const uint64_t* batches;
  int64_t W_rep;
  uint32_t warp_smem;       // bytes of dynamic smem per warp
  uint32_t block_smem;      // bytes of the per-block area before the warp areas (Eval::block_bytes)
};

// Per-warp shared-memory carve-up.  Offsets are computed identically on host
// (sokol_abi.cu) and device.
struct WarpSmem {
  int8_t* s8;     // full sequence, zero padded: s8[OFF + i] = s_i, i in [0, L)
  int32_t* ce;    // ce[j] = C_{2j}, j in [0, K]
  int32_t* dl;    // current delta vector (D entries)
  uint32_t* occ;  // visited occupancy bitmap
  uint64_t* keys; // visited keys (smem or global)
  void* ext;      // evaluator-private area
  char* blk;      // per-block area shared by the block's warps (read-only after Eval::block_init)
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

struct SmemLayout {
  uint32_t off_s8, off_ce, off_dl, off_occ, off_keys, off_ext, total;
  int span_off;  // OFF: s8 index of position 0
  uint32_t span;  // s8 bytes
  // span_hi: highest position index the evaluator reads (scalar: 2L-2, fast: L-1+K).
  // ce_alias_keys: the int32 C array is only read during init, so it may share
  // the visited-set key storage (cleared after init) when that is in smem.
  // visited: SK_VISITED_SMEM (keys + bitmap in smem), _FINGERPRINT (fingerprints
  // in smem), _GLOBAL (bitmap in smem); keys live in global memory in the last two
  __host__ __device__ static SmemLayout make(int L, int K, int D, uint32_t cap, int visited,
                                             uint32_t ext_bytes, bool need_dl, int span_hi, bool ce_alias_keys,
                                             int span_lo) {
    SmemLayout s;
    s.span_off = span_lo;  // zero cells below position 0 (>= L + 1, see the evaluators' span_lo)
    s.span = uint32_t(span_lo + span_hi + 1);
    const bool keys_in_smem = visited == SK_VISITED_SMEM;
    const bool alias = ce_alias_keys && keys_in_smem && cap * 8u >= 4u * uint32_t(K + 1);
    uint32_t o = 0;
    s.off_keys = o;
    if (keys_in_smem) o += cap * 8u;
    s.off_s8 = o;
    o = align_up(o + s.span, 16);
    if (alias) {
      s.off_ce = s.off_keys;
    } else {
      s.off_ce = o;
      o = align_up(o + 4u * uint32_t(K + 1), 16);
    }
    s.off_dl = o;
    if (need_dl) o = align_up(o + 4u * uint32_t(D), 16);
    s.off_occ = o;  // occupancy bitmap (keys in smem) or per-slot fingerprints (keys in global)
    o = align_up(o + 4u * (visited == SK_VISITED_FINGERPRINT ? cap : cap / 32u), 16);
    o = align_up(o, 32);  // evaluator area 32-byte aligned (signal blocks are 32-byte units)
    s.off_ext = o;
    o = align_up(o + ext_bytes, 32);  // every warp's area starts 32-byte aligned
    s.total = o;
    return s;
  }
};

constexpr int32_t kExcluded = 0x7fffffff;
constexpr int kRenormSteps = 1 << 16;

// KS = 1: the visited keys are in shared memory (compile-time; see VisitedSet)
template <int NW, bool TRACE, class Eval, int KS>
__device__ __forceinline__ void run_one_walk(const WalkParams& P, const SmemLayout& lay, char* blk, char* wbase,
                                             uint64_t* gkeys_warp, int64_t w, int lane) {
  const int L = P.L, D = P.D, K = P.K, n = P.n;
  const int OFF = lay.span_off;
  WarpSmem sm;
  sm.s8 = reinterpret_cast<int8_t*>(wbase + lay.off_s8);
  sm.ce = reinterpret_cast<int32_t*>(wbase + lay.off_ce);
  sm.dl = reinterpret_cast<int32_t*>(wbase + lay.off_dl);
  sm.occ = reinterpret_cast<uint32_t*>(wbase + lay.off_occ);
  sm.keys = gkeys_warp ? gkeys_warp : reinterpret_cast<uint64_t*>(wbase + lay.off_keys);
  sm.ext = wbase + lay.off_ext;
  sm.blk = blk;
  int8_t* s = sm.s8 + OFF;  // s[i] valid for i in [-span_lo, span_hi], zero outside [0, L)

  // ---- first pivot (_kernels.py:201-209) --------------------------------
  uint64_t master = P.master, batch = P.batch;
  int64_t wi = w;  // walker index within its search (before walker_begin)
  sk_batch_summary* summary = P.summary;
  if (P.masters) {
    const int64_t r = w / P.W_rep;
    wi = w - r * P.W_rep;
    master = P.masters[r];
    batch = P.batches[r];
    summary += r;
  }
  const uint64_t seed = P.seeds ? P.seeds[w] : derive_walk_seed(master, batch, P.walker_begin + uint64_t(wi));
  for (int i = lane; i < int(lay.span); i += 32) sm.s8[i] = 0;
  __syncwarp();
  for (int h = lane; h < D; h += 32) {
    const uint64_t z = mix64(seed + uint64_t(h + 1) * kGolden);  // counter form of _next64
    s[h] = (z >> 63) ? int8_t(-1) : int8_t(1);
  }
  __syncwarp();
  for (int i = 1 + lane; i < D; i += 32) s[D - 1 + i] = (i & 1) ? int8_t(-s[D - 1 - i]) : s[D - 1 - i];
  __syncwarp();

  // ---- packed words (_kernels.py:214-218) --------------------------------
  uint64_t words[NW];
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const int b0 = 64 * i + lane, b1 = b0 + 32;
    const uint32_t lo = __ballot_sync(kFull, b0 < D && s[D - 1 - b0] < 0);
    const uint32_t hi = __ballot_sync(kFull, b1 < D && s[D - 1 - b1] < 0);
    words[i] = uint64_t(lo) | (uint64_t(hi) << 32);
  }

  // ---- sidelobes and energy (_kernels.py:70-82; odd lags vanish) --------
  int32_t epart = 0;
  for (int j = lane; j <= K; j += 32) {
    const int k = 2 * j;
    int32_t acc = 0;
    for (int i = 0; i < L - k; i++) acc += int32_t(s[i]) * int32_t(s[i + k]);
    sm.ce[j] = acc;
    if (j > 0) epart += acc * acc;
  }
  int32_t E = warp_sum_i32(epart);
  __syncwarp();

  Eval ev;
  ev.init(P, sm, s, lane);

  // ---- visited set with P1 (_kernels.py:220-226) ------------------------
  VisitedSet vs{sm.keys, sm.occ, P.cap - 1u, uint32_t(__clz(P.cap) + 1)};
  vs.bind(P.visited_mode);
  vs.clear<KS>(lane);
  __syncwarp();
  KeyState<NW> ks;
  ks.init(words);
  vs.probe<KS>(ks.u_of(words), lane, true);

  int32_t best_e = E;
  uint64_t best_w[NW];
#pragma unroll
  for (int i = 0; i < NW; i++) best_w[i] = words[i];
  const int nw_rt = (D + 63) >> 6;
  if (TRACE) {
    if (lane < nw_rt) {
      uint64_t v = 0;
#pragma unroll
      for (int i = 0; i < NW; i++) if (i == lane) v = words[i];
      P.trace_words[(int64_t(w) * (n + 1)) * nw_rt + lane] = v;
    }
  }

  int steps = 0;
  bool dead = false;
  int last = -1;  // half index of the previous move: N_last = P_{t-1} is visited
  // Steps run in chunks of kRenormSteps; between chunks the evaluator may
  // re-normalise state that drifts by a bounded amount per step (EvalTC's
  // padding slots), at no per-step cost.
  for (int base = 0; base < n && !dead; base += kRenormSteps) {
  const int lim = n - base < kRenormSteps ? n : base + kRenormSteps;
  for (int step = base; step < lim; step++) {
    // ---- neighbourhood (_kernels.py:239-243) ----------------------------
    ev.evaluate(P, sm, s, lane, TRACE ? P.trace_deltas + (int64_t(w) * n + step) * D : nullptr);
    // undoing the last move returns to P_{t-1}, whose key is in the set:
    // rejected without hashing (the same membership answer)
    if (last >= 0) ev.exclude(last, lane);
    // ---- best unvisited neighbour (_kernels.py:244-261) -----------------
    int hs = -1;
    int32_t dsel = 0;
    int fwi = 0;
    uint64_t fbit = 0;
    for (;;) {
      const uint32_t m = warp_min_u32(ev.local_min());
      if (m >= kKeyLimit) break;
      const int hc = cand_h(m);
      ev.prefetch(P, hc, lane);  // the move's operands load while the candidate is probed
      uint64_t chain[NW];
      const uint64_t nk = ks.u_of_flip(words, D, hc, chain, fwi, fbit);
      if (!vs.probe<KS>(nk, lane, true)) {  // absent: inserted = _visited_add(best_key)
        hs = hc;
        dsel = cand_delta(m);
        ks.commit(D, hc, chain);
        break;
      }
      ev.exclude(hc, lane);
    }
    if (hs < 0) {
      dead = true;
      break;
    }
    // ---- move (_kernels.py:262-274) -------------------------------------
    ev.apply(P, sm, s, hs, lane);
    last = hs;
    E += dsel;
    toggle_word<NW>(words, fwi, fbit);  // the accepted candidate's flip (last u_of_flip)
    steps += 1;
    if (TRACE) {
      if (lane < nw_rt) {
        uint64_t v = 0;
#pragma unroll
        for (int i = 0; i < NW; i++) if (i == lane) v = words[i];
        P.trace_words[(int64_t(w) * (n + 1) + steps) * nw_rt + lane] = v;
      }
    }
    if (__builtin_expect(E < best_e, 0)) {  // rare after the first descent: a uniform branch, not selects
      best_e = E;
#pragma unroll
      for (int i = 0; i < NW; i++) best_w[i] = words[i];
    }
  }
  ev.renormalize(P, lane);
  }

  // ---- outputs (_kernels.py:283-287) and batch reduction ------------------
  if (lane == 0) {
    if (P.best_e) P.best_e[w] = best_e;
    if (P.steps_out) P.steps_out[w] = steps;
    if (P.dead_out) P.dead_out[w] = dead ? 1 : 0;
    if (summary) {
      const uint64_t key = (uint64_t(uint32_t(best_e)) << 32) | uint64_t(uint32_t(P.walker_begin + uint64_t(wi)));
      atomicMin(reinterpret_cast<unsigned long long*>(&summary->min_key), (unsigned long long)key);
      atomicAdd(reinterpret_cast<unsigned long long*>(&summary->steps_sum), (unsigned long long)steps);
    }
  }
  if (P.best_words && lane < nw_rt) {
    uint64_t v = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) if (i == lane) v = best_w[i];
    P.best_words[int64_t(w) * nw_rt + lane] = v;
  }
  __syncwarp();
}

// Register cap for kMinBlocks resident blocks: 64K registers per SM, allocated
// per warp in units of 8 per thread.  Set with __maxnreg__ (a hard cap) rather
// than __launch_bounds__' minimum-blocks hint, which makes ptxas aim well
// below the cap.
template <class Eval, int WPB>
constexpr int kMaxRegs = (65536 / (Eval::kMinBlocks * WPB * 32)) / 8 * 8 > 255
                             ? 255
                             : (65536 / (Eval::kMinBlocks * WPB * 32)) / 8 * 8;

template <int NW, bool TRACE, class Eval, int WPB, int KS = 0>
__global__ void __launch_bounds__(WPB * 32) __maxnreg__((kMaxRegs<Eval, WPB>)) saw_walk_kernel(WalkParams P, SmemLayout lay) {
  extern __shared__ __align__(128) char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = int64_t(blockIdx.x) * WPB + wib;
  const int64_t nwarps = int64_t(gridDim.x) * WPB;
  Eval::block_init(P, smem_raw, int(threadIdx.x), int(blockDim.x));
  __syncthreads();
  char* wbase = smem_raw + P.block_smem + size_t(wib) * P.warp_smem;
  uint64_t* gkeys = P.gkeys ? P.gkeys + size_t(gwarp) * P.cap : nullptr;
  for (int64_t w = gwarp; w < P.W; w += nwarps)
    run_one_walk<NW, TRACE, Eval, KS>(P, lay, smem_raw, wbase, gkeys, w, lane);
}

// Evaluator probe (sk_eval_states): the walk's own evaluator on caller-given
// states.  Warp w loads half sequence w (+-1 int8), builds the state exactly
// as the walk init does (skew expansion, O(L^2) sidelobes, Eval::init), writes
// the raw delta vector (the trace row of _kernels.py:241-243), then applies
// moves[w][0..M) one after another (apply_neighbor, _kernels.py:126-158, no
// visited check), writing the delta vector after each.  Lets tests drive the
// production evaluator on states a random walk never reaches (all +1,
// periodic, published optima: |C_k| near its bound L - k).
template <int NW, class Eval, int WPB>
__global__ void __launch_bounds__(WPB * 32, 1) eval_states_kernel(WalkParams P, SmemLayout lay, const int8_t* halves,
                                                                    int M, const int32_t* moves, int64_t* deltas) {
  extern __shared__ __align__(128) char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int L = P.L, D = P.D, K = P.K;
  Eval::block_init(P, smem_raw, int(threadIdx.x), int(blockDim.x));
  __syncthreads();
  char* wbase = smem_raw + P.block_smem + size_t(wib) * P.warp_smem;
  WarpSmem sm;
  sm.blk = smem_raw;
  sm.s8 = reinterpret_cast<int8_t*>(wbase + lay.off_s8);
  sm.ce = reinterpret_cast<int32_t*>(wbase + lay.off_ce);
  sm.dl = reinterpret_cast<int32_t*>(wbase + lay.off_dl);
  sm.occ = reinterpret_cast<uint32_t*>(wbase + lay.off_occ);
  sm.keys = reinterpret_cast<uint64_t*>(wbase + lay.off_keys);
  sm.ext = wbase + lay.off_ext;
  int8_t* s = sm.s8 + lay.span_off;
  for (int64_t w = int64_t(blockIdx.x) * WPB + wib; w < P.W; w += int64_t(gridDim.x) * WPB) {
    for (int i = lane; i < int(lay.span); i += 32) sm.s8[i] = 0;
    __syncwarp();
    for (int h = lane; h < D; h += 32) s[h] = halves[w * D + h];
    __syncwarp();
    for (int i = 1 + lane; i < D; i += 32) s[D - 1 + i] = (i & 1) ? int8_t(-s[D - 1 - i]) : s[D - 1 - i];
    __syncwarp();
    for (int j = lane; j <= K; j += 32) {
      int32_t acc = 0;
      for (int i = 0; i < L - 2 * j; i++) acc += int32_t(s[i]) * int32_t(s[i + 2 * j]);
      sm.ce[j] = acc;
    }
    __syncwarp();
    Eval ev;
    ev.init(P, sm, s, lane);
    int64_t* row = deltas + w * int64_t(M + 1) * D;
    ev.evaluate(P, sm, s, lane, row);
    for (int m = 0; m < M; m++) {
      __syncwarp();
      const int h = moves[w * M + m];
      if (h >= 0 && h < D) ev.apply(P, sm, s, h, lane);  // out of range: state unchanged
      row += D;
      ev.evaluate(P, sm, s, lane, row);
    }
    __syncwarp();
  }
}

// Summary init / finish (tiny kernels on the same stream), one block per
// search: summary r covers walks [r * W_rep, (r + 1) * W_rep).
__global__ void summary_init_kernel(sk_batch_summary* s) {
  s += blockIdx.x;
  if (threadIdx.x == 0) {
    s->min_key = ~0ull;
    s->steps_sum = 0;
  }
  if (threadIdx.x < SK_MAX_WORDS) s->best_words[threadIdx.x] = 0;
}

__global__ void summary_finish_kernel(sk_batch_summary* s, const uint64_t* best_words, int nw,
                                      uint64_t walker_begin, int64_t W_rep) {
  s += blockIdx.x;
  const uint64_t key = s->min_key;
  if (key == ~0ull) return;
  const uint64_t local = uint64_t(blockIdx.x) * uint64_t(W_rep) + (uint64_t(uint32_t(key)) - uint32_t(walker_begin));
  if (threadIdx.x < nw) s->best_words[threadIdx.x] = best_words[local * nw + threadIdx.x];
}

}  // namespace sk
