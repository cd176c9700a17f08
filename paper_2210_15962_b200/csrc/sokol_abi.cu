// sokol_abi.cu -- C ABI of libsokol.so (declared in include/sokol.h).
//
// Host side of the drop-in boundary: argument validation (the reference's
// RunConfig / WalkConfig rules, runner.py:81-97, saw.py:49-55), launch
// geometry (persistent grid sized from the occupancy calculator, a multiple
// of the SM count), per-device cached scratch, and the host-buffer entry
// points that mirror _kernels.saw_batch / saw_walk argument for argument.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/sokol.h"
#include "eval_scalar.cuh"
#include "eval_fast.cuh"
#include "eval_tc.cuh"
#include "exhaustive.cuh"
#include "neighborhood.cuh"
#include "walk_engine.cuh"

namespace {

thread_local std::string g_err;
int g_variant = SK_VARIANT_AUTO;
int g_visited = SK_VISITED_AUTO;
std::mutex g_mu;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SK_CUDA(call)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(SK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));         \
  } while (0)

struct DevCache {
  void* gkeys = nullptr;
  size_t gkeys_bytes = 0;
  void* words = nullptr;
  size_t words_bytes = 0;
  // host-API staging
  void* h_in = nullptr;
  size_t h_in_bytes = 0;
  void* h_out = nullptr;
  size_t h_out_bytes = 0;
  void* h_walk = nullptr;  // sk_saw_walk_host staging (seed, outputs, trace)
  size_t h_walk_bytes = 0;
};
// Scratch is cached per (device, stream): launches on different streams of one
// device may run concurrently (engine.BatchEngine with several slices on one
// device), so they must not share visited-key or word scratch.
std::map<std::pair<int, uintptr_t>, DevCache> g_cache;
std::mutex g_host_mu;  // serialises the synchronous host-buffer entry points

int grow(void** p, size_t* have, size_t need) {
  if (*have >= need) return SK_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  if (cudaMalloc(p, need) != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return fail(SK_ERR_NOMEM, "cudaMalloc of " + std::to_string(need) + " bytes failed");
  }
  *have = need;
  return SK_OK;
}

DevCache& cache_for(int dev, cudaStream_t st) {
  return g_cache[std::make_pair(dev, reinterpret_cast<uintptr_t>(st))];
}

constexpr uint64_t kMaxVisitedCap = uint64_t(1) << 30;  // keys scratch per resident walk <= 8 GiB

uint64_t visited_capacity(int n) {
  // strictly larger than the n+1 keys a walk can insert, load <= 15/16
  const uint64_t need = std::max<uint64_t>(32, (uint64_t(n) + 1) * 16 / 15 + 1);
  uint64_t cap = 32;
  while (cap < need) cap <<= 1;
  return cap;
}

int validate(int L, int n, int64_t W) {
  if (L < 3 || (L % 2) == 0) return fail(SK_ERR_ARG, "length must be odd and >= 3, got " + std::to_string(L));
  if (L > SK_MAX_L)
    return fail(SK_ERR_UNSUPPORTED, "length " + std::to_string(L) + " exceeds SK_MAX_L=" + std::to_string(SK_MAX_L));
  if (n < 1) return fail(SK_ERR_ARG, "walk step count n must be >= 1");
  if (visited_capacity(n) > kMaxVisitedCap)
    return fail(SK_ERR_UNSUPPORTED, "walk step count n=" + std::to_string(n) + " needs a visited set beyond 2^30 slots");
  if (W < 0) return fail(SK_ERR_ARG, "walker count must be >= 0");
  return SK_OK;
}

#ifndef SK_WPB
#define SK_WPB 4
#endif
constexpr int kWPB = SK_WPB;             // warps per block (one walk per warp)
constexpr uint32_t kSmemKeysMax = 32768;  // keys in smem up to 32 KB per walk

struct Plan {
  sk::WalkParams P;
  sk::SmemLayout lay[4];  // per visited-set layout (SK_VISITED_SMEM / _FINGERPRINT / _GLOBAL)
  bool smem_keys_ok;
  int nw;
  bool dry_run = false;  // compute the launch geometry only
  int64_t resident = 0;  // walks resident at once (grid warps)
};

// Shared-memory carve-up per visited-set layout for the evaluator Eval (its
// area size and spin-array margins); recomputed for the evaluator a launch
// actually instantiates.
template <class Eval>
void plan_layouts(Plan& pl) {
  const int L = pl.P.L, D = pl.P.D;
  for (int v = SK_VISITED_SMEM; v <= SK_VISITED_GLOBAL; v++)
    pl.lay[v] = sk::SmemLayout::make(L, D - 1, D, pl.P.cap, v, Eval::ext_bytes(L, D), Eval::kNeedsDl,
                                     Eval::span_hi(L, D), Eval::kCeAliasKeys, Eval::span_lo(L, D));
}

template <class Eval>
Plan make_plan(int L, int n) {
  Plan pl{};
  const int D = (L + 1) / 2;
  pl.nw = (D + 63) / 64;
  pl.P.L = L;
  pl.P.n = n;
  pl.P.D = D;
  pl.P.K = D - 1;
  pl.P.cap = uint32_t(visited_capacity(n));
  pl.smem_keys_ok = pl.P.cap * 8u <= kSmemKeysMax;
  plan_layouts<Eval>(pl);
  return pl;
}

// Occupancy-driven placement of the visited set: keys in shared memory, or
// keys in an L2-resident global scratch with fingerprints or an occupancy
// bitmap in shared memory -- whichever lets the most walks be resident (ties:
// fingerprints, then shared-memory keys; measured).  The production kernels
// (Eval::kSmemKeysVariant, no trace) are compiled per layout (KS = 1 / 2 / 3);
// the others decide at run time (KS = 0).
template <int NW, bool TRACE, class Eval>
int launch_nw(Plan& pl, cudaStream_t st, int dev) {
  plan_layouts<Eval>(pl);
  using KernT = void (*)(sk::WalkParams, sk::SmemLayout);
  KernT kern[4] = {nullptr, sk::saw_walk_kernel<NW, TRACE, Eval, kWPB, 0>, nullptr, nullptr};
  kern[2] = kern[3] = kern[1];
  if constexpr (Eval::kSmemKeysVariant && !TRACE) {
    kern[1] = sk::saw_walk_kernel<NW, TRACE, Eval, kWPB, 1>;
    kern[2] = sk::saw_walk_kernel<NW, TRACE, Eval, kWPB, 2>;
    kern[3] = sk::saw_walk_kernel<NW, TRACE, Eval, kWPB, 3>;
  }
  int sms = 0, max_optin = 0, per[4] = {0, 0, 0, 0};
  SK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SK_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  pl.P.block_smem = Eval::block_bytes(pl.P.L);
  for (int v = SK_VISITED_SMEM; v <= SK_VISITED_GLOBAL; v++) {
    const size_t smem = pl.P.block_smem + size_t(pl.lay[v].total) * kWPB;
    if (smem > size_t(max_optin) || (v == SK_VISITED_SMEM && !pl.smem_keys_ok)) continue;
    SK_CUDA(cudaFuncSetAttribute(kern[v], cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[v], kern[v], kWPB * 32, smem));
  }
  int mode = 0;
  if (g_visited != SK_VISITED_AUTO && per[g_visited] > 0) {
    mode = g_visited;
  } else {
    for (int v : {SK_VISITED_FINGERPRINT, SK_VISITED_SMEM, SK_VISITED_GLOBAL})
      if (per[v] > 0 && (mode == 0 || per[v] > per[mode])) mode = v;
  }
  if (mode == 0) return fail(SK_ERR_UNSUPPORTED, "walk state does not fit one SM");
  const int per_sm = per[mode];
  const sk::SmemLayout lay = pl.lay[mode];
  pl.P.warp_smem = lay.total;
  pl.P.visited_mode = mode;
  const size_t smem = pl.P.block_smem + size_t(lay.total) * kWPB;
  const int64_t want = (pl.P.W + kWPB - 1) / kWPB;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, int64_t(per_sm) * sms));
  pl.resident = int64_t(per_sm) * sms * kWPB;
  if (pl.dry_run) return SK_OK;
  if (mode != SK_VISITED_SMEM) {
    DevCache& c = cache_for(dev, st);
    int rc = grow(&c.gkeys, &c.gkeys_bytes, size_t(grid) * kWPB * pl.P.cap * 8u);
    if (rc) return rc;
    pl.P.gkeys = static_cast<uint64_t*>(c.gkeys);
  } else {
    pl.P.gkeys = nullptr;
  }
  SK_CUDA(cudaFuncSetAttribute(kern[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern[mode]<<<dim3(unsigned(grid)), dim3(kWPB * 32), smem, st>>>(pl.P, lay);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

// Evaluator dispatch: calls f(std::integral_constant<int, NW>, (Eval*)0) with
// the word count and the evaluator the walk kernels use for this length
// (scalar, or the production evaluator with a compile-time tile bound
// MT = ceil(NW/2) and, for one tile, a compile-time MMA count).  Every
// launch -- walks, traces, the evaluator probe -- goes through here, so the
// probe runs exactly the instantiation the batch kernel runs.
#ifdef SK_OLD_FAST_EVALUATOR
template <int NW, class F>
int dispatch_fast_small(int L, F&& f) {
  const sk::FastGeom g = sk::fast_geom(L);
  const int nm = ((g.MHI - g.MLO + 1) + 1) & ~1;
  using NWc = std::integral_constant<int, NW>;
  switch (nm) {
    case 2: return f(NWc{}, (sk::EvalFast<1, 2>*)nullptr);
    case 4: return f(NWc{}, (sk::EvalFast<1, 4>*)nullptr);
    case 6: return f(NWc{}, (sk::EvalFast<1, 6>*)nullptr);
    case 8: return f(NWc{}, (sk::EvalFast<1, 8>*)nullptr);
    case 10: return f(NWc{}, (sk::EvalFast<1, 10>*)nullptr);
    case 12: return f(NWc{}, (sk::EvalFast<1, 12>*)nullptr);
  }
  return f(NWc{}, (sk::EvalFast<1, 0>*)nullptr);
}
#endif

// L <= 511: the one- / two-tile evaluator with a compile-time k-block count
// (NI = ceil(D / 16) fixes the word count too: nw = ceil(NI / 4)).
template <int NI, class F>
int dispatch_tc_at(F&& f) {
  return f(std::integral_constant<int, (NI + 3) / 4>{}, (sk::EvalTC<NI>*)nullptr);
}

template <class F>
int dispatch_tc(int L, F&& f) {
  switch (((L + 1) / 2 + 15) / 16) {
    case 1: return dispatch_tc_at<1>(f);
    case 2: return dispatch_tc_at<2>(f);
    case 3: return dispatch_tc_at<3>(f);
    case 4: return dispatch_tc_at<4>(f);
    case 5: return dispatch_tc_at<5>(f);
    case 6: return dispatch_tc_at<6>(f);
    case 7: return dispatch_tc_at<7>(f);
    case 8: return dispatch_tc_at<8>(f);
#ifndef SK_TC_ONE_TILE_ONLY
    case 9: return dispatch_tc_at<9>(f);
    case 10: return dispatch_tc_at<10>(f);
    case 11: return dispatch_tc_at<11>(f);
    case 12: return dispatch_tc_at<12>(f);
    case 13: return dispatch_tc_at<13>(f);
    case 14: return dispatch_tc_at<14>(f);
    case 15: return dispatch_tc_at<15>(f);
    case 16: return dispatch_tc_at<16>(f);
#endif
#if SK_TC_MAX_L > 511 && !defined(SK_TC_ONE_TILE_ONLY)
    case 17: return dispatch_tc_at<17>(f);
    case 18: return dispatch_tc_at<18>(f);
    case 19: return dispatch_tc_at<19>(f);
    case 20: return dispatch_tc_at<20>(f);
    case 21: return dispatch_tc_at<21>(f);
    case 22: return dispatch_tc_at<22>(f);
    case 23: return dispatch_tc_at<23>(f);
    case 24: return dispatch_tc_at<24>(f);
    case 25: return dispatch_tc_at<25>(f);
    case 26: return dispatch_tc_at<26>(f);
    case 27: return dispatch_tc_at<27>(f);
    case 28: return dispatch_tc_at<28>(f);
    case 29: return dispatch_tc_at<29>(f);
    case 30: return dispatch_tc_at<30>(f);
    case 31: return dispatch_tc_at<31>(f);
    case 32: return dispatch_tc_at<32>(f);
#endif
  }
  return fail(SK_ERR_UNSUPPORTED, "no EvalTC instantiation for this length");
}

template <class F>
int dispatch_eval(int L, int nw, bool scalar, F&& f) {
  if (scalar) {
    switch (nw) {
      case 1: return f(std::integral_constant<int, 1>{}, (sk::EvalScalar*)nullptr);
      case 2: return f(std::integral_constant<int, 2>{}, (sk::EvalScalar*)nullptr);
      case 3: return f(std::integral_constant<int, 3>{}, (sk::EvalScalar*)nullptr);
      case 4: return f(std::integral_constant<int, 4>{}, (sk::EvalScalar*)nullptr);
      case 5: return f(std::integral_constant<int, 5>{}, (sk::EvalScalar*)nullptr);
      case 6: return f(std::integral_constant<int, 6>{}, (sk::EvalScalar*)nullptr);
      case 7: return f(std::integral_constant<int, 7>{}, (sk::EvalScalar*)nullptr);
      case 8: return f(std::integral_constant<int, 8>{}, (sk::EvalScalar*)nullptr);
    }
    return fail(SK_ERR_UNSUPPORTED, "unsupported word count");
  }
#ifndef SK_OLD_FAST_EVALUATOR
  // production: the transposed-signal evaluator for every supported length
#ifdef SK_TC_ONE_TILE_ONLY
  if (L > 255) return fail(SK_ERR_UNSUPPORTED, "one-tile development build");
#endif
  return dispatch_tc(L, f);
#else
  // round-1 evaluator, kept for A/B reference builds (-DSK_OLD_FAST_EVALUATOR)
  switch (nw) {
    case 1: return dispatch_fast_small<1>(L, f);
    case 2: return dispatch_fast_small<2>(L, f);
    case 3: return f(std::integral_constant<int, 3>{}, (sk::EvalFast<2>*)nullptr);
    case 4: return f(std::integral_constant<int, 4>{}, (sk::EvalFast<2>*)nullptr);
    case 5: return f(std::integral_constant<int, 5>{}, (sk::EvalFast<3>*)nullptr);
    case 6: return f(std::integral_constant<int, 6>{}, (sk::EvalFast<3>*)nullptr);
    case 7: return f(std::integral_constant<int, 7>{}, (sk::EvalFast<4>*)nullptr);
    case 8: return f(std::integral_constant<int, 8>{}, (sk::EvalFast<4>*)nullptr);
  }
  return fail(SK_ERR_UNSUPPORTED, "unsupported word count");
#endif
}

template <bool TRACE>
int launch_walks(Plan& pl, bool scalar, cudaStream_t st, int dev) {
  return dispatch_eval(pl.P.L, pl.nw, scalar, [&](auto nwc, auto* evp) {
    using Eval = std::remove_pointer_t<decltype(evp)>;
    return launch_nw<decltype(nwc)::value, TRACE, Eval>(pl, st, dev);
  });
}

// R > 0 with masters/batches: multi-search mode, W walks per search
template <bool TRACE>
int run(int L, int n, const uint64_t* seeds, uint64_t master, uint64_t batch, uint64_t walker_begin, int64_t W,
        int64_t* best_e, uint64_t* best_words, int64_t* steps, uint8_t* dead, sk_batch_summary* summary,
        uint64_t* trace_words, int64_t* trace_deltas, cudaStream_t st, const uint64_t* masters = nullptr,
        const uint64_t* batches = nullptr, int R = 1) {
  int rc = validate(L, n, W);
  if (rc) return rc;
  if (summary && walker_begin + uint64_t(W) > (uint64_t(1) << 32))
    return fail(SK_ERR_ARG, "walker_begin + W must be < 2^32 when a summary is requested");
  const int64_t W_rep = W;
  if (masters) {
    if (R < 1) return fail(SK_ERR_ARG, "search count must be >= 1");
    if (W > (int64_t(1) << 40) / R) return fail(SK_ERR_ARG, "R * W too large");
    W = W_rep * R;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  const bool scalar = g_variant == SK_VARIANT_SCALAR || !sk::EvalTC<1>::supports(L);
  Plan pl = scalar ? make_plan<sk::EvalScalar>(L, n) : make_plan<sk::EvalTC<1>>(L, n);
  pl.P.seeds = seeds;
  pl.P.master = master;
  pl.P.batch = batch;
  pl.P.walker_begin = walker_begin;
  pl.P.W = W;
  pl.P.best_e = best_e;
  pl.P.steps_out = steps;
  pl.P.dead_out = dead;
  pl.P.summary = summary;
  pl.P.trace_words = trace_words;
  pl.P.trace_deltas = trace_deltas;
  pl.P.best_words = best_words;
  pl.P.masters = masters;
  pl.P.batches = batches;
  pl.P.W_rep = W_rep;
  if (summary && !best_words && W > 0) {
    DevCache& c = cache_for(dev, st);
    rc = grow(&c.words, &c.words_bytes, size_t(W) * pl.nw * 8u);
    if (rc) return rc;
    pl.P.best_words = static_cast<uint64_t*>(c.words);
  }
  if (summary) {
    sk::summary_init_kernel<<<masters ? R : 1, 32, 0, st>>>(summary);
    SK_CUDA(cudaGetLastError());
  }
  if (W > 0) {
    rc = launch_walks<TRACE>(pl, scalar, st, dev);
    if (rc) return rc;
  }
  if (summary && W > 0) {
    sk::summary_finish_kernel<<<masters ? R : 1, 32, 0, st>>>(summary, pl.P.best_words, pl.nw, walker_begin, W_rep);
    SK_CUDA(cudaGetLastError());
  }
  return SK_OK;
}

// ---- exhaustive scan (exhaustive.cuh) ---------------------------------------
int exh_validate(int L) {
  if (L < 3 || (L % 2) == 0) return fail(SK_ERR_ARG, "length must be odd and >= 3, got " + std::to_string(L));
  if ((L + 1) / 2 > SK_MAX_EXHAUSTIVE_D)
    return fail(SK_ERR_UNSUPPORTED, "L=" + std::to_string(L) + " has D=" + std::to_string((L + 1) / 2) +
                                        " free components; the device scan is capped at D=" +
                                        std::to_string(SK_MAX_EXHAUSTIVE_D));
  return SK_OK;
}

// chunk of consecutive Gray indices per thread: long enough to amortise the
// O(L^2) state rebuild, short enough to give every SM work
int exh_chunk_log2(int D) { return std::max(4, std::min(16, D - 19)); }

template <int G>
int exh_launch(int L, uint64_t g_begin, uint64_t g_end, unsigned long long* key, cudaStream_t st, int dev) {
  auto kern = sk::exhaustive_kernel<G>;
  const int cl2 = exh_chunk_log2((L + 1) / 2);
  const uint64_t nchunks = ((g_end - g_begin) + (1ull << cl2) - 1) >> cl2;
  int sms = 0, per = 0;
  SK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0));
  const uint64_t want = (nchunks + 255) / 256;
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(std::max(per, 1)) * sms));
  kern<<<unsigned(grid), 256, 0, st>>>(L, g_begin, g_end, cl2, key);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

// lag groups of four: G = ceil(K / 4), bucketed (unused lags are C = 0 bytes)
int exh_run(int L, uint64_t g_begin, uint64_t g_end, unsigned long long* key, cudaStream_t st, int dev) {
  const int K = (L + 1) / 2 - 1;
  const int G = (K + 3) / 4;
  if (G <= 4) return exh_launch<4>(L, g_begin, g_end, key, st, dev);
  if (G <= 6) return exh_launch<6>(L, g_begin, g_end, key, st, dev);
  if (G <= 8) return exh_launch<8>(L, g_begin, g_end, key, st, dev);
  if (G <= 9) return exh_launch<9>(L, g_begin, g_end, key, st, dev);
  if (G <= 10) return exh_launch<10>(L, g_begin, g_end, key, st, dev);
  if (G <= 11) return exh_launch<11>(L, g_begin, g_end, key, st, dev);
  return exh_launch<12>(L, g_begin, g_end, key, st, dev);
}

__global__ void exh_key_init(unsigned long long* k) { *k = ~0ull; }

}  // namespace

extern "C" {

int sk_abi_version(void) { return SK_ABI_VERSION; }
const char* sk_last_error(void) { return g_err.c_str(); }
int sk_max_length(void) { return SK_MAX_L; }

int sk_set_variant(int v) {
  if (v != SK_VARIANT_AUTO && v != SK_VARIANT_SCALAR && v != SK_VARIANT_FAST)
    return fail(SK_ERR_ARG, "unknown variant " + std::to_string(v));
  g_variant = v;
  return SK_OK;
}
int sk_get_variant(void) { return g_variant; }

int sk_set_visited_layout(int mode) {
  if (mode != SK_VISITED_AUTO && mode != SK_VISITED_SMEM && mode != SK_VISITED_FINGERPRINT &&
      mode != SK_VISITED_GLOBAL)
    return fail(SK_ERR_ARG, "unknown visited-set layout " + std::to_string(mode));
  g_visited = mode;
  return SK_OK;
}

int sk_saw_batch(int L, int n, const uint64_t* d_seeds, uint64_t master_seed, uint64_t batch, uint64_t walker_begin,
                 int64_t W, int64_t* d_best_e, uint64_t* d_best_words, int64_t* d_steps, uint8_t* d_dead,
                 sk_batch_summary* d_summary, void* stream) {
  return run<false>(L, n, d_seeds, master_seed, batch, walker_begin, W, d_best_e, d_best_words, d_steps, d_dead,
                    d_summary, nullptr, nullptr, static_cast<cudaStream_t>(stream));
}

int sk_saw_multi(int L, int n, const uint64_t* d_masters, const uint64_t* d_batches, int R, uint64_t walker_begin,
                 int64_t W, sk_batch_summary* d_summaries, void* stream) {
  if (!d_masters || !d_batches || !d_summaries) return fail(SK_ERR_ARG, "sk_saw_multi needs masters, batches, summaries");
  if (R < 1) return fail(SK_ERR_ARG, "search count R must be >= 1");
  return run<false>(L, n, nullptr, 0, 0, walker_begin, W, nullptr, nullptr, nullptr, nullptr, d_summaries, nullptr,
                    nullptr, static_cast<cudaStream_t>(stream), d_masters, d_batches, R);
}

int sk_saw_trace(int L, int n, const uint64_t* d_seeds, int64_t W, int64_t* d_best_e, uint64_t* d_best_words,
                 int64_t* d_steps, uint8_t* d_dead, uint64_t* d_trace_words, int64_t* d_trace_deltas, void* stream) {
  if (!d_seeds || !d_trace_words || !d_trace_deltas) return fail(SK_ERR_ARG, "sk_saw_trace needs seeds and trace buffers");
  return run<true>(L, n, d_seeds, 0, 0, 0, W, d_best_e, d_best_words, d_steps, d_dead, nullptr, d_trace_words,
                   d_trace_deltas, static_cast<cudaStream_t>(stream));
}

int sk_saw_batch_host(int L, int n, const uint64_t* seeds, int64_t W, int64_t* best_e_out, uint64_t* best_words_out,
                      int64_t* steps_out, uint8_t* dead_out) {
  int rc = validate(L, n, W);
  if (rc) return rc;
  if (W == 0) return SK_OK;
  if (!seeds || !best_e_out || !best_words_out || !steps_out || !dead_out)
    return fail(SK_ERR_ARG, "sk_saw_batch_host: null buffer");
  const int D = (L + 1) / 2, nw = (D + 63) / 64;
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  const size_t in_b = size_t(W) * 8;
  const size_t o_e = 0, o_w = o_e + size_t(W) * 8, o_s = o_w + size_t(W) * nw * 8, o_d = o_s + size_t(W) * 8;
  const size_t out_b = o_d + size_t(W);
  char *din, *dout;
  std::lock_guard<std::mutex> hlk(g_host_mu);  // staging buffers are reused: one host call at a time
  {
    std::lock_guard<std::mutex> lk(g_mu);
    DevCache& c = cache_for(dev, nullptr);
    rc = grow(&c.h_in, &c.h_in_bytes, in_b);
    if (rc) return rc;
    rc = grow(&c.h_out, &c.h_out_bytes, out_b);
    if (rc) return rc;
    din = static_cast<char*>(c.h_in);
    dout = static_cast<char*>(c.h_out);
  }
  cudaStream_t st = 0;
  SK_CUDA(cudaMemcpyAsync(din, seeds, in_b, cudaMemcpyHostToDevice, st));
  rc = run<false>(L, n, reinterpret_cast<const uint64_t*>(din), 0, 0, 0, W, reinterpret_cast<int64_t*>(dout + o_e),
                  reinterpret_cast<uint64_t*>(dout + o_w), reinterpret_cast<int64_t*>(dout + o_s),
                  reinterpret_cast<uint8_t*>(dout + o_d), nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  SK_CUDA(cudaMemcpyAsync(best_e_out, dout + o_e, size_t(W) * 8, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(best_words_out, dout + o_w, size_t(W) * nw * 8, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(steps_out, dout + o_s, size_t(W) * 8, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(dead_out, dout + o_d, size_t(W), cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaStreamSynchronize(st));
  return SK_OK;
}

int sk_saw_walk_host(int L, int n, uint64_t seed, uint64_t* best_words, uint64_t* trace_words, int64_t* trace_deltas,
                     int record, int64_t* best_e_out, int64_t* steps_out, uint8_t* dead_out) {
  int rc = validate(L, n, 1);
  if (rc) return rc;
  if (!best_words || !best_e_out || !steps_out || !dead_out) return fail(SK_ERR_ARG, "sk_saw_walk_host: null buffer");
  if (record && (!trace_words || !trace_deltas)) return fail(SK_ERR_ARG, "sk_saw_walk_host: record needs trace buffers");
  const int D = (L + 1) / 2, nw = (D + 63) / 64;
  const size_t tw_b = record ? size_t(n + 1) * nw * 8 : 0, td_b = record ? size_t(n) * D * 8 : 0;
  const size_t o_seed = 0, o_e = 8, o_s = 16, o_d = 24, o_w = 32, o_tw = o_w + size_t(nw) * 8, o_td = o_tw + tw_b;
  std::lock_guard<std::mutex> hlk(g_host_mu);  // the staging buffer is reused: one host call at a time
  char* buf = nullptr;
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_mu);
    DevCache& c = cache_for(dev, nullptr);
    rc = grow(&c.h_walk, &c.h_walk_bytes, o_td + td_b);  // cached: no cudaMalloc per replayed walk
    if (rc) return rc;
    buf = static_cast<char*>(c.h_walk);
  }
  cudaStream_t st = 0;
  SK_CUDA(cudaMemcpyAsync(buf + o_seed, &seed, 8, cudaMemcpyHostToDevice, st));
  if (record) {
    rc = run<true>(L, n, reinterpret_cast<uint64_t*>(buf + o_seed), 0, 0, 0, 1, reinterpret_cast<int64_t*>(buf + o_e),
                   reinterpret_cast<uint64_t*>(buf + o_w), reinterpret_cast<int64_t*>(buf + o_s),
                   reinterpret_cast<uint8_t*>(buf + o_d), nullptr, reinterpret_cast<uint64_t*>(buf + o_tw),
                   reinterpret_cast<int64_t*>(buf + o_td), st);
  } else {
    rc = run<false>(L, n, reinterpret_cast<uint64_t*>(buf + o_seed), 0, 0, 0, 1, reinterpret_cast<int64_t*>(buf + o_e),
                    reinterpret_cast<uint64_t*>(buf + o_w), reinterpret_cast<int64_t*>(buf + o_s),
                    reinterpret_cast<uint8_t*>(buf + o_d), nullptr, nullptr, nullptr, st);
  }
  if (rc) return rc;
  SK_CUDA(cudaMemcpyAsync(best_e_out, buf + o_e, 8, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(steps_out, buf + o_s, 8, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(dead_out, buf + o_d, 1, cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaMemcpyAsync(best_words, buf + o_w, size_t(nw) * 8, cudaMemcpyDeviceToHost, st));
  if (record) {
    // rows past the walk's end are left untouched by the kernel: copy only
    // what was written so that caller-initialised rows survive (saw.py:108-110)
    SK_CUDA(cudaStreamSynchronize(st));
    const int64_t rows_w = *steps_out + 1, rows_d = *steps_out + (*dead_out ? 1 : 0);
    SK_CUDA(cudaMemcpyAsync(trace_words, buf + o_tw, size_t(rows_w) * nw * 8, cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaMemcpyAsync(trace_deltas, buf + o_td, size_t(rows_d) * D * 8, cudaMemcpyDeviceToHost, st));
  }
  SK_CUDA(cudaStreamSynchronize(st));
  return SK_OK;
}

int64_t sk_resident_walks(int L, int n) {
  if (validate(L, n, 1)) return -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  const bool scalar = g_variant == SK_VARIANT_SCALAR || !sk::EvalTC<1>::supports(L);
  Plan pl = scalar ? make_plan<sk::EvalScalar>(L, n) : make_plan<sk::EvalTC<1>>(L, n);
  pl.P.W = int64_t(1) << 40;
  pl.dry_run = true;
  const int rc = launch_walks<false>(pl, scalar, 0, dev);
  return rc ? -1 : pl.resident;
}

int sk_exhaustive_scan(int L, uint64_t g_begin, uint64_t g_count, uint64_t* d_min_key, void* stream) {
  int rc = exh_validate(L);
  if (rc) return rc;
  if (!d_min_key) return fail(SK_ERR_ARG, "sk_exhaustive_scan: null key");
  const int D = (L + 1) / 2;
  const uint64_t total = 1ull << D;
  if (g_begin > total || g_count > total - g_begin)
    return fail(SK_ERR_ARG, "Gray index range exceeds 2^D");
  if (g_count == 0) return SK_OK;
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  return exh_run(L, g_begin, g_begin + g_count, reinterpret_cast<unsigned long long*>(d_min_key),
                 static_cast<cudaStream_t>(stream), dev);
}

int sk_exhaustive_scan_host(int L, int64_t* best_e_out, int64_t* best_bits_out) {
  int rc = exh_validate(L);
  if (rc) return rc;
  if (!best_e_out || !best_bits_out) return fail(SK_ERR_ARG, "sk_exhaustive_scan_host: null output");
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  unsigned long long* dkey = nullptr;
  SK_CUDA(cudaMalloc(&dkey, 8));
  cudaStream_t st = 0;
  exh_key_init<<<1, 1, 0, st>>>(dkey);
  const int D = (L + 1) / 2;
  const uint64_t total = 1ull << D, slice = 1ull << 36;  // bounded launches (~0.6 s each at D = 44)
  for (uint64_t b = 0; b < total && rc == SK_OK; b += slice) rc = exh_run(L, b, std::min(total, b + slice), dkey, st, dev);
  unsigned long long key = 0;
  if (rc == SK_OK && cudaMemcpy(&key, dkey, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(SK_ERR_CUDA, std::string("sk_exhaustive_scan_host: ") + cudaGetErrorString(cudaGetLastError()));
  cudaFree(dkey);
  if (rc) return rc;
  const uint64_t g = key & ((1ull << sk::kExhKeyShift) - 1);
  if (int64_t(key >> sk::kExhKeyShift) >= sk::kExhEMax)
    return fail(SK_ERR_UNSUPPORTED, "minimum energy beyond the scan's key range");
  *best_e_out = int64_t(key >> sk::kExhKeyShift);
  *best_bits_out = int64_t(g ^ (g >> 1));
  return SK_OK;
}

// ---- batched neighbourhood (neighborhood.cuh) --------------------------------
static int nb_grid(int64_t S, int dev, int* grid) {
  int sms = 0;
  SK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t want = (S + 7) / 8;  // 8 warps (states) per 256-thread block
  *grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 8)));
  return SK_OK;
}

int sk_all_neighbor_deltas(int L, int64_t S, const int64_t* d_s, const int64_t* d_c, int64_t* d_deltas, void* stream) {
  int rc = validate(L, 1, S);
  if (rc) return rc;
  if (S == 0) return SK_OK;
  if (!d_s || !d_c || !d_deltas) return fail(SK_ERR_ARG, "sk_all_neighbor_deltas: null buffer");
  int dev = 0, grid = 1;
  SK_CUDA(cudaGetDevice(&dev));
  if ((rc = nb_grid(S, dev, &grid))) return rc;
  sk::neighbor_deltas_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(L, S, d_s, d_c, d_deltas);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

int sk_apply_neighbor(int L, int64_t S, int64_t* d_s, int64_t* d_c, const int64_t* d_h, void* stream) {
  int rc = validate(L, 1, S);
  if (rc) return rc;
  if (S == 0) return SK_OK;
  if (!d_s || !d_c || !d_h) return fail(SK_ERR_ARG, "sk_apply_neighbor: null buffer");
  int dev = 0, grid = 1;
  SK_CUDA(cudaGetDevice(&dev));
  if ((rc = nb_grid(S, dev, &grid))) return rc;
  sk::apply_neighbor_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(L, S, d_s, d_c, d_h);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

int sk_eval_states(int L, int64_t S, const int8_t* d_halves, int M, const int32_t* d_moves, int64_t* d_deltas,
                   void* stream) {
  int rc = validate(L, 1, S);
  if (rc) return rc;
  if (M < 0) return fail(SK_ERR_ARG, "move count must be >= 0");
  if (S == 0) return SK_OK;
  if (!d_halves || !d_deltas || (M > 0 && !d_moves)) return fail(SK_ERR_ARG, "sk_eval_states: null buffer");
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0, sms = 0;
  SK_CUDA(cudaGetDevice(&dev));
  SK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int D = (L + 1) / 2, nw = (D + 63) / 64;
  const bool scalar = g_variant == SK_VARIANT_SCALAR || !sk::EvalTC<1>::supports(L);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dispatch_eval(L, nw, scalar, [&](auto nwc, auto* evp) {
    using Eval = std::remove_pointer_t<decltype(evp)>;
    Plan pl = make_plan<Eval>(L, 1);
    const sk::SmemLayout lay = pl.lay[SK_VISITED_GLOBAL];  // no visited set: the smallest layout
    pl.P.W = S;
    pl.P.warp_smem = lay.total;
    pl.P.block_smem = Eval::block_bytes(L);
    auto kern = sk::eval_states_kernel<decltype(nwc)::value, Eval, kWPB>;
    const size_t smem = pl.P.block_smem + size_t(lay.total) * kWPB;
    SK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per = 0;
    SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kWPB * 32, smem));
    if (per < 1) return fail(SK_ERR_UNSUPPORTED, "evaluator state does not fit one SM");
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((S + kWPB - 1) / kWPB, int64_t(per) * sms));
    kern<<<dim3(unsigned(grid)), dim3(kWPB * 32), smem, st>>>(pl.P, lay, d_halves, M, d_moves, d_deltas);
    SK_CUDA(cudaGetLastError());
    return SK_OK;
  });
}

int sk_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_cache) {
    DevCache& c = kv.second;
    if (!c.gkeys && !c.words && !c.h_in && !c.h_out && !c.h_walk) continue;
    cudaSetDevice(kv.first.first);
    if (c.gkeys) cudaFree(c.gkeys);
    if (c.words) cudaFree(c.words);
    if (c.h_in) cudaFree(c.h_in);
    if (c.h_out) cudaFree(c.h_out);
    if (c.h_walk) cudaFree(c.h_walk);
  }
  g_cache.clear();
  cudaSetDevice(cur);
  return SK_OK;
}

}  // extern "C"
