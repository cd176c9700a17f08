/*
 * sokol.h -- C ABI of libsokol.so, the B200 (sm_100a) self-avoiding-walk
 * engine for skew-symmetric LABS (arXiv 2210.15962, "sokol_skew").
 *
 * This is the drop-in boundary for the reference's hot path, the numba
 * kernels in /root/reference/pkg/src/skewsaw/_kernels.py.  Each entry point
 * names the reference interface it replaces (file:line).  Plain pointers and
 * sizes only; no torch types.  Every call returns SK_OK (0) or a negative
 * SK_ERR_* code, with a message available from sk_last_error().
 *
 * Data conventions (identical to the reference, _kernels.py:1-13):
 *   L odd, 3 <= L <= SK_MAX_L;  D = (L+1)/2 free spins;  nw = ceil(D/64).
 *   words: little-endian uint64, bit D-1-h set iff half spin h is -1
 *          (equals the hex codec integer, codec.py:34-41).
 *   seeds: per-walk uint64 seeds as produced by derive_walk_seed
 *          (runner.py:53-57).
 *
 * Concurrency: device entry points are asynchronous on the given stream and
 * may run concurrently on different streams (internal scratch is private per
 * (device, stream)).  The *_host entry points are synchronous and serialised.
 */
#ifndef SOKOL_H
#define SOKOL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 1
#define SK_MAX_L 1023   /* D <= 512, nw <= 8 */
#define SK_MAX_WORDS 8

#define SK_OK 0
#define SK_ERR_ARG (-1)         /* invalid argument (L even / out of range, n < 1, W < 0, null) */
#define SK_ERR_UNSUPPORTED (-2) /* valid for the reference but beyond SK_MAX_L */
#define SK_ERR_CUDA (-3)        /* CUDA runtime error (message in sk_last_error) */
#define SK_ERR_NOMEM (-4)       /* device or host allocation failed */

/* Kernel variants (sk_set_variant).  All produce identical results. */
#define SK_VARIANT_AUTO 0
#define SK_VARIANT_SCALAR 1 /* reference-formula scalar evaluator (cross-check) */
#define SK_VARIANT_FAST 2   /* production evaluator */

/*
 * Per-batch reduction written by sk_saw_batch (device memory).  The merge of
 * runner.py:252-256 (lowest energy wins, ties to the lowest walker index) is
 * a min over min_key = (best_E << 32) | global_walker_index.
 */
typedef struct sk_batch_summary {
    uint64_t min_key;                  /* (best_E << 32) | walker (global index) */
    int64_t steps_sum;                 /* sum of steps over the batch's walks (runner.py:251) */
    uint64_t best_words[SK_MAX_WORDS]; /* packed best half of the winning walk */
} sk_batch_summary;

int sk_abi_version(void);
const char *sk_last_error(void);
int sk_max_length(void);

/* Select the evaluator used by subsequent calls (process-global). */
int sk_set_variant(int variant);
int sk_get_variant(void);

/*
 * Visited-set layout of subsequent walk launches (process-global).  AUTO
 * picks by occupancy; SMEM keeps the 64-bit keys in shared memory;
 * FINGERPRINT keeps 32-bit fingerprints in shared memory and the keys in an
 * L2-resident global scratch; GLOBAL keeps only an occupancy bitmap in shared
 * memory and the keys in the scratch.  Membership, and so every result, is
 * identical in all of them.
 */
#define SK_VISITED_AUTO 0
#define SK_VISITED_SMEM 1
#define SK_VISITED_FINGERPRINT 2
#define SK_VISITED_GLOBAL 3
int sk_set_visited_layout(int mode);

/*
 * Batch of independent walks on the current CUDA device, asynchronous on
 * `stream` (a cudaStream_t; NULL = legacy default stream).
 * Replaces skewsaw._kernels.saw_batch(length, n, seeds, best_e_out,
 * best_words_out, steps_out, dead_out)  (_kernels.py:278-287), called by
 * runner._BatchLoop.run_batch (runner.py:232-256).
 *
 *   d_seeds      W device seeds, or NULL: seed[i] is derived on device as
 *                derive_walk_seed(master_seed, batch, walker_begin + i).
 *   d_best_e, d_best_words [W*nw], d_steps, d_dead:  per-walk outputs in
 *                device memory; each may be NULL (throughput mode).
 *   d_summary    device sk_batch_summary, or NULL.  Overwritten (not
 *                accumulated) by this call; walker indices in min_key are
 *                global (walker_begin + i).
 */
int sk_saw_batch(int L, int n, const uint64_t *d_seeds, uint64_t master_seed, uint64_t batch,
                 uint64_t walker_begin, int64_t W, int64_t *d_best_e, uint64_t *d_best_words,
                 int64_t *d_steps, uint8_t *d_dead, sk_batch_summary *d_summary, void *stream);

/*
 * R independent searches in one launch: the batch step
 * of R concurrent solves, as run by runner.target_campaign
 * (runner.py:294-317), whose repetitions the reference runs one after the
 * other, each a full runner.solve batch loop (runner.py:213-291).
 * Search r runs walkers [walker_begin, walker_begin + W) of batch
 * d_batches[r] under master seed d_masters[r] (seeds derived on device
 * exactly as sk_saw_batch with d_seeds == NULL) and writes d_summaries[r],
 * which is therefore identical to the summary sk_saw_batch gives for that
 * (master, batch, walker range).  Device arrays of R entries; asynchronous.
 */
int sk_saw_multi(int L, int n, const uint64_t *d_masters, const uint64_t *d_batches, int R,
                 uint64_t walker_begin, int64_t W, sk_batch_summary *d_summaries, void *stream);

/*
 * Traced batch: as sk_saw_batch plus the trajectory record of
 * _kernels.py:231-243, 267-270 (record=True), device memory:
 *   d_trace_words  [W][n+1][nw]  pivot after t moves (row 0 = first pivot)
 *   d_trace_deltas [W][n][D]     raw delta vector evaluated at pivot t
 *                                (a dead walk records one extra row)
 * Rows beyond a walk's steps (+1 if dead) are left untouched.
 */
int sk_saw_trace(int L, int n, const uint64_t *d_seeds, int64_t W, int64_t *d_best_e,
                 uint64_t *d_best_words, int64_t *d_steps, uint8_t *d_dead,
                 uint64_t *d_trace_words, int64_t *d_trace_deltas, void *stream);

/*
 * Host-buffer drop-in of skewsaw._kernels.saw_batch (_kernels.py:278-287):
 * identical argument list and meaning (host C-contiguous arrays, outputs
 * written in place).  Copies seeds in, runs on the current device, copies
 * outputs back, synchronises.  This is the call a ctypes binding of the
 * reference's batch kernel makes.
 */
int sk_saw_batch_host(int L, int n, const uint64_t *seeds, int64_t W, int64_t *best_e_out,
                      uint64_t *best_words_out, int64_t *steps_out, uint8_t *dead_out);

/*
 * Host-buffer drop-in of skewsaw._kernels.saw_walk(length, n, seed,
 * best_words, trace_words, trace_deltas, record) -> (best_e, steps, dead)
 * (_kernels.py:189-275, called by saw._walk, saw.py:104-130).
 * trace_words [n+1][nw] and trace_deltas [n][D] are read only if record != 0.
 */
int sk_saw_walk_host(int L, int n, uint64_t seed, uint64_t *best_words, uint64_t *trace_words,
                     int64_t *trace_deltas, int record, int64_t *best_e_out, int64_t *steps_out,
                     uint8_t *dead_out);

/*
 * Device count of resident walk slots the batch kernel uses for (L, n) on the
 * current device (persistent grid size in warps).  Informational.
 */
int64_t sk_resident_walks(int L, int n);

/*
 * Exhaustive Gray-code scan of the half-sequence space on the current device
 * (SURVEY §8(f) row 2).  Replaces skewsaw._kernels.exhaustive_scan(length)
 * (_kernels.py:290-323), called by saw.exhaustive_optimum (saw.py:151-168),
 * whose single-threaded loop is capped at D <= 28 (saw.py:36); the device
 * scan accepts D <= SK_MAX_EXHAUSTIVE_D.
 *
 * sk_exhaustive_scan: Gray indices g in [g_begin, g_begin + g_count) (the
 *   half after reference step g is gray(g) = g ^ (g >> 1); g = 0 is the
 *   all-plus start), asynchronous on `stream`.  Folds
 *   key = (min(E, 2^17 - 1) << 47) | g into *d_min_key with an atomic min
 *   (optima lie far below the saturation), so the caller
 *   initialises it to UINT64_MAX and may split the space into any slices;
 *   the final key's (E, g) is the reference's first minimum.
 * sk_exhaustive_scan_host: the whole space, synchronous; returns exactly the
 *   reference's (best_energy, best_bits), bit h of best_bits set iff half
 *   spin h is -1.
 */
#define SK_MAX_EXHAUSTIVE_D 47
int sk_exhaustive_scan(int L, uint64_t g_begin, uint64_t g_count, uint64_t *d_min_key, void *stream);
int sk_exhaustive_scan_host(int L, int64_t *best_e_out, int64_t *best_bits_out);

/*
 * Batched neighbourhood evaluation and moves, S
 * independent states in the reference's own array layout, device memory,
 * asynchronous on `stream`:
 *   d_s [S][L] int64 full +-1 sequence,  d_c [S][L] int64, d_c[k] = C_k,
 *   d_deltas [S][D] int64,  d_h [S] int64 half index in [0, D).
 * sk_all_neighbor_deltas replaces skewsaw._kernels.all_neighbor_deltas(s, c,
 *   out) (_kernels.py:162-165 over neighbor_delta, 85-123), called by
 *   neighborhood.compute_deltas (neighborhood.py:80-90).
 * sk_apply_neighbor replaces skewsaw._kernels.apply_neighbor(s, c, h)
 *   (_kernels.py:126-158), called by neighborhood.apply_flip
 *   (neighborhood.py:93-100); a state whose h is out of range is left
 *   unchanged (the Python layer raises before calling, as the reference does).
 * Same int64 four-product arithmetic as the reference, for any +-1 input.
 */
int sk_all_neighbor_deltas(int L, int64_t S, const int64_t *d_s, const int64_t *d_c, int64_t *d_deltas,
                           void *stream);
int sk_apply_neighbor(int L, int64_t S, int64_t *d_s, int64_t *d_c, const int64_t *d_h, void *stream);

/*
 * Evaluator probe: the walk kernels' own neighbourhood evaluator (the one
 * sk_saw_batch selects for L under the current variant) run on S caller-given
 * states instead of walk pivots.  Device memory, asynchronous on `stream`:
 *   d_halves [S][D] int8 half sequences (+-1);
 *   d_moves  [S][M] int32 half indices applied in order (M may be 0; an index
 *            outside [0, D) leaves the state unchanged);
 *   d_deltas [S][M+1][D] int64: row 0 = all_neighbor_deltas of the start
 *            state (_kernels.py:162-165 over neighbor_delta, 85-123), row
 *            i+1 = the same after apply_neighbor(moves[i]) (126-158).
 * Exactly the rows the traced walk records (_kernels.py:241-243), for
 * arbitrary (e.g. maximal-|C_k|) states; used to test the evaluator at its
 * exactness bounds.
 */
int sk_eval_states(int L, int64_t S, const int8_t *d_halves, int M, const int32_t *d_moves, int64_t *d_deltas,
                   void *stream);

/* Release the library's cached device buffers (safe to call at any time). */
int sk_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* SOKOL_H */
