/*
 * sokol_oracle.c -- CPU restatement of the reference's SAW hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2210_15962_b200/ links, imports
 * or executes this file; it is the checker that tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs compare the CUDA path
 * against.  It is pinned to the real reference by tests/golden/ (fixtures
 * produced by oracle/gen_golden.py, which imports /root/reference/pkg/src).
 *
 * Every function restates one numba kernel of the reference; citations are to
 * /root/reference/pkg/src/skewsaw/.  The arithmetic is the reference's own
 * (int64 spins, natural-order correlation vector, per-neighbour O(L) delta),
 * deliberately NOT the GPU formulation, so that the two are independent.
 *
 * Conventions (identical to _kernels.py:1-13):
 *   s[0..L-1]   full +-1 sequence, c[k] = C_k (c[0] = L)
 *   words[nw]   little-endian uint64 words; bit D-1-h set iff half spin h is -1
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define SO_GOLDEN 0x9E3779B97F4A7C15ULL   /* _kernels.py:22 */
#define SO_KEY_SEED 0xA0761D6478BD642FULL /* _kernels.py:23 */
#define SO_REP_STREAM 0xD1B54A32D192ED03ULL /* runner.py:43 */

/* splitmix64 finaliser, _kernels.py:32-37 (bijection on uint64). */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t so_mix64(uint64_t z) { return mix64(z); }

/* key_of_words, _kernels.py:46-53. */
uint64_t so_key_of_words(const uint64_t *words, int nw) {
    uint64_t h = SO_KEY_SEED;
    for (int i = 0; i < nw; i++) h = mix64(h ^ words[i]);
    return h;
}

/* derive_walk_seed, runner.py:53-57. */
uint64_t so_derive_walk_seed(uint64_t master, uint64_t batch, uint64_t walker) {
    uint64_t h = mix64(master ^ SO_GOLDEN);
    h = mix64(h ^ batch);
    return mix64(h ^ walker);
}

/* derive_repetition_seed, runner.py:60-62. */
uint64_t so_derive_repetition_seed(uint64_t master, uint64_t rep) {
    uint64_t h = mix64(master ^ SO_REP_STREAM);
    return mix64(h ^ rep);
}

/* expand_in_place, _kernels.py:62-67. */
static void expand_in_place(int64_t *s, int d) {
    int64_t sign = -1;
    for (int i = 1; i < d; i++) {
        s[d - 1 + i] = sign * s[d - 1 - i];
        sign = -sign;
    }
}

/* init_sidelobes, _kernels.py:70-82: all C_k and E = sum_{k>=1} C_k^2. */
static int64_t init_sidelobes(const int64_t *s, int64_t *c, int L) {
    int64_t e = 0;
    for (int k = 0; k < L; k++) {
        int64_t acc = 0;
        for (int i = 0; i < L - k; i++) acc += s[i] * s[i + k];
        c[k] = acc;
        if (k > 0) e += acc * acc;
    }
    return e;
}

/* neighbor_delta, _kernels.py:85-123: exact dE for flipping half index h. */
static int64_t neighbor_delta(const int64_t *s, const int64_t *c, int L, int h) {
    const int p = h, q = L - 1 - h;
    const int64_t sp = s[p];
    int64_t acc = 0;
    if (p == q) {
        for (int k = 2; k < L; k += 2) {
            int64_t d = 0;
            if (p + k < L) d -= sp * s[p + k];
            if (p - k >= 0) d -= s[p - k] * sp;
            d += d;
            acc += d * (2 * c[k] + d);
        }
    } else {
        const int64_t sq = s[q];
        for (int k = 2; k < L; k += 2) {
            int64_t d = 0;
            const int pk = p + k, qk = q - k;
            if (pk < L && pk != q) d -= sp * s[pk];
            if (p - k >= 0) d -= s[p - k] * sp;
            if (q + k < L) d -= sq * s[q + k];
            if (qk >= 0 && qk != p) d -= s[qk] * sq;
            d += d;
            acc += d * (2 * c[k] + d);
        }
    }
    return acc;
}

/* apply_neighbor, _kernels.py:126-158. */
static void apply_neighbor(int64_t *s, int64_t *c, int L, int h) {
    const int p = h, q = L - 1 - h;
    const int64_t sp = s[p];
    if (p == q) {
        for (int k = 2; k < L; k += 2) {
            int64_t d = 0;
            if (p + k < L) d -= sp * s[p + k];
            if (p - k >= 0) d -= s[p - k] * sp;
            c[k] += 2 * d;
        }
        s[p] = -sp;
    } else {
        const int64_t sq = s[q];
        for (int k = 2; k < L; k += 2) {
            int64_t d = 0;
            const int pk = p + k, qk = q - k;
            if (pk < L && pk != q) d -= sp * s[pk];
            if (p - k >= 0) d -= s[p - k] * sp;
            if (q + k < L) d -= sq * s[q + k];
            if (qk >= 0 && qk != p) d -= s[qk] * sq;
            c[k] += 2 * d;
        }
        s[p] = -sp;
        s[q] = -sq;
    }
}

/* Public wrappers for the neighbourhood API (neighborhood.py:73-100). */
void so_all_neighbor_deltas(int L, const int64_t *s, const int64_t *c, int64_t *out) {
    const int d = (L + 1) / 2;
    for (int h = 0; h < d; h++) out[h] = neighbor_delta(s, c, L, h);
}

void so_apply_neighbor(int L, int64_t *s, int64_t *c, int h) { apply_neighbor(s, c, L, h); }

int64_t so_init_sidelobes(int L, const int64_t *s, int64_t *c) { return init_sidelobes(s, c, L); }

/* Open-addressed visited set, _kernels.py:168-186 (linear probing). */
static int visited_contains(const uint64_t *table, const uint8_t *used, int64_t mask, uint64_t key) {
    int64_t idx = (int64_t)(key & (uint64_t)mask);
    while (used[idx]) {
        if (table[idx] == key) return 1;
        idx = (idx + 1) & mask;
    }
    return 0;
}

static void visited_add(uint64_t *table, uint8_t *used, int64_t mask, uint64_t key) {
    int64_t idx = (int64_t)(key & (uint64_t)mask);
    while (used[idx]) {
        if (table[idx] == key) return;
        idx = (idx + 1) & mask;
    }
    table[idx] = key;
    used[idx] = 1;
}

/*
 * saw_walk, _kernels.py:189-275.  Returns 0, or -1 on allocation failure.
 * trace_words[(n+1)*nw] and trace_deltas[n*D] are written when record != 0.
 */
int so_saw_walk(int L, int n, uint64_t seed, uint64_t *best_words, int nw,
                uint64_t *trace_words, int64_t *trace_deltas, int record,
                int64_t *best_e_out, int64_t *steps_out, uint8_t *dead_out) {
    const int d = (L + 1) / 2;
    int64_t cap = 1;
    while (cap < 2 * ((int64_t)n + 1)) cap <<= 1;
    const int64_t mask = cap - 1;

    int64_t *s = (int64_t *)malloc(sizeof(int64_t) * L);
    int64_t *c = (int64_t *)calloc(L, sizeof(int64_t));
    int64_t *deltas = (int64_t *)malloc(sizeof(int64_t) * d);
    uint64_t *words = (uint64_t *)calloc(nw, sizeof(uint64_t));
    uint64_t *table = (uint64_t *)calloc(cap, sizeof(uint64_t));
    uint8_t *used = (uint8_t *)calloc(cap, 1);
    if (!s || !c || !deltas || !words || !table || !used) {
        free(s); free(c); free(deltas); free(words); free(table); free(used);
        return -1;
    }

    /* first pivot: _next64 stream (_kernels.py:40-43, 204-208) */
    uint64_t state = seed;
    for (int h = 0; h < d; h++) {
        state += SO_GOLDEN;
        const uint64_t z = mix64(state);
        s[h] = 1 - 2 * (int64_t)(z >> 63);
    }
    expand_in_place(s, d);
    int64_t e = init_sidelobes(s, c, L);

    for (int h = 0; h < d; h++) {
        if (s[h] < 0) {
            const int b = d - 1 - h;
            words[b >> 6] |= 1ULL << (b & 63);
        }
    }
    visited_add(table, used, mask, so_key_of_words(words, nw));

    int64_t best_e = e;
    memcpy(best_words, words, sizeof(uint64_t) * nw);
    if (record) memcpy(trace_words, words, sizeof(uint64_t) * nw);

    int64_t steps = 0;
    uint8_t dead = 0;
    for (int step = 0; step < n; step++) {
        for (int h = 0; h < d; h++) deltas[h] = neighbor_delta(s, c, L, h);
        if (record) memcpy(trace_deltas + (int64_t)step * d, deltas, sizeof(int64_t) * d);
        int best_h = -1;
        int64_t best_d = 0;
        uint64_t best_key = 0;
        for (int h = 0; h < d; h++) {
            if (best_h >= 0 && deltas[h] >= best_d) continue;
            const int b = d - 1 - h;
            const uint64_t bit = 1ULL << (b & 63);
            words[b >> 6] ^= bit;
            const uint64_t nk = so_key_of_words(words, nw);
            words[b >> 6] ^= bit;
            if (!visited_contains(table, used, mask, nk)) {
                best_h = h;
                best_d = deltas[h];
                best_key = nk;
            }
        }
        if (best_h < 0) {
            dead = 1;
            break;
        }
        apply_neighbor(s, c, L, best_h);
        e += best_d;
        const int b = d - 1 - best_h;
        words[b >> 6] ^= 1ULL << (b & 63);
        visited_add(table, used, mask, best_key);
        steps += 1;
        if (record) memcpy(trace_words + steps * nw, words, sizeof(uint64_t) * nw);
        if (e < best_e) {
            best_e = e;
            memcpy(best_words, words, sizeof(uint64_t) * nw);
        }
    }
    *best_e_out = best_e;
    *steps_out = steps;
    *dead_out = dead;
    free(s); free(c); free(deltas); free(words); free(table); free(used);
    return 0;
}

/*
 * saw_batch, _kernels.py:278-287: one walk per seed.  Walks are independent,
 * so the thread schedule (a shared atomic work counter over pthreads, the
 * analogue of numba's prange) cannot change any output.  threads <= 0 means
 * all online cores.
 */
typedef struct {
    int L, n, nw;
    const uint64_t *seeds;
    int64_t W;
    int64_t *best_e;
    uint64_t *best_words;
    int64_t *steps;
    uint8_t *dead;
    int64_t next; /* atomic work counter */
    int err;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    for (;;) {
        const int64_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= j->W) break;
        if (so_saw_walk(j->L, j->n, j->seeds[i], j->best_words + i * j->nw, j->nw, NULL, NULL, 0,
                        j->best_e + i, j->steps + i, j->dead + i) != 0)
            __atomic_store_n(&j->err, 1, __ATOMIC_RELAXED);
    }
    return NULL;
}

int so_num_procs(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

int so_saw_batch(int L, int n, const uint64_t *seeds, int64_t W, int64_t *best_e,
                 uint64_t *best_words, int64_t *steps, uint8_t *dead, int threads) {
    const int d = (L + 1) / 2;
    batch_job job = {L, n, (d + 63) / 64, seeds, W, best_e, best_words, steps, dead, 0, 0};
    if (threads <= 0) threads = so_num_procs();
    if (threads > W) threads = W > 0 ? (int)W : 1;
    if (threads <= 1) {
        batch_worker(&job);
        return job.err ? -1 : 0;
    }
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    if (!tid) return -1;
    int started = 0;
    for (; started < threads; started++)
        if (pthread_create(&tid[started], NULL, batch_worker, &job) != 0) break;
    if (started == 0) batch_worker(&job);
    for (int t = 0; t < started; t++) pthread_join(tid[t], NULL);
    free(tid);
    return job.err ? -1 : 0;
}

/* Seeds derived in-process (runner.py:234-240) for large oracle batches. */
void so_derive_walk_seeds(uint64_t master, uint64_t batch, uint64_t walker_begin, int64_t W,
                          uint64_t *out) {
    for (int64_t i = 0; i < W; i++) out[i] = so_derive_walk_seed(master, batch, walker_begin + (uint64_t)i);
}

/*
 * exhaustive_scan, _kernels.py:290-323: Gray-code enumeration of all 2^D
 * halves.  Returns best energy; *best_bits has bit h set iff half spin h is -1.
 */
int64_t so_exhaustive_scan(int L, int64_t *best_bits_out) {
    const int d = (L + 1) / 2;
    int64_t *s = (int64_t *)malloc(sizeof(int64_t) * L);
    int64_t *c = (int64_t *)calloc(L, sizeof(int64_t));
    for (int h = 0; h < d; h++) s[h] = 1;
    expand_in_place(s, d);
    int64_t e = init_sidelobes(s, c, L);
    int64_t best_e = e, best_bits = 0, bits = 0;
    const int64_t total = (int64_t)1 << d;
    for (int64_t g = 1; g < total; g++) {
        int64_t gg = g;
        int h = 0;
        while ((gg & 1) == 0) { gg >>= 1; h++; }
        e += neighbor_delta(s, c, L, h);
        apply_neighbor(s, c, L, h);
        bits ^= (int64_t)1 << h;
        if (e < best_e) { best_e = e; best_bits = bits; }
    }
    free(s); free(c);
    *best_bits_out = best_bits;
    return best_e;
}


/*
 * Slice of the same enumeration (test support for the device scan, which
 * splits the Gray index range): the state entering index g_begin is the half
 * gray(g_begin) (the reference's `bits` after step g_begin, _kernels.py:321),
 * then steps g_begin+1 .. g_begin+g_count-1 run exactly as
 * _kernels.py:313-322.  Returns the first minimum's energy and its index g.
 */
int64_t so_exhaustive_range(int L, uint64_t g_begin, uint64_t g_count, uint64_t *best_g_out) {
    const int d = (L + 1) / 2;
    int64_t *s = (int64_t *)malloc(sizeof(int64_t) * L);
    int64_t *c = (int64_t *)calloc(L, sizeof(int64_t));
    const uint64_t x = g_begin ^ (g_begin >> 1);
    for (int h = 0; h < d; h++) s[h] = ((x >> h) & 1) ? -1 : 1;
    expand_in_place(s, d);
    int64_t e = init_sidelobes(s, c, L);
    int64_t best_e = e;
    uint64_t best_g = g_begin;
    for (uint64_t g = g_begin + 1; g < g_begin + g_count; g++) {
        uint64_t gg = g;
        int h = 0;
        while ((gg & 1) == 0) { gg >>= 1; h++; }
        e += neighbor_delta(s, c, L, h);
        apply_neighbor(s, c, L, h);
        if (e < best_e) { best_e = e; best_g = g; }
    }
    free(s); free(c);
    *best_g_out = best_g;
    return best_e;
}
