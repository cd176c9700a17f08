"""ctypes wrapper around the CPU oracle (oracle/sokol_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs as the checker.  The
product package ``paper_2210_15962_b200`` never imports this module.

Each wrapper mirrors one entry of the reference (file:line cited on the C side):
    saw_batch      -> skewsaw._kernels.saw_batch      (_kernels.py:278-287)
    saw_walk       -> skewsaw._kernels.saw_walk       (_kernels.py:189-275)
    key_of_words   -> skewsaw._kernels.key_of_words   (_kernels.py:46-53)
    derive_walk_seed -> skewsaw.runner.derive_walk_seed (runner.py:53-57)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsokol_oracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> str:
    """Compile the oracle with its Makefile (gcc); returns the .so path."""
    src = os.path.join(_HERE, "sokol_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.so_mix64.argtypes = [ctypes.c_uint64]
        L.so_mix64.restype = ctypes.c_uint64
        L.so_key_of_words.argtypes = [_u64p, ctypes.c_int]
        L.so_key_of_words.restype = ctypes.c_uint64
        L.so_derive_walk_seed.argtypes = [ctypes.c_uint64] * 3
        L.so_derive_walk_seed.restype = ctypes.c_uint64
        L.so_derive_repetition_seed.argtypes = [ctypes.c_uint64] * 2
        L.so_derive_repetition_seed.restype = ctypes.c_uint64
        L.so_derive_walk_seeds.argtypes = [ctypes.c_uint64] * 3 + [ctypes.c_int64, _u64p]
        L.so_derive_walk_seeds.restype = None
        L.so_all_neighbor_deltas.argtypes = [ctypes.c_int, _i64p, _i64p, _i64p]
        L.so_all_neighbor_deltas.restype = None
        L.so_apply_neighbor.argtypes = [ctypes.c_int, _i64p, _i64p, ctypes.c_int]
        L.so_apply_neighbor.restype = None
        L.so_init_sidelobes.argtypes = [ctypes.c_int, _i64p, _i64p]
        L.so_init_sidelobes.restype = ctypes.c_int64
        L.so_saw_walk.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _u64p, ctypes.c_int,
            _u64p, _i64p, ctypes.c_int, _i64p, _i64p, _u8p,
        ]
        L.so_saw_walk.restype = ctypes.c_int
        L.so_saw_batch.argtypes = [
            ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int64, _i64p, _u64p, _i64p, _u8p,
            ctypes.c_int,
        ]
        L.so_saw_batch.restype = ctypes.c_int
        L.so_exhaustive_scan.argtypes = [ctypes.c_int, _i64p]
        L.so_exhaustive_scan.restype = ctypes.c_int64
        L.so_exhaustive_range.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _u64p]
        L.so_exhaustive_range.restype = ctypes.c_int64
        L.so_num_procs.argtypes = []
        L.so_num_procs.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


def num_procs() -> int:
    return int(lib().so_num_procs())


def mix64(z: int) -> int:
    return int(lib().so_mix64(z & (2**64 - 1)))


def key_of_words(words) -> int:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(lib().so_key_of_words(_p(w, _u64p), w.size))


def derive_walk_seed(master: int, batch: int, walker: int) -> int:
    return int(lib().so_derive_walk_seed(master, batch, walker))


def derive_repetition_seed(master: int, rep: int) -> int:
    return int(lib().so_derive_repetition_seed(master, rep))


def derive_walk_seeds(master: int, batch: int, W: int, walker_begin: int = 0) -> np.ndarray:
    out = np.empty(W, dtype=np.uint64)
    lib().so_derive_walk_seeds(master, batch, walker_begin, W, _p(out, _u64p))
    return out


def init_state(length: int, half):
    """Full sequence and natural-order correlations of a half (int64)."""
    d = (length + 1) // 2
    h = np.asarray(half, dtype=np.int64)
    assert h.size == d
    s = np.empty(length, dtype=np.int64)
    s[:d] = h
    sign = -1
    for i in range(1, d):
        s[d - 1 + i] = sign * s[d - 1 - i]
        sign = -sign
    c = np.zeros(length, dtype=np.int64)
    e = int(lib().so_init_sidelobes(length, _p(s, _i64p), _p(c, _i64p)))
    return s, c, e


def all_neighbor_deltas(length: int, s, c) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.int64)
    c = np.ascontiguousarray(c, dtype=np.int64)
    out = np.empty((length + 1) // 2, dtype=np.int64)
    lib().so_all_neighbor_deltas(length, _p(s, _i64p), _p(c, _i64p), _p(out, _i64p))
    return out


def apply_neighbor(length: int, s, c, h: int):
    """In place on int64 arrays (_kernels.py:126-158)."""
    lib().so_apply_neighbor(length, _p(s, _i64p), _p(c, _i64p), int(h))


def saw_walk(length: int, n: int, seed: int, record: bool = False):
    """Returns (best_e, steps, dead, best_words, trace_words|None, trace_deltas|None)."""
    d = (length + 1) // 2
    nw = (d + 63) // 64
    best_words = np.zeros(nw, dtype=np.uint64)
    if record:
        tw = np.zeros((n + 1, nw), dtype=np.uint64)
        td = np.zeros((n, d), dtype=np.int64)
    else:
        tw = np.zeros((1, 1), dtype=np.uint64)
        td = np.zeros((1, 1), dtype=np.int64)
    be = np.zeros(1, dtype=np.int64)
    st = np.zeros(1, dtype=np.int64)
    dd = np.zeros(1, dtype=np.uint8)
    rc = lib().so_saw_walk(
        length, n, seed, _p(best_words, _u64p), nw, _p(tw, _u64p), _p(td, _i64p),
        1 if record else 0, _p(be, _i64p), _p(st, _i64p), _p(dd, _u8p),
    )
    if rc != 0:
        raise MemoryError("oracle saw_walk allocation failed")
    if record:
        return int(be[0]), int(st[0]), bool(dd[0]), best_words, tw, td
    return int(be[0]), int(st[0]), bool(dd[0]), best_words, None, None


def saw_batch(length, n, seeds, best_e_out, best_words_out, steps_out, dead_out, threads: int = 0):
    """Same signature as skewsaw._kernels.saw_batch (plus a thread count)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    for a, t in ((best_e_out, np.int64), (best_words_out, np.uint64), (steps_out, np.int64), (dead_out, np.uint8)):
        assert a.dtype == t and a.flags.c_contiguous
    rc = lib().so_saw_batch(
        length, n, _p(seeds, _u64p), seeds.size, _p(best_e_out, _i64p), _p(best_words_out, _u64p),
        _p(steps_out, _i64p), _p(dead_out, _u8p), threads,
    )
    if rc != 0:
        raise MemoryError("oracle saw_batch allocation failed")


def batch_outputs(length: int, n: int, seeds, threads: int = 0):
    """Convenience: allocate outputs, run saw_batch, return them."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    d = (length + 1) // 2
    nw = (d + 63) // 64
    W = seeds.size
    be = np.empty(W, dtype=np.int64)
    bw = np.empty((W, nw), dtype=np.uint64)
    st = np.empty(W, dtype=np.int64)
    dd = np.empty(W, dtype=np.uint8)
    saw_batch(length, n, seeds, be, bw, st, dd, threads)
    return be, bw, st, dd


def exhaustive_scan(length: int):
    bits = np.zeros(1, dtype=np.int64)
    e = int(lib().so_exhaustive_scan(length, _p(bits, _i64p)))
    return e, int(bits[0])


def exhaustive_range(length: int, g_begin: int, g_count: int):
    """(first-min energy, its Gray index g) over g in [g_begin, g_begin + g_count)."""
    g = np.zeros(1, dtype=np.uint64)
    e = int(lib().so_exhaustive_range(length, g_begin, g_count, _p(g, _u64p)))
    return e, int(g[0])


def exhaustive_scan_threaded(length: int, threads: int = 0, slices: int = 0):
    """exhaustive_scan over all host threads: the Gray index range is cut
    into slices scanned concurrently (ctypes releases the GIL); the first
    minimum in Gray order is the minimum of the per-slice (E, g).  Returns
    (E, bits) exactly as exhaustive_scan."""
    from concurrent.futures import ThreadPoolExecutor

    threads = threads or num_procs()
    total = 1 << ((length + 1) // 2)
    k = slices or 4 * threads
    cuts = [total * i // k for i in range(k + 1)]
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda ab: exhaustive_range(length, ab[0], ab[1] - ab[0]), zip(cuts, cuts[1:])))
    e, g = min(parts)
    return e, g ^ (g >> 1)


def solve_record(L, walkers, walk_factor=8, master_seed=1, max_nses=None, target_E=None, threads: int = 0):
    """The reference's batch loop (runner.py:213-291) over the oracle's
    saw_batch; returns the RunRecord JSON dict minus wall_time_s.  Runtime
    stops are not supported (records must be deterministic)."""
    d = (L + 1) // 2
    n = walk_factor * d
    best_e = best_words = None
    total = batches = 0
    stop = None
    while stop is None:
        seeds = derive_walk_seeds(master_seed, batches, walkers)
        be, bw, st, _ = batch_outputs(L, n, seeds, threads)
        batches += 1
        total += int(st.sum()) * (d - 1)
        for w in range(walkers):
            if best_e is None or int(be[w]) < best_e:
                best_e = int(be[w])
                best_words = bw[w].copy()
        if target_E is not None and best_e <= target_E:
            stop = "target_reached"
        elif max_nses is not None and total >= max_nses:
            stop = "nses_exhausted"
        elif max_nses is None and target_E is None:
            raise ValueError("need a deterministic stopping condition")
    value = sum(int(w) << (64 * i) for i, w in enumerate(best_words))
    width = -(-d // 4)
    return {
        "L": L, "walkers": walkers, "walk_factor": walk_factor, "master_seed": master_seed,
        "max_nses": max_nses, "max_runtime_s": None, "target_E": target_E,
        "best_E": best_e, "best_F": L * L / (2.0 * best_e) if best_e > 0 else None,
        "best_hex": "0x" + format(value, f"0{width}X"), "total_nses": total, "batches": batches,
        "stop_reason": stop,
    }
