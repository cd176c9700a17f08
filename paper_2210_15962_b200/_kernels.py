"""Drop-in replacement for ``skewsaw._kernels``' walk entry points.

Same names, argument order, dtypes and in-place output semantics as the
reference's numba kernels, executed by libsokol.so on the current CUDA device:

    saw_batch(length, n, seeds, best_e_out, best_words_out, steps_out, dead_out)
        -> skewsaw._kernels.saw_batch   (_kernels.py:278-287)
    saw_walk(length, n, seed, best_words, trace_words, trace_deltas, record)
        -> skewsaw._kernels.saw_walk    (_kernels.py:189-275)
    key_of_words(words)
        -> skewsaw._kernels.key_of_words (_kernels.py:46-53)
    exhaustive_scan(length) -> (best_e, best_bits)
        -> skewsaw._kernels.exhaustive_scan (_kernels.py:290-323)
    eval_states(length, halves, moves) -> deltas [S, M+1, D]
        the walk's evaluator on given states (all_neighbor_deltas +
        apply_neighbor, _kernels.py:85-165), a test probe (sk_eval_states)

Unlike numba, the C ABI validates its arguments and raises ``SokolError``
(a RuntimeError) on bad input or a CUDA failure.
"""

from __future__ import annotations

import numpy as np

from . import _lib

MASK64 = (1 << 64) - 1
KEY_SEED = 0xA0761D6478BD642F
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """splitmix64 finaliser on Python ints (_kernels.py:32-37)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def key_of_words(words) -> np.uint64:
    """Chained key of packed words; host utility (not on the batch path)."""
    h = KEY_SEED
    for w in np.asarray(words, dtype=np.uint64).ravel():
        h = mix64(h ^ int(w))
    return np.uint64(h)


def _req(arr, dtype, name, shape=None):
    if not isinstance(arr, np.ndarray) or arr.dtype != dtype or not arr.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous numpy array of {np.dtype(dtype).name}")
    if shape is not None and arr.shape != shape:
        raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
    return arr.ctypes.data


def saw_batch(length, n, seeds, best_e_out, best_words_out, steps_out, dead_out):
    """Run one independent walk per seed on the GPU; outputs written in place."""
    length = int(length)
    n = _lib.check_steps(n)
    d = (length + 1) // 2
    nw = (d + 63) // 64
    W = int(np.asarray(seeds).shape[0])
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    p_seeds = seeds.ctypes.data
    p_e = _req(best_e_out, np.int64, "best_e_out", (W,))
    p_w = _req(best_words_out, np.uint64, "best_words_out", (W, nw))
    p_s = _req(steps_out, np.int64, "steps_out", (W,))
    p_d = _req(dead_out, np.uint8, "dead_out", (W,))
    _lib.check(_lib.load().sk_saw_batch_host(length, n, p_seeds, W, p_e, p_w, p_s, p_d))


def saw_walk(length, n, seed, best_words, trace_words, trace_deltas, record):
    """One walk; returns (best_e, steps, dead) like the reference."""
    length = int(length)
    n = _lib.check_steps(n)
    d = (length + 1) // 2
    nw = (d + 63) // 64
    p_bw = _req(best_words, np.uint64, "best_words", (nw,))
    if record:
        p_tw = _req(trace_words, np.uint64, "trace_words", (n + 1, nw))
        p_td = _req(trace_deltas, np.int64, "trace_deltas", (n, d))
    else:
        p_tw = p_td = None
    be = np.zeros(1, np.int64)
    st = np.zeros(1, np.int64)
    dd = np.zeros(1, np.uint8)
    _lib.check(_lib.load().sk_saw_walk_host(
        length, n, int(seed) & MASK64, p_bw, p_tw, p_td, 1 if record else 0,
        be.ctypes.data, st.ctypes.data, dd.ctypes.data,
    ))
    return np.int64(be[0]), np.int64(st[0]), bool(dd[0])


def exhaustive_scan(length):
    """Minimum energy over all 2^D half sequences and the reference's argmin
    (first minimum in Gray order); bit h of best_bits set iff half spin h is
    -1.  Runs the device Gray-code scan (D <= SK_MAX_EXHAUSTIVE_D)."""
    be = np.zeros(1, np.int64)
    bb = np.zeros(1, np.int64)
    _lib.check(_lib.load().sk_exhaustive_scan_host(int(length), be.ctypes.data, bb.ctypes.data))
    return np.int64(be[0]), np.int64(bb[0])


def _device_copy(arr):
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def all_neighbor_deltas(s, c, out):
    """out[h] = neighbor_delta(s, c, h) for every half index h
    (_kernels.py:162-165); `s`, `c` int64[L] (c[k] = C_k), `out` int64[D].
    Also accepts stacked states: s, c int64[S, L], out int64[S, D]."""
    import torch

    s = np.asarray(s)
    L = int(s.shape[-1])
    S = int(np.prod(s.shape[:-1], dtype=np.int64)) if s.ndim > 1 else 1
    _req(out, np.int64, "out", s.shape[:-1] + ((L + 1) // 2,))
    ds, dc = _device_copy(s.astype(np.int64, copy=False)), _device_copy(np.asarray(c, dtype=np.int64))
    dout = torch.empty(out.shape, dtype=torch.int64, device=ds.device)
    _lib.check(_lib.load().sk_all_neighbor_deltas(L, S, ds.data_ptr(), dc.data_ptr(), dout.data_ptr(),
                                                  torch.cuda.current_stream().cuda_stream))
    out[...] = dout.cpu().numpy()


def apply_neighbor(s, c, h):
    """Move to neighbour h in place (_kernels.py:126-158): even-lag sidelobes
    of `c` updated, spins p = h and q = L-1-h of `s` negated.  Stacked
    states (s, c int64[S, L]) take h as an int64[S] array."""
    import torch

    _req(s, np.int64, "s")
    _req(c, np.int64, "c", s.shape)
    L = int(s.shape[-1])
    S = int(np.prod(s.shape[:-1], dtype=np.int64)) if s.ndim > 1 else 1
    hv = np.asarray(h, dtype=np.int64).reshape(S)
    if np.any((hv < 0) | (hv >= (L + 1) // 2)):
        raise ValueError(f"flip index out of range for D={(L + 1) // 2}")
    ds, dc, dh = _device_copy(s), _device_copy(c), _device_copy(hv)
    _lib.check(_lib.load().sk_apply_neighbor(L, S, ds.data_ptr(), dc.data_ptr(), dh.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    s[...] = ds.cpu().numpy()
    c[...] = dc.cpu().numpy()


def eval_states(length, halves, moves=None):
    """Delta vectors from the walk kernels' evaluator on given states.

    halves: int8-convertible [S, D] of +-1; moves: int [S, M] half indices
    (or None).  Returns int64 [S, M+1, D]: row 0 is the neighbourhood of the
    start state, row i+1 the neighbourhood after applying moves[:, :i+1]
    (apply_neighbor semantics, no visited check)."""
    import torch

    length = int(length)
    d = (length + 1) // 2
    h = np.ascontiguousarray(halves, dtype=np.int8)
    if h.ndim != 2 or h.shape[1] != d or not np.all(np.abs(h) == 1):
        raise ValueError(f"halves must be [S, {d}] of +-1")
    S = h.shape[0]
    mv = np.zeros((S, 0), np.int32) if moves is None else np.ascontiguousarray(moves, dtype=np.int32)
    if mv.ndim != 2 or mv.shape[0] != S or (mv.size and (mv.min() < 0 or mv.max() >= d)):
        raise ValueError(f"moves must be [S, M] half indices in [0, {d})")
    M = mv.shape[1]
    dev = torch.device("cuda", torch.cuda.current_device())
    dh = torch.from_numpy(h).to(dev)
    dm = torch.from_numpy(mv).to(dev) if M else None
    out = torch.empty((S, M + 1, d), dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.check(_lib.load().sk_eval_states(length, S, dh.data_ptr(), M, dm.data_ptr() if M else None,
                                          out.data_ptr(), st.cuda_stream))
    st.synchronize()
    return out.cpu().numpy()
