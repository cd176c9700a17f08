"""ctypes binding of libsokol.so (the C ABI declared in include/sokol.h).

The library is built in-tree by ``paper_2210_15962_b200.build`` (nvcc,
sm_100a) and loaded from the package directory.  There is no fallback: if the
library is missing or fails to load, every entry point raises, so a GPU run
can never silently take a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SOKOL_LIB: load an alternative in-tree build (kernel experiments, tools/); default libsokol.so
LIB_PATH = os.environ.get("SOKOL_LIB") or os.path.join(_HERE, "libsokol.so")

SK_OK = 0
SK_ERR_ARG = -1
SK_ERR_UNSUPPORTED = -2
SK_ERR_CUDA = -3
SK_ERR_NOMEM = -4
SK_MAX_L = 1023
SK_MAX_WORDS = 8
SK_MAX_EXHAUSTIVE_D = 47

VARIANT_AUTO = 0
VARIANT_SCALAR = 1
VARIANT_FAST = 2

VISITED_AUTO = 0
VISITED_SMEM = 1
VISITED_FINGERPRINT = 2
VISITED_GLOBAL = 3

# Every symbol include/sokol.h declares; tests/test_abi.py checks the export
# table against this list and against the header itself.
EXPORTS = (
    "sk_abi_version",
    "sk_last_error",
    "sk_max_length",
    "sk_set_variant",
    "sk_get_variant",
    "sk_set_visited_layout",
    "sk_saw_batch",
    "sk_saw_multi",
    "sk_saw_trace",
    "sk_saw_batch_host",
    "sk_saw_walk_host",
    "sk_resident_walks",
    "sk_exhaustive_scan",
    "sk_exhaustive_scan_host",
    "sk_all_neighbor_deltas",
    "sk_apply_neighbor",
    "sk_eval_states",
    "sk_shutdown",
)


class BatchSummary(ctypes.Structure):
    """Mirror of sk_batch_summary (include/sokol.h)."""

    _fields_ = [
        ("min_key", ctypes.c_uint64),
        ("steps_sum", ctypes.c_int64),
        ("best_words", ctypes.c_uint64 * SK_MAX_WORDS),
    ]


SUMMARY_BYTES = ctypes.sizeof(BatchSummary)  # 80


class SokolError(RuntimeError):
    """Raised for any non-zero return of the C ABI."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libsokol error {code}: {message}")
        self.code = code


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i = ctypes.c_int
_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64


def _declare(lib):
    lib.sk_abi_version.restype = _i
    lib.sk_last_error.restype = ctypes.c_char_p
    lib.sk_max_length.restype = _i
    lib.sk_set_variant.argtypes = [_i]
    lib.sk_set_variant.restype = _i
    lib.sk_get_variant.restype = _i
    lib.sk_set_visited_layout.argtypes = [_i]
    lib.sk_set_visited_layout.restype = _i
    lib.sk_saw_batch.argtypes = [_i, _i, _vp, _u64, _u64, _u64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
    lib.sk_saw_batch.restype = _i
    lib.sk_saw_multi.argtypes = [_i, _i, _vp, _vp, _i, _u64, _i64, _vp, _vp]
    lib.sk_saw_multi.restype = _i
    lib.sk_saw_trace.argtypes = [_i, _i, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    lib.sk_saw_trace.restype = _i
    lib.sk_saw_batch_host.argtypes = [_i, _i, _vp, _i64, _vp, _vp, _vp, _vp]
    lib.sk_saw_batch_host.restype = _i
    lib.sk_saw_walk_host.argtypes = [_i, _i, _u64, _vp, _vp, _vp, _i, _vp, _vp, _vp]
    lib.sk_saw_walk_host.restype = _i
    lib.sk_resident_walks.argtypes = [_i, _i]
    lib.sk_resident_walks.restype = _i64
    lib.sk_exhaustive_scan.argtypes = [_i, _u64, _u64, _vp, _vp]
    lib.sk_exhaustive_scan.restype = _i
    lib.sk_exhaustive_scan_host.argtypes = [_i, _vp, _vp]
    lib.sk_exhaustive_scan_host.restype = _i
    lib.sk_all_neighbor_deltas.argtypes = [_i, _i64, _vp, _vp, _vp, _vp]
    lib.sk_all_neighbor_deltas.restype = _i
    lib.sk_apply_neighbor.argtypes = [_i, _i64, _vp, _vp, _vp, _vp]
    lib.sk_apply_neighbor.restype = _i
    lib.sk_eval_states.argtypes = [_i, _i64, _vp, _i, _vp, _vp, _vp]
    lib.sk_eval_states.restype = _i
    lib.sk_shutdown.restype = _i


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raise if unavailable."""
    global _lib
    with _lock:
        if _lib is None:
            p = path or LIB_PATH
            if not os.path.exists(p):
                raise SokolError(
                    SK_ERR_UNSUPPORTED,
                    f"{p} not built; run `python -m paper_2210_15962_b200.build` (nvcc, sm_100a)",
                )
            lib = ctypes.CDLL(p)
            _declare(lib)
            _lib = lib
        return _lib


def check(rc: int):
    if rc != SK_OK:
        msg = load().sk_last_error()
        raise SokolError(rc, msg.decode() if msg else "")


INT32_MAX = (1 << 31) - 1


def check_steps(n: int) -> int:
    """The C ABI takes the walk step count as a C int; ctypes would truncate
    a larger value silently, so it is rejected here (the reference accepts any
    n >= 1, runner.py:81-97, but a walk of 2^31 steps needs a 2^35-byte
    visited set per walk)."""
    n = int(n)
    if n > INT32_MAX:
        raise SokolError(SK_ERR_UNSUPPORTED, f"walk step count n={n} exceeds the C ABI's int range")
    return n


def set_variant(variant: int):
    check(load().sk_set_variant(variant))


def get_variant() -> int:
    return int(load().sk_get_variant())


def set_visited_layout(mode: int):
    check(load().sk_set_visited_layout(mode))
