"""The C ABI library loads, exports exactly what include/sokol.h declares,
and rejects bad arguments before touching the device (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

from paper_2210_15962_b200 import _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sokol.h")).read()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(sk_[a-z_0-9]+)\s*\(", text, re.M))


def test_header_matches_python_export_list():
    assert header_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for sym in _lib.EXPORTS:
        assert sym in exported, sym
        assert getattr(lib, sym) is not None


def test_abi_constants():
    lib = _lib.load()
    assert lib.sk_abi_version() == 1
    assert lib.sk_max_length() == _lib.SK_MAX_L
    assert _lib.SUMMARY_BYTES == 80


def test_variant_switch():
    lib = _lib.load()
    old = lib.sk_get_variant()
    try:
        for v in (_lib.VARIANT_SCALAR, _lib.VARIANT_FAST, _lib.VARIANT_AUTO):
            assert lib.sk_set_variant(v) == 0
            assert lib.sk_get_variant() == v
        assert lib.sk_set_variant(7) == _lib.SK_ERR_ARG
    finally:
        lib.sk_set_variant(old)


@pytest.mark.parametrize(
    "L,n,W,code",
    [(8, 10, 1, _lib.SK_ERR_ARG), (1, 10, 1, _lib.SK_ERR_ARG), (21, 0, 1, _lib.SK_ERR_ARG),
     (21, 10, -1, _lib.SK_ERR_ARG), (1025, 10, 1, _lib.SK_ERR_UNSUPPORTED)],
)
def test_argument_errors_without_device(L, n, W, code):
    lib = _lib.load()
    rc = lib.sk_saw_batch(L, n, None, 1, 0, 0, W, None, None, None, None, None, None)
    assert rc == code
    assert lib.sk_last_error()
    z = np.zeros(4, np.uint64)
    rc = lib.sk_saw_batch_host(L, n, z.ctypes.data, W, None, None, None, None)
    assert rc == code
    with pytest.raises(_lib.SokolError):
        _lib.check(rc)


def test_walk_host_rejects_missing_trace_buffers():
    lib = _lib.load()
    bw = np.zeros(1, np.uint64)
    e = np.zeros(1, np.int64)
    s = np.zeros(1, np.int64)
    d = np.zeros(1, np.uint8)
    rc = lib.sk_saw_walk_host(21, 88, 5, bw.ctypes.data, None, None, 1, e.ctypes.data, s.ctypes.data, d.ctypes.data)
    assert rc == _lib.SK_ERR_ARG


def test_summary_struct_layout():
    s = _lib.BatchSummary()
    assert ctypes.sizeof(s) == 80
    assert _lib.BatchSummary.min_key.offset == 0
    assert _lib.BatchSummary.steps_sum.offset == 8
    assert _lib.BatchSummary.best_words.offset == 16


def test_exhaustive_scan_validation():
    lib = _lib.load()
    be = np.zeros(1, np.int64)
    bb = np.zeros(1, np.int64)
    assert lib.sk_exhaustive_scan_host(4, be.ctypes.data, bb.ctypes.data) == _lib.SK_ERR_ARG
    assert lib.sk_exhaustive_scan_host(95, be.ctypes.data, bb.ctypes.data) == _lib.SK_ERR_UNSUPPORTED
    assert lib.sk_exhaustive_scan_host(27, None, bb.ctypes.data) == _lib.SK_ERR_ARG
    assert lib.sk_exhaustive_scan(27, 1 << 14, 1, None, None) == _lib.SK_ERR_ARG
