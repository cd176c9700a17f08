"""CPU check of the production evaluator's layout algebra (eval_tc.cuh).

tools/tc_emulate.py restates EvalTC on a byte array with the kernel's own
offsets: Q records gathered into the MMA's A fragments, the mirrored /
swapped G pairs of the B fragments, the key epilogue (S2 signs, C_{q-p},
s_{3h-2K}), the lag-pair C update through the shifted f16 spin copies, the
R update and the scattered flip stores.  Every delta vector must equal the
oracle's all_neighbor_deltas along a chain of moves (including centre and
end moves), at one- and two-tile lengths.  The device itself is checked by
the -m gpu suite; this pins the algebra without a GPU.
"""

import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "tools"))
import tc_emulate  # noqa: E402


@pytest.mark.parametrize("L", [3, 5, 7, 27, 63, 101, 129, 201, 253, 255, 257, 301, 449, 511, 513, 769, 1023])
def test_emulated_evaluator_matches_oracle(oracle, L):
    d = (L + 1) // 2
    rng = np.random.default_rng(L)
    for half in (np.ones(d, np.int64), rng.choice([-1, 1], size=d)):
        em = tc_emulate.Emu(L, half)
        s, c, _ = oracle.init_state(L, half.astype(np.int64))
        np.testing.assert_array_equal(em.evaluate(), oracle.all_neighbor_deltas(L, s, c))
        for h in [d - 1, 0, d - 1] + list(rng.integers(0, d, size=3)):
            em.apply(int(h))
            oracle.apply_neighbor(L, s, c, int(h))
            np.testing.assert_array_equal(em.evaluate(), oracle.all_neighbor_deltas(L, s, c), err_msg=f"L={L} h={h}")


def test_layout_properties_every_length():
    """Alignment, row bounds, zero reads past K and bank spacing for every odd L."""
    for L in range(3, 1024, 2):
        tc_emulate.check_geometry(L)


def test_emulator_geometry_is_the_kernels(tmp_path):
    """tc_emulate.Geom equals eval_tc.cuh's tc_geom (compiled for the host) at every length."""
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "tc_geom_dump")
    subprocess.run([nvcc, "-std=c++17", "-arch=sm_100a", "-I", os.path.join(ROOT, "paper_2210_15962_b200", "csrc"),
                    "-o", exe, os.path.join(ROOT, "tools", "tc_geom_dump.cu")], check=True, capture_output=True)
    rows = [list(map(int, line.split())) for line in subprocess.run([exe], check=True, capture_output=True,
                                                                     text=True).stdout.splitlines() if line.strip()]
    assert len(rows) == 511
    for L, *v in rows:
        g = tc_emulate.Geom(L)
        assert v == [g.NT, g.TOFF, g.MT, g.q_off, g.ge_off, g.go_off, g.t_off, g.s2_off, g.bytes], L
