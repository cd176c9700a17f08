"""bench.py's roofline block (CPU): the binding on-chip resource is named
from the committed ncu capture's per-step counts (profiles/ncu_walk_kernel.json)
times the live step rate, and the tensor-pipe and INT32-equivalence figures
ride beside it."""

import json
import os

from conftest import ROOT

import bench


def test_mma_per_step_matches_the_evaluator_geometry():
    # eval_tc.cuh: sum over tiles of the k-block range [mlo(tau), mhi(tau)]
    assert bench.mma_per_step(201) == 10
    assert bench.mma_per_step(255) == 12
    assert bench.mma_per_step(301) == 25
    assert bench.mma_per_step(449) == 37
    assert bench.mma_per_step(3) == 1


def test_roofline_names_the_binding_resource():
    with open(os.path.join(ROOT, "profiles", "ncu_walk_kernel.json")) as f:
        cap = json.load(f)
    assert cap["L"] == 201 and cap["inst_executed"] > 0 and cap["smem_wavefronts"] > 0
    r = bench.roofline(201, 808, 1 << 20, 2.0e11, 1.0, {"sm_mhz": 1965.0})
    assert r["bound"] in ("smem", "issue")
    other = "issue" if r["bound"] == "smem" else "smem"
    assert r["frac"] == r[r["bound"]]["frac"] >= r[other]["frac"]
    assert 0 < r["frac"] < 1.2
    steps = 2.0e11 / 100
    assert abs(r["issue"]["achieved"] - cap["inst_executed"] / cap["walk_steps"] * steps / 1e9) < 1e-6
    assert r["pipes"]["tensor"]["mma_per_step"] == 10
    assert "equivalence" in r["int32_equivalent"]["note"]
