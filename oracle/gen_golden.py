"""Generate tests/golden/ fixtures by running the REAL reference package.

Runs only in the build container (it imports /root/reference/pkg/src, which
does not exist on the GPU box).  The fixtures are reference OUTPUTS; no
reference source is copied.  Re-run with:

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

The files it writes pin both the CPU oracle (oracle/sokol_oracle.c) and,
through it, the CUDA path.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("SKEWSAW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from skewsaw import _kernels  # noqa: E402
from skewsaw.neighborhood import compute_deltas, naive_oracle  # noqa: E402
from skewsaw.runner import (  # noqa: E402
    RunConfig,
    derive_repetition_seed,
    derive_walk_seed,
    solve,
    target_campaign,
)
from skewsaw.saw import (  # noqa: E402
    WalkConfig,
    exhaustive_optimum,
    half_to_words,
    key,
    run_walk_traced,
)
from skewsaw.codec import encode  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha16(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def main():
    os.makedirs(OUT, exist_ok=True)
    t0 = time.time()
    meta = {"generator": "oracle/gen_golden.py", "reference": REF}

    # --- seeds and keys (runner.py:53-62, _kernels.py:46-53) -----------------
    seeds = []
    for m, b, w in [(1, 0, 0), (1, 0, 1), (1, 7, 3), (0, 0, 0), (2**64 - 1, 12345, 987654), (99, 3, 2**40)]:
        seeds.append({"master": str(m), "batch": b, "walker": w, "seed": str(derive_walk_seed(m, b, w))})
    reps = []
    for m, r in [(1, 0), (4, 2), (71717, 99)]:
        reps.append({"master": str(m), "rep": r, "seed": str(derive_repetition_seed(m, r))})
    rng = np.random.default_rng(7)
    keys = []
    for d in [1, 2, 14, 51, 63, 64, 65, 101, 128, 151, 225, 300]:
        for _ in range(3):
            half = rng.choice([-1, 1], size=d)
            keys.append({"D": d, "hex": encode(half), "key": str(key(half))})
    keys.append({"D": 101, "hex": encode(np.ones(101, dtype=np.int64)), "key": str(key(np.ones(101, dtype=np.int64)))})
    with open(os.path.join(OUT, "seeds_keys.json"), "w") as f:
        json.dump({"meta": meta, "walk_seeds": seeds, "rep_seeds": reps, "keys": keys}, f, indent=1)

    # --- neighbourhood deltas (neighborhood.py:73-82) -------------------------
    rng = np.random.default_rng(2025)
    cases = []
    for _ in range(200):
        length = int(rng.choice(np.arange(3, 63, 2)))
        d = (length + 1) // 2
        half = rng.choice([-1, 1], size=d)
        st = naive_oracle(half)
        cases.append({"L": length, "hex": encode(half), "E": int(st.E), "deltas": [int(x) for x in compute_deltas(st)]})
    with open(os.path.join(OUT, "deltas.json"), "w") as f:
        json.dump({"meta": meta, "cases": cases}, f)

    # --- traced walks (saw.py:139-148, _kernels.py:189-275) -------------------
    traces = {}
    summary = []
    small = [(3, 5), (5, 0), (9, 1), (15, 0), (21, 1), (27, 3), (31, 99)]
    for length, seed in small:
        d = (length + 1) // 2
        res, tr = run_walk_traced(WalkConfig(L=length, n=8 * d, seed=seed))
        traces[f"L{length}_s{seed}_pivots"] = tr.pivots.astype(np.int8)
        traces[f"L{length}_s{seed}_deltas"] = tr.deltas.astype(np.int32)
        summary.append({"L": length, "seed": str(seed), "n": 8 * d, "best_E": res.best_E, "steps": res.steps_taken,
                        "dead": bool(res.dead_end), "best_hex": encode(res.best_half)})
    for length, ws in [(101, range(3)), (201, range(3)), (301, range(1)), (449, range(1))]:
        d = (length + 1) // 2
        for w in ws:
            seed = derive_walk_seed(1, 0, w)
            res, tr = run_walk_traced(WalkConfig(L=length, n=8 * d, seed=seed))
            piv8 = tr.pivots.astype(np.int8)
            row = {"L": length, "seed": str(seed), "n": 8 * d, "best_E": res.best_E, "steps": res.steps_taken,
                   "dead": bool(res.dead_end), "best_hex": encode(res.best_half),
                   "sha_pivots_i8": sha16(piv8), "sha_deltas_i64": sha16(tr.deltas.astype(np.int64)),
                   "first_deltas": [int(x) for x in tr.deltas[0, :8]],
                   "last_deltas": [int(x) for x in tr.deltas[-1, :8]]}
            if length == 101:
                traces[f"L{length}_s{seed}_pivots"] = piv8
                traces[f"L{length}_s{seed}_deltas"] = tr.deltas.astype(np.int32)
            summary.append(row)
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **traces)
    with open(os.path.join(OUT, "traces.json"), "w") as f:
        json.dump({"meta": meta, "walks": summary}, f, indent=1)

    # --- batch outputs (_kernels.py:278-287 with runner.py:234-249 seeds) -----
    batches = {}
    bsum = []
    for length, W, m, b in [(3, 16, 1, 0), (5, 16, 1, 0), (27, 64, 1, 0), (101, 4096, 1, 0), (201, 512, 1, 0),
                            (201, 64, 3, 5), (301, 64, 1, 0), (449, 32, 1, 0), (63, 256, 2, 1), (65, 256, 2, 1),
                            (127, 128, 4, 0), (129, 128, 4, 0)]:
        d = (length + 1) // 2
        nw = (d + 63) // 64
        n = 8 * d
        sd = np.array([derive_walk_seed(m, b, w) for w in range(W)], dtype=np.uint64)
        be = np.empty(W, np.int64)
        bw = np.empty((W, nw), np.uint64)
        st = np.empty(W, np.int64)
        dd = np.empty(W, np.uint8)
        _kernels.saw_batch(length, n, sd, be, bw, st, dd)
        tag = f"L{length}_m{m}_b{b}_W{W}"
        batches[tag + "_best_e"] = be
        batches[tag + "_best_words"] = bw
        batches[tag + "_steps"] = st
        batches[tag + "_dead"] = dd
        bsum.append({"tag": tag, "L": length, "W": W, "master": m, "batch": b, "n": n})
    np.savez_compressed(os.path.join(OUT, "batches.npz"), **batches)
    with open(os.path.join(OUT, "batches.json"), "w") as f:
        json.dump({"meta": meta, "batches": bsum}, f, indent=1)

    # --- RunRecords (runner.py:259-291) ---------------------------------------
    configs = [
        dict(L=21, walkers=4, master_seed=7, target_E=26, max_nses=10**6),
        dict(L=21, walkers=3, master_seed=5, max_nses=3 * 88 * 10),
        dict(L=21, walkers=3, master_seed=4, target_E=26, max_nses=10**6),
        dict(L=35, walkers=2, master_seed=11, max_nses=200_000),
        dict(L=27, walkers=8, master_seed=0, target_E=37, max_nses=10**6),
        dict(L=27, walkers=8, master_seed=1, target_E=37, max_nses=10**6),
        dict(L=27, walkers=4, master_seed=9, max_nses=4 * 112 * 13 * 3),
        dict(L=71, walkers=2, master_seed=99, max_nses=2_000_000),
        dict(L=101, walkers=64, master_seed=1, max_nses=3_916_800),
        dict(L=201, walkers=16, master_seed=2, max_nses=2_585_600),
        dict(L=15, walkers=2, master_seed=4, target_E=15, max_nses=100_000, walk_factor=3),
    ]
    records = []
    for cfg in configs:
        rec = solve(RunConfig(**cfg)).to_json_dict()
        rec.pop("wall_time_s")
        records.append({"config": cfg, "record": rec})
    camp = target_campaign(RunConfig(L=15, walkers=2, master_seed=4, target_E=15, max_nses=100_000), 5)
    with open(os.path.join(OUT, "records.json"), "w") as f:
        json.dump({"meta": meta, "records": records,
                   "campaign_L15": {"nses": camp.nses, "censored": camp.censored}}, f, indent=1)

    # --- exhaustive optima (saw.py:151-168) -----------------------------------
    optima = []
    for length in range(3, 42, 2):
        rec, half = exhaustive_optimum(length)
        optima.append({"L": length, "E": rec.E, "hex": encode(half)})
    with open(os.path.join(OUT, "optima.json"), "w") as f:
        json.dump({"meta": meta, "optima": optima}, f, indent=1)

    print(f"golden fixtures written to {os.path.abspath(OUT)} in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
