"""Generate the round-2 golden fixtures by running the REAL reference package.

Like gen_golden.py this runs only in the build container (it imports
/root/reference/pkg/src).  It writes reference OUTPUTS only:

  tests/golden/config2_traces.json   BASELINE config 2: run_walk_traced for
        derive_walk_seed(1, 0, w), w < 64, at L=101 (saw.py:139-148;
        _kernels.py:231-243, 267-270): sha256 of pivots (int8) and raw deltas
        (int64), best_E / steps / dead / best_hex.
  tests/golden/config_records.json   BASELINE config 2 RunRecord
        RunConfig(L=101, walkers=4096, master_seed=1, max_nses=167,116,800)
        and config 1: RunConfig(L=27, walkers=8, master_seed=s, target_E=37,
        max_nses=10**6) for every s < 100 (runner.py:213-291).
  tests/golden/optima_43_55.json     exhaustive_optimum(L) for L = 43..55
        (saw.py:151-168), extending optima.json (3..41).

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_r2.py [--skip-optima]
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

from skewsaw.codec import encode  # noqa: E402
from skewsaw.runner import RunConfig, derive_walk_seed, solve  # noqa: E402
from skewsaw.saw import WalkConfig, exhaustive_optimum, run_walk_traced  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def main():
    meta = {"generator": "oracle/gen_golden_r2.py", "reference": REF}
    t0 = time.time()

    walks = []
    for w in range(64):
        seed = derive_walk_seed(1, 0, w)
        res, tr = run_walk_traced(WalkConfig(L=101, n=408, seed=seed))
        walks.append({"w": w, "seed": str(seed), "best_E": res.best_E, "steps": res.steps_taken,
                      "dead": bool(res.dead_end), "best_hex": encode(res.best_half),
                      "sha_pivots_i8": sha(tr.pivots.astype(np.int8)),
                      "sha_deltas_i64": sha(tr.deltas.astype(np.int64)),
                      "rows_pivots": int(tr.pivots.shape[0]), "rows_deltas": int(tr.deltas.shape[0])})
    with open(os.path.join(OUT, "config2_traces.json"), "w") as f:
        json.dump({"meta": meta, "L": 101, "n": 408, "master": 1, "batch": 0, "walks": walks}, f, indent=0)
    print(f"traces done {time.time() - t0:.1f}s", flush=True)

    records = []
    cfg = dict(L=101, walkers=4096, master_seed=1, max_nses=4096 * 408 * 50 * 2)
    rec = solve(RunConfig(**cfg)).to_json_dict()
    rec.pop("wall_time_s")
    records.append({"config": cfg, "record": rec})
    print(f"config 2 record done {time.time() - t0:.1f}s", flush=True)
    for s in range(100):
        cfg = dict(L=27, walkers=8, master_seed=s, target_E=37, max_nses=10**6)
        rec = solve(RunConfig(**cfg)).to_json_dict()
        rec.pop("wall_time_s")
        records.append({"config": cfg, "record": rec})
    with open(os.path.join(OUT, "config_records.json"), "w") as f:
        json.dump({"meta": meta, "records": records}, f, indent=0)
    print(f"config 1 records done {time.time() - t0:.1f}s", flush=True)

    if "--skip-optima" not in sys.argv:
        optima = []
        for length in range(43, 56, 2):
            t1 = time.time()
            rec, half = exhaustive_optimum(length)
            optima.append({"L": length, "E": rec.E, "hex": encode(half), "ref_scan_s": round(time.time() - t1, 1)})
            print(optima[-1], flush=True)
            with open(os.path.join(OUT, "optima_43_55.json"), "w") as f:
                json.dump({"meta": meta, "optima": optima}, f, indent=1)
    print(f"done {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
