"""BASELINE config 5: large instances (L=301, 449), walk-length / restart sweep.

    python tools/config5.py --lengths 301,449 --walk-factors 1,2,4,8,16,32 --seconds 30

Each point is one runner.solve with a fixed wall-time budget (max_runtime), the
walker count per batch sized so that a batch takes ~1 s.  Walk factor f sets
the walk length n = f*D, i.e. how often a walk restarts from a fresh random
pivot.  Prints NSE/s and the best energy / merit factor reached per point.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="301,449")
    ap.add_argument("--walk-factors", default="1,2,4,8,16,32")
    ap.add_argument("--seconds", type=float, default=30.0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    from paper_2210_15962_b200 import _lib
    from paper_2210_15962_b200.runner import RunConfig, solve

    lib = _lib.load()
    for L in [int(x) for x in a.lengths.split(",")]:
        D = (L + 1) // 2
        for wf in [int(x) for x in a.walk_factors.split(",")]:
            res = int(lib.sk_resident_walks(L, wf * D))
            # ~1 s per batch at ~1.3e11 NSE/s, whole resident waves
            W = max(res, int(1.3e11 / (wf * D * (D - 1)) // res * res))
            rec = solve(RunConfig(L=L, walkers=W, walk_factor=wf, master_seed=a.seed, max_runtime=a.seconds))
            print(json.dumps({"L": L, "walk_factor": wf, "walkers": W, "batches": rec.batches,
                              "seconds": rec.wall_time_s, "nse_per_s": rec.total_nses / rec.wall_time_s,
                              "best_E": rec.best_E, "best_F": rec.best_F, "best_hex": rec.best_hex}), flush=True)


if __name__ == "__main__":
    main()
