"""Small walk workloads for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py

Runs, at L = 27, 101, 201, 449 and with each visited-set layout, a small
batch through sk_saw_batch (device seeds + summary), the traced kernel
(sk_saw_trace via run_walk_traced), the evaluator probe (sk_eval_states) and
one multi-search launch (sk_saw_multi), and checks every result against the
CPU oracle so that a sanitizer run is also a parity run.  Exit code 0 iff all
results match; the sanitizer's own verdict is in its log.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle  # noqa: E402
import torch  # noqa: E402

from paper_2210_15962_b200 import _kernels, _lib, engine  # noqa: E402
from paper_2210_15962_b200.saw import WalkConfig, run_walk_traced  # noqa: E402


def main():
    W = int(os.environ.get("SANITIZE_W", "48"))
    lib = _lib.load()
    bad = 0
    lengths = [int(x) for x in os.environ.get("SANITIZE_LENGTHS", "27,101,201,449").split(",")]
    for L in lengths:
        d = (L + 1) // 2
        n = int(os.environ.get("SANITIZE_WF", "8")) * d  # walk factor (racecheck at L=449 needs short walks)
        layouts = [int(x) for x in os.environ.get("SANITIZE_LAYOUTS", "1,2,3").split(",")]
        for layout in layouts:
            for variant in (_lib.VARIANT_FAST, _lib.VARIANT_SCALAR):
                _lib.set_variant(variant)
                _lib.set_visited_layout(layout)
                seeds = oracle.derive_walk_seeds(7, L, W)
                want = oracle.batch_outputs(L, n, seeds)
                nw = (d + 63) // 64
                got = (np.empty(W, np.int64), np.empty((W, nw), np.uint64), np.empty(W, np.int64),
                       np.empty(W, np.uint8))
                _kernels.saw_batch(L, n, seeds, *got)
                ok = all(np.array_equal(a, b) for a, b in zip(got, want))
                # device-seeded batch with the on-device summary
                eng = engine.BatchEngine(L, W, n, 7)
                res = eng.run_batch(L)
                i = min(range(W), key=lambda j: (int(want[0][j]), j))
                ok &= (res.best_E, res.walker, res.steps_sum) == (int(want[0][i]), i, int(want[2].sum()))
                multi = eng.run_multi([7, 8], [L, 0])
                ok &= (multi[0].best_E, multi[0].walker) == (res.best_E, res.walker)
                print(f"L={L} layout={layout} variant={variant} batch {'ok' if ok else 'MISMATCH'}", flush=True)
                bad += not ok
        _lib.set_variant(_lib.VARIANT_AUTO)
        _lib.set_visited_layout(_lib.VISITED_AUTO)
        res, tr = run_walk_traced(WalkConfig(L=L, n=n, seed=oracle.derive_walk_seed(1, 0, 3)))
        be, st, dead, bw, tw, td = oracle.saw_walk(L, n, oracle.derive_walk_seed(1, 0, 3), record=True)
        ok = (res.best_E, res.steps_taken) == (be, st) and np.array_equal(tr.deltas, td[: st + (1 if dead else 0)])
        rng = np.random.default_rng(L)
        halves = rng.choice([-1, 1], size=(8, d)).astype(np.int8)
        halves[0] = 1
        moves = rng.integers(0, d, size=(8, 4)).astype(np.int32)
        got = _kernels.eval_states(L, halves, moves)
        for s in range(8):
            sv, cv, _ = oracle.init_state(L, halves[s].astype(np.int64))
            ok &= np.array_equal(got[s, 0], oracle.all_neighbor_deltas(L, sv, cv))
            for m in range(4):
                oracle.apply_neighbor(L, sv, cv, int(moves[s, m]))
                ok &= np.array_equal(got[s, m + 1], oracle.all_neighbor_deltas(L, sv, cv))
        print(f"L={L} trace+probe {'ok' if ok else 'MISMATCH'}", flush=True)
        bad += not ok
    torch.cuda.synchronize()
    print("sanitize workload:", "OK" if bad == 0 else f"{bad} MISMATCHES")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
