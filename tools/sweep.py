"""Throughput sweep over sequence lengths / walk factors (BASELINE configs 3, 5).

    python tools/sweep.py --lengths 27,101,201,301,449 --walk-factors 8 --seconds 2

For each (L, walk_factor): device-derived seeds, one batch sized to ~`seconds`
of work, CUDA-event timed after a warm-up batch.  Prints one JSON line per point
with NSE/s, walk steps/s, lag-terms/s and the best energy / merit factor seen.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="27,101,121,151,171,201,223,255,257,301,401,449,511,1023")
    ap.add_argument("--walk-factors", default="8")
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--variant", default="fast", choices=["fast", "scalar"])
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2210_15962_b200 import _lib, engine

    lib = _lib.load()
    _lib.set_variant(_lib.VARIANT_FAST if a.variant == "fast" else _lib.VARIANT_SCALAR)
    _lib.set_visited_layout(int(os.environ.get("SK_SWEEP_LAYOUT", "0")))
    dev = torch.device("cuda", 0)
    summ = torch.empty(engine.SUMMARY_WORDS, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream()
    for L in [int(x) for x in a.lengths.split(",")]:
        for wf in [int(x) for x in a.walk_factors.split(",")]:
            D = (L + 1) // 2
            n = wf * D
            res = lib.sk_resident_walks(L, n)
            W = max(int(res), 1024)

            def run(W, batch):
                _lib.check(lib.sk_saw_batch(L, n, None, 1, batch, 0, W, None, None, None, None,
                                            summ.data_ptr(), st.cuda_stream))

            run(W, 99)  # warm-up + calibration
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(W, 98)
            e1.record()
            torch.cuda.synchronize()
            t1 = e0.elapsed_time(e1) / 1e3
            W2 = int(W * max(1.0, a.seconds / max(t1, 1e-6)))
            W2 = min(W2, 1 << 22)
            e0.record()
            run(W2, 0)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            r = engine.decode_summary(summ.cpu().numpy().view(np.uint64), (D + 63) // 64)
            nse = r.steps_sum * (D - 1)
            print(json.dumps({"L": L, "walk_factor": wf, "n": n, "walkers": W2, "resident": int(res),
                              "seconds": t, "nse_per_s": nse / t, "walk_steps_per_s": r.steps_sum / t,
                              "lag_terms_per_s": nse * D / t, "best_E": r.best_E,
                              "best_F": L * L / (2.0 * r.best_E), "variant": a.variant}), flush=True)


if __name__ == "__main__":
    main()
