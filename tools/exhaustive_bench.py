"""Throughput of the device exhaustive scan.

    python tools/exhaustive_bench.py --lengths 55,61,67,71 [--cpu-length 41]

Per L: one full scan through sk_exhaustive_scan_host (the drop-in of
_kernels.exhaustive_scan), wall-timed around the synchronous call; prints
one JSON line with E, the argmin hex, seconds and Gray steps/s.  The CPU
oracle (single thread, the reference's algorithm) is timed at --cpu-length
for a same-box baseline.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="55,61,67,71")
    ap.add_argument("--cpu-length", type=int, default=41)
    a = ap.parse_args()
    import torch

    from paper_2210_15962_b200 import _kernels
    from paper_2210_15962_b200.codec import encode
    from paper_2210_15962_b200.saw import exhaustive_optimum

    torch.cuda.init()
    _kernels.exhaustive_scan(21)  # module load / warm-up
    for L in [int(x) for x in a.lengths.split(",")]:
        t0 = time.perf_counter()
        rec, half = exhaustive_optimum(L)
        dt = time.perf_counter() - t0
        D = (L + 1) // 2
        print(json.dumps({"L": L, "D": D, "E": rec.E, "F": rec.F, "hex": encode(half), "seconds": dt,
                          "gray_steps_per_s": (1 << D) / dt, "impl": "device"}), flush=True)
    if a.cpu_length:
        import oracle

        oracle.build()
        L = a.cpu_length
        t0 = time.perf_counter()
        e, bits = oracle.exhaustive_scan(L)
        dt = time.perf_counter() - t0
        D = (L + 1) // 2
        print(json.dumps({"L": L, "D": D, "E": e, "seconds": dt, "gray_steps_per_s": (1 << D) / dt,
                          "impl": "cpu oracle (reference algorithm, 1 thread)"}), flush=True)


if __name__ == "__main__":
    main()
