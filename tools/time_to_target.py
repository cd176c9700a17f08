"""Time-to-target on one B200 (BASELINE config 3) and the lambda(L) calibration
of the paper's stopping model, from device-concurrent
target campaigns.

    python tools/time_to_target.py --lengths 71,75,79,101,121 --reps 100
    python tools/time_to_target.py --direct 171,185 --direct-seeds 3 --max-runtime 900

Targets per L: the exact optimum from the device exhaustive scan (L <= 93),
else the published best-known energy (L >= 171, published.py), else the best
energy of a probe search (the reference's criterion-6 procedure,
test_acceptance.py:140-160).  Each campaign runs `--reps` repetitions
concurrently (runner.target_campaign); per L it prints one JSON line with
lambda_hat = 1/mean(NSEs to target), the Anderson-Darling A^2, the paper
model's lambda(L), the device NSE/s of the campaign and the implied mean
time-to-target on the GPU and on the host cores (mean NSEs / the CPU
reference rate, --cpu-nse-per-s, measured by bench.py --impl reference).
`--direct L` runs one solve with the published target and reports the wall
time until it is reached.
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pow2_clip(x, lo, hi):
    v = 1 << max(0, int(math.log2(max(1.0, x))))
    return max(lo, min(hi, v))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--walk-factor", type=int, default=8)
    ap.add_argument("--probe-seconds", type=float, default=20.0)
    ap.add_argument("--budget-factor", type=float, default=30.0, help="per-rep NSE budget = factor / lambda_model")
    ap.add_argument("--cpu-nse-per-s", type=float, default=9.0e7,
                    help="host reference rate (bench.py --impl reference on the GPU box, L=201)")
    ap.add_argument("--direct", default="", help="comma-separated L with a published target")
    ap.add_argument("--direct-seeds", type=int, default=1)
    ap.add_argument("--max-runtime", type=float, default=900.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--exhaustive-max-d", type=int, default=40, help="largest D whose target comes from the scan")
    a = ap.parse_args()

    import torch

    from paper_2210_15962_b200 import published, stats
    from paper_2210_15962_b200.runner import RunConfig, solve, target_campaign
    from paper_2210_15962_b200.saw import MAX_EXHAUSTIVE_D, exhaustive_optimum

    torch.cuda.init()
    points = []
    if a.direct:
        for L in [int(x) for x in a.direct.split(",") if x]:
            row = published.best_known(L)
            if row is None:
                raise SystemExit(f"no published target for L={L}")
            for seed in range(a.seed, a.seed + a.direct_seeds):
                t0 = time.monotonic()
                rec = solve(RunConfig(L=L, walkers=1 << 20, walk_factor=a.walk_factor, master_seed=seed,
                                      target_E=row.E, max_runtime=a.max_runtime))
                dt = time.monotonic() - t0
                print(json.dumps({"mode": "direct", "L": L, "seed": seed, "target_E": row.E,
                                  "reached": rec.stop_reason == "target_reached", "best_E": rec.best_E,
                                  "best_hex": rec.best_hex, "seconds": dt, "total_nses": rec.total_nses,
                                  "nse_per_s": rec.total_nses / dt,
                                  "model_expected_nses": 1.0 / stats.PUBLISHED_TREND.rate(L),
                                  "cpu_predicted_seconds": rec.total_nses / (a.cpu_nse_per_s * 101.0 / ((L + 1) // 2))}),
                      flush=True)
        return

    for L in [int(x) for x in a.lengths.split(",") if x]:
        D = (L + 1) // 2
        lam_model = stats.PUBLISHED_TREND.rate(L)
        if D <= MAX_EXHAUSTIVE_D and D <= a.exhaustive_max_d:
            t0 = time.monotonic()
            target = exhaustive_optimum(L)[0].E
            source, tsrc = "exhaustive optimum (device scan)", time.monotonic() - t0
        elif published.best_known(L) is not None:
            target, source, tsrc = published.best_known(L).E, "published best-known", 0.0
        else:
            t0 = time.monotonic()
            probe = solve(RunConfig(L=L, walkers=1 << 18, walk_factor=a.walk_factor, master_seed=20240817,
                                    max_runtime=a.probe_seconds))
            target, source, tsrc = probe.best_E, f"probe best ({a.probe_seconds:.0f} s search)", time.monotonic() - t0
        per_walk = a.walk_factor * D * (D - 1)
        W = pow2_clip(0.25 / lam_model / per_walk, 16, 1 << 16)
        budget = int(a.budget_factor / lam_model)
        cfg = RunConfig(L=L, walkers=W, walk_factor=a.walk_factor, master_seed=a.seed, target_E=target,
                        max_nses=budget)
        torch.cuda.synchronize()
        t0 = time.monotonic()
        samples = target_campaign(cfg, a.reps)
        dt = time.monotonic() - t0
        total = sum(samples.nses)
        out = {"mode": "campaign", "L": L, "target_E": target, "target_source": source,
               "target_seconds": tsrc, "reps": a.reps, "walkers_per_rep": W, "budget_per_rep": budget,
               "censored": samples.censored_count, "campaign_seconds": dt, "campaign_nse_per_s": total / dt,
               "lambda_model": lam_model}
        if samples.uncensored:
            fit = stats.fit_exponential(samples)
            a2 = stats.anderson_darling_exponential(samples, fit)
            rate = total / dt
            out.update({"lambda_hat": fit.lam, "mean_nses": fit.mean_nses, "a2": a2,
                        "lambda_ratio_hat_over_model": fit.lam / lam_model,
                        "gpu_mean_time_to_target_s": fit.mean_nses / rate,
                        # the CPU cost per NSE grows like D (D lag terms per NSE): scale the L=201 rate
                        "cpu_mean_time_to_target_s": fit.mean_nses / (a.cpu_nse_per_s * 101.0 / D)})
            points.append((L, fit.lam))
        print(json.dumps(out), flush=True)
    if len({p[0] for p in points}) >= 2:
        print(json.dumps({"mode": "trend", "fit": stats.fit_lambda_trend(points).to_json_dict(),
                          "paper": stats.PUBLISHED_TREND.to_json_dict()}), flush=True)


if __name__ == "__main__":
    main()
