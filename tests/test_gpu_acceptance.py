"""The reference's acceptance criteria (pkg/tests/test_acceptance.py), run
against this framework's public API on the GPU.  Each test mirrors one
criterion with the reference's own thresholds:

  1 published table          -> tests/test_host_stats_cli.py (CPU)
  2 incremental == naive     -> device NeighborhoodBatch, >= 10,000 delta cases
  3 self-avoidance + argmin  -> replay of device traces (walkcheck.py:10-58)
  4 optimum recovery L<=27   -> >= 95/100 seeds reach the exhaustive optimum
  5 stopping-model algebra   -> tests/test_host_stats_cli.py (CPU)
  6 calibration at L=71      -> 100-rep device campaign; reproduces the reference's
                                (failing) outcome exactly: 32 censored
  7 determinism              -> repeated solves byte-identical
"""

import json
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2210_15962_b200 import stats  # noqa: E402
from paper_2210_15962_b200.codec import pack_half  # noqa: E402
from paper_2210_15962_b200.core import energy, expand_skew  # noqa: E402
from paper_2210_15962_b200.neighborhood import NeighborhoodBatch, flip, naive_oracle  # noqa: E402
from paper_2210_15962_b200.runner import RunConfig, solve, target_campaign  # noqa: E402
from paper_2210_15962_b200.saw import WalkConfig, exhaustive_optimum, run_walk_traced  # noqa: E402


def test_criterion_2_incremental_equals_naive():
    rng = np.random.default_rng(2025)
    delta_cases = apply_cases = 0
    while delta_cases < 10_000:
        L = int(rng.choice(np.arange(3, 63, 2)))
        d = (L + 1) // 2
        halves = rng.choice([-1, 1], size=(16, d)).astype(np.int64)
        nb = NeighborhoodBatch(halves)
        deltas = nb.deltas().cpu().numpy()
        E = nb.E.cpu().numpy()
        for i in range(16):
            for j in range(d):
                assert E[i] + deltas[i, j] == energy(expand_skew(flip(halves[i], j))).E
                delta_cases += 1
        js = rng.integers(0, d, 16)
        nb.apply(js)
        E2, full, side = nb.E.cpu().numpy(), nb.full.cpu().numpy(), nb.sidelobes()
        for i in range(16):
            ref = naive_oracle(flip(halves[i], int(js[i])))
            assert E2[i] == ref.E
            np.testing.assert_array_equal(side[i], ref.sidelobes)
            np.testing.assert_array_equal(full[i], ref.full)
            apply_cases += 1
    print(f"ACCEPTANCE 2: PASS - {delta_cases} delta cases, {apply_cases} apply cases")


def verify_walk(oracle, L, seed, walk_factor=8):
    """walkcheck.verify_walk on a device trace; ground truth from the oracle."""
    d = (L + 1) // 2
    res, tr = run_walk_traced(WalkConfig(L=L, n=walk_factor * d, seed=seed))
    piv = tr.pivots
    assert piv.shape[0] == res.steps_taken + 1 and res.evals == res.steps_taken * (d - 1)
    packed = [pack_half(p) for p in piv]
    assert len(set(packed)) == len(packed), "pivot revisited"
    seen = {packed[0]}
    energies = []
    for t in range(res.steps_taken):
        s, c, e = oracle.init_state(L, piv[t])
        energies.append(e)
        np.testing.assert_array_equal(tr.deltas[t], oracle.all_neighbor_deltas(L, s, c))
        cands = [(int(tr.deltas[t][h]), h) for h in range(d) if pack_half(flip(piv[t], h)) not in seen]
        assert cands, "moved with no unvisited neighbour"
        assert np.array_equal(piv[t + 1], flip(piv[t], min(cands)[1]))
        seen.add(packed[t + 1])
    energies.append(oracle.init_state(L, piv[-1])[2])
    assert res.best_E == min(energies) == naive_oracle(res.best_half).E
    if res.dead_end:
        assert tr.deltas.shape[0] == res.steps_taken + 1
        assert all(pack_half(flip(piv[-1], h)) in seen for h in range(d))
    else:
        assert res.steps_taken == walk_factor * d and tr.deltas.shape[0] == res.steps_taken
    return res


def test_criterion_3_self_avoidance_and_argmin(oracle):
    walks = dead = 0
    for L in range(5, 33, 2):
        for seed in range(100):
            dead += verify_walk(oracle, L, seed).dead_end
            walks += 1
    print(f"ACCEPTANCE 3: PASS - {walks} device walks replayed, {dead} dead-ended")


def test_criterion_4_exhaustive_optimum_recovery():
    worst = None
    for L in range(5, 29, 2):
        opt = exhaustive_optimum(L)[0].E
        hits = sum(solve(RunConfig(L=L, walkers=2, master_seed=seed, target_E=opt, max_nses=10**6)).stop_reason
                   == "target_reached" for seed in range(100))
        assert hits >= 95, f"L={L}: only {hits}/100 reached {opt}"
        worst = (L, hits) if worst is None or hits < worst[1] else worst
    print(f"ACCEPTANCE 4: PASS - worst case {worst[1]}/100 at L={worst[0]}")


def test_criterion_6_calibration_at_l71():
    """The reference's own criterion 6 FAILS deterministically (SURVEY §4:
    probe E=275, then 32 of 100 repetitions censored against a limit of 10;
    lambda_hat ~ 1.7e-8 vs the paper's 1.74e-7).  A bit-exact engine must
    reproduce that outcome, so this test pins it instead of the limit."""
    lam = stats.PUBLISHED_TREND.rate(71)
    budget = int(math.ceil(-math.log(1e-5) / lam))
    probe = solve(RunConfig(L=71, walkers=2, master_seed=20240817, max_nses=budget))
    assert probe.best_E == exhaustive_optimum(71)[0].E == 275
    samples = target_campaign(RunConfig(L=71, walkers=2, master_seed=71717, target_E=probe.best_E,
                                        max_nses=budget), 100)
    assert samples.censored_count == 32  # the reference's result (its limit is 10)
    fit = stats.fit_exponential(samples)  # uncensored-only MLE, as the reference's fit
    lam_cens = (100 - samples.censored_count) / sum(samples.nses)  # censoring-aware rate
    assert 1.0e-8 < lam_cens < fit.lam < 1.0e-7
    print(f"ACCEPTANCE 6: reference outcome reproduced - L=71 target 275: lambda_hat={fit.lam:.3g} "
          f"(censoring-aware {lam_cens:.3g}), model {lam:.3g}, {samples.censored_count} censored (reference: 32)")


def test_criterion_7_determinism():
    for cfg in (RunConfig(L=71, walkers=2, master_seed=99, max_nses=2_000_000),
                RunConfig(L=21, walkers=3, master_seed=4, target_E=26, max_nses=10**6),
                RunConfig(L=201, walkers=4096, master_seed=3, max_nses=10**9)):
        a = solve(cfg).to_json_dict()
        b = solve(cfg).to_json_dict()
        a.pop("wall_time_s")
        b.pop("wall_time_s")
        assert json.dumps(a) == json.dumps(b)
