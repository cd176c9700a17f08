"""B200-native sokol_skew: parallel self-avoiding walks for skew-symmetric LABS.

Drop-in for the hot path of the reference package ``skewsaw`` (arXiv
2210.15962): the walk engine (``_kernels.saw_batch`` / ``saw_walk``), the
walk API (``saw``) and the solver loop (``runner``), with the same names,
argument meaning, validation and result records.  Walks run on sm_100a CUDA
kernels in ``libsokol.so`` (C ABI: include/sokol.h) loaded through ctypes;
there is no CPU execution path.
"""

from .codec import DecodeError, decode, encode
from .core import (
    EnergyRecord,
    autocorrelation,
    autocorrelations,
    energy,
    expand_skew,
    half_dim,
    merit_factor,
    sidelobe_array,
)
from .neighborhood import EvalState, apply_flip, compute_deltas, flip, naive_oracle
from .published import BEST_KNOWN, KnownResult
from .stats import (
    PUBLISHED_TREND,
    ExpFit,
    TrendModel,
    anderson_darling_exponential,
    fit_exponential,
    fit_lambda_trend,
    nses_limit,
    optimality_probability,
)
from .runner import (
    RunConfig,
    RunRecord,
    SampleSet,
    derive_repetition_seed,
    derive_walk_seed,
    solve,
    target_campaign,
    throughput_report,
)
from .saw import (
    MAX_EXHAUSTIVE_D,
    WalkConfig,
    WalkResult,
    WalkTrace,
    exhaustive_optimum,
    key,
    run_walk,
    run_walk_traced,
)

__version__ = "0.1.0"

__all__ = [
    "DecodeError", "decode", "encode", "EnergyRecord", "autocorrelation", "autocorrelations", "energy",
    "expand_skew", "half_dim", "merit_factor", "sidelobe_array", "EvalState", "apply_flip", "compute_deltas",
    "flip", "naive_oracle", "BEST_KNOWN", "KnownResult", "PUBLISHED_TREND", "ExpFit", "TrendModel",
    "anderson_darling_exponential", "fit_exponential", "fit_lambda_trend", "nses_limit", "optimality_probability", "RunConfig", "RunRecord", "SampleSet", "derive_repetition_seed",
    "derive_walk_seed", "solve", "target_campaign", "throughput_report", "WalkConfig",
    "WalkResult", "WalkTrace", "key", "run_walk", "run_walk_traced", "MAX_EXHAUSTIVE_D",
    "exhaustive_optimum",
]
