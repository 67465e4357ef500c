"""paper_2402_15678_b200 — B200-native speculate-vote-verify (Minions, arXiv 2402.15678).

The reference package's hot-path API (aggspec/__init__.py:58-100) re-exported
under the same names; the compute behind it is libminions.so (sm_100a
kernels, C-ABI in include/minions.h).  Importing the device-facing modules
requires the built library: there is no CPU fallback.
"""
from .core import (  # noqa: F401
    AggSpecError,
    ConfigInvalid,
    ContextTooLong,
    DistMismatch,
    EngineConfig,
    IllegalTransition,
    InvalidSample,
    LengthMismatch,
    ProbDist,
    Request,
    RequestState,
    UnknownSSM,
    seeded_rng,
    tv_distance,
    validate_config,
)
from .selector import (  # noqa: F401
    Decision,
    MonitorSample,
    SelectorState,
    geometric_vl,
    maybe_adjust,
    observe,
    optimal_s_oracle,
)

# Device-facing names load libminions.so on first use (so that `build` can run
# before the library exists); a missing library raises there — no fallback.
_LAZY = {
    "VerificationResult": "verification", "acceptance_rate": "verification", "verify": "verification",
    "MajorityOutput": "voting", "SpeculationTree": "voting", "WeightTable": "voting",
    "merge": "voting", "record_acr": "voting", "select_majority": "voting",
    "update_weights": "voting",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
