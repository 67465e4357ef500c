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
from .verification import VerificationResult, acceptance_rate, verify  # noqa: F401
from .voting import (  # noqa: F401
    MajorityOutput,
    SpeculationTree,
    WeightTable,
    merge,
    record_acr,
    select_majority,
    update_weights,
)
