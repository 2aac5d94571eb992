"""B200-native (sm_100a) low-rank Matrix Exponentiated Gradient hot path (arXiv 2012.10469).

Drop-in for the per-iteration path of the reference `specmeg` package:
`meg.lowrank_meg_step` and the `linalg.lanczos_top_r` it calls, with the same
names, arguments, results and errors.  All numerics run in hand-written CUDA
kernels in libmegb200.so (csrc/), called through the C ABI of
include/megb200.h; there is no CPU fallback.
"""

from .errors import EighError, LanczosError, ParameterError, RankDeficiencyError
from .linalg import SymmetricOperator, TopREigen, lanczos_top_r, project_simplex, symmetrize
from .meg import (
    CertificateRecord,
    EpsilonSchedule,
    LogmapOperator,
    LowRankIterate,
    HostStepResult,
    HostStepper,
    LowRankStepResult,
    StepConfig,
    certificate_cheap,
    certificate_full,
    eps_schedule_eval,
    logmap_operator,
    lowrank_meg_step,
    lowrank_meg_step_host,
    merge_certificates,
    step_eval,
    warm_start_wrap,
)
from .callbacks import device_callable
from .shadow import BregmanValue, bregman, bregman_structured, exact_meg_step, shadow_lowrank_step
from .objectives import (
    CallbackGradient,
    DenseGradient,
    FrobeniusObjective,
    GradientOperator,
    QuadMeasObjective,
    QuadMeasStochasticOracle,
    SampledObjective,
    StochasticFrobeniusObjective,
    ZeroGradient,
)

__all__ = [
    "BregmanValue", "bregman", "bregman_structured", "exact_meg_step", "shadow_lowrank_step",
    "CallbackGradient", "CertificateRecord", "DenseGradient", "device_callable", "HostStepResult", "HostStepper", "EighError", "EpsilonSchedule", "FrobeniusObjective", "GradientOperator",
    "LanczosError", "LogmapOperator", "QuadMeasObjective", "QuadMeasStochasticOracle", "LowRankIterate", "LowRankStepResult", "ParameterError", "RankDeficiencyError",
    "SampledObjective", "StepConfig", "StochasticFrobeniusObjective", "SymmetricOperator", "TopREigen",
    "ZeroGradient", "certificate_cheap", "certificate_full", "eps_schedule_eval", "lanczos_top_r", "logmap_operator",
    "lowrank_meg_step", "lowrank_meg_step_host", "merge_certificates", "project_simplex", "step_eval", "symmetrize", "warm_start_wrap",
]
