"""paper_1708_06290_b200 -- B200-native batched shifted solver.

Drop-in for the shifted-solve hot path of the reference package
``shiftsolve`` (arXiv 1708.06290): the one-time controller-Hessenberg
reduction and the batched window RQ solves that evaluate
``G(sigma) = C (sigma I - A)^{-1} B`` for many complex shifts, computed by
hand-written sm_100a CUDA behind the C ABI in include/shiftsolve_b200.h.
"""

from .counters import PhaseCounters
from .errors import (
    DimensionMismatchError,
    EigensolverError,
    SingularDiagonalError,
    SingularShiftError,
)
from .hessenberg import ControllerHessForm, reduce_controller_hessenberg
from .irka import (
    IrkaState,
    IterationRecord,
    ReducedModel,
    default_initial_data,
    irka_iterate,
    pair_conjugates,
    relative_hausdorff,
    small_eig_pencil,
)
from .schedule import AnnihilationSchedule, greedy_schedule, mirrored_schedule
from .solvers import (
    ShiftedSolveResult,
    TransferFunctionResult,
    default_singular_rtol,
    eval_transfer_function,
    residual_certificate,
    solve_shifted_reduced,
    solve_shifted_transposed,
    structured_pseudospectrum_grid,
    two_norm_small,
)
from .systems import SystemBundle, random_stable_system

__version__ = "0.1.0"

__all__ = [
    "AnnihilationSchedule",
    "IrkaState",
    "IterationRecord",
    "ReducedModel",
    "default_initial_data",
    "irka_iterate",
    "pair_conjugates",
    "relative_hausdorff",
    "small_eig_pencil",
    "ControllerHessForm",
    "DimensionMismatchError",
    "EigensolverError",
    "PhaseCounters",
    "ShiftedSolveResult",
    "SingularDiagonalError",
    "SingularShiftError",
    "SystemBundle",
    "TransferFunctionResult",
    "default_singular_rtol",
    "eval_transfer_function",
    "greedy_schedule",
    "random_stable_system",
    "reduce_controller_hessenberg",
    "residual_certificate",
    "solve_shifted_reduced",
    "solve_shifted_transposed",
    "mirrored_schedule",
    "structured_pseudospectrum_grid",
    "two_norm_small",
]
