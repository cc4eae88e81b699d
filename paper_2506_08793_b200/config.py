"""Solver configuration and result records of the drop-in API.

Same field names, defaults, validation and error type as the reference's
SolverConfig / SolverTrace / DehazeResult (pdehaze/solver.py:56-149), so a
reference user can pass the same objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["ABLATIONS", "LAMBDA_MODES", "SolverConfig", "SolverTrace", "DehazeResult",
           "normalize_ablation"]

#: stage switches of dehaze (solver.py:56-63); none set = full model
ABLATIONS = (
    "no-pde",
    "no-nonlocal",
    "no-adaptive",
    "no-edge",
    "no-guided",
    "no-multiscale",
)

#: the two readings of the adaptive weight (solver.py:65, :262)
LAMBDA_MODES = ("as-printed", "prose")


@dataclass(frozen=True)
class SolverConfig:
    """Pipeline tunables with the reference defaults (solver.py:78-94)."""

    epsilon: float = 1e-3
    sigma: float = 2.0
    kernel_size: int = 5
    lambda0: float = 0.5
    beta: float = 3.0
    tau: float = 0.2
    t_floor: float = 0.1
    omega: float = 0.95
    patch_radius: int = 7
    max_iters: int = 200
    rel_tol: float = 1e-4
    lambda_monotonicity: str = "as-printed"
    guided_radius: int = 30
    guided_reg: float = 1e-3
    multiscale_radii: tuple[int, ...] = (3, 7, 15)
    multiscale_weights: tuple[float, ...] | None = None
    airlight_fraction: float = 0.001

    def __post_init__(self):
        checks = (
            (self.epsilon > 0.0, "epsilon must be > 0"),
            (self.sigma > 0.0, "sigma must be > 0"),
            (self.kernel_size >= 1 and self.kernel_size % 2 == 1,
             "kernel_size must be odd and >= 1"),
            (self.lambda0 > 0.0, "lambda0 must be > 0"),
            (self.beta >= 0.0, "beta must be >= 0"),
            (self.tau > 0.0, "tau must be > 0"),
            (self.t_floor > 0.0, "t_floor must be > 0"),
            (0.0 < self.omega <= 1.0, "omega must lie in (0, 1]"),
            (self.patch_radius >= 0, "patch_radius must be >= 0"),
            (self.max_iters >= 1, "max_iters must be >= 1"),
            (self.rel_tol > 0.0, "rel_tol must be > 0"),
            (self.lambda_monotonicity in LAMBDA_MODES,
             f"lambda_monotonicity must be one of {LAMBDA_MODES}"),
            (self.guided_radius >= 1, "guided_radius must be >= 1"),
            (self.guided_reg > 0.0, "guided_reg must be > 0"),
            (bool(self.multiscale_radii), "multiscale_radii must be nonempty"),
            (0.0 < self.airlight_fraction <= 1.0, "airlight_fraction must lie in (0, 1]"),
        )
        for ok, message in checks:
            if not ok:
                raise ValueError(message)


@dataclass
class SolverTrace:
    """Per-channel iteration record (solver.py:131-139)."""

    residual_norms: list[float] = field(default_factory=list)
    iterations_run: int = 0
    converged: bool = False
    tau_used: float = 0.0
    tau_bound: float = 0.0


@dataclass
class DehazeResult:
    """Intermediate products returned by dehaze (solver.py:142-149)."""

    airlight: np.ndarray
    transmission: np.ndarray
    traces: list[SolverTrace]
    ablation: frozenset[str]


def normalize_ablation(ablation) -> frozenset[str]:
    """None / one name / iterable of names -> validated frozenset (solver.py:362-372)."""
    if ablation is None:
        flags: frozenset[str] = frozenset()
    elif isinstance(ablation, str):
        flags = frozenset((ablation,))
    else:
        flags = frozenset(ablation)
    unknown = flags - set(ABLATIONS)
    if unknown:
        raise ValueError(f"unknown ablation flags {sorted(unknown)}; known: {ABLATIONS}")
    return flags
