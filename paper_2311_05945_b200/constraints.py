"""Augmented-Lagrangian kinematic targets (ref: pkg/src/srsim/constraints.py).

    E_A(q, λ) = (κ_A/2)‖q − q̃‖² − √m_k λ·(q − q̃)

Energy, gradient and Hessian (κ_A I) are evaluated on the GPU inside the
Newton assembly; the multiplier update after each inner solve runs on the
device too. The dataclass here is the host-side record the scene carries.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .bodies import AffineBody

KAPPA_A_GROWTH_CAP = 1e6  # ref constraints.py:23


def default_kinematic_stiffness(body_mass: float, h: float) -> float:
    """ref constraints.py:26."""
    return 1e6 * body_mass / (h * h)


@dataclass
class KinematicConstraint:
    """Target tracking for a kinematic affine body (ref constraints.py:36)."""

    body: AffineBody
    target: np.ndarray
    kappa: float
    mass_scale: float
    lam: np.ndarray = field(default_factory=lambda: np.zeros(12))
    kappa0: float = 0.0
    last_residual: float = np.inf

    def __post_init__(self):
        if self.kappa <= 0:
            raise ValueError("kinematic penalty stiffness must be positive")
        if not self.body.kinematic:
            raise ValueError("kinematic constraint on a non-kinematic body")
        self.target = np.asarray(self.target, dtype=np.float64)
        if self.kappa0 == 0.0:
            self.kappa0 = self.kappa


def kinematic_value(c: KinematicConstraint, q_b) -> float:
    d = np.asarray(q_b) - c.target
    return 0.5 * c.kappa * (d @ d) - np.sqrt(c.mass_scale) * (c.lam @ d)
