"""Barrier parameters and stiffness schedule (ref: pkg/src/srsim/energy/barrier.py).

The barrier itself, b(s) = −(s − ŝ)² ln(s/ŝ) on squared distance s < ŝ,
is evaluated on the device (csrc/ipc_math.cuh); only the scalar schedule
lives on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KAPPA_GROWTH_CAP = 1e8  # ref barrier.py:82


@dataclass
class BarrierParams:
    dhat: float
    kappa: float

    def __post_init__(self):
        if self.dhat <= 0 or self.kappa <= 0:
            raise ValueError("dhat and kappa must be positive")

    @property
    def shat(self) -> float:
        return self.dhat * self.dhat


def kappa_init(avg_vertex_mass: float, dhat: float) -> float:
    """ref barrier.py:77."""
    return 1e4 * avg_vertex_mass / (dhat * dhat)


def adapt_kappa(params: BarrierParams, min_dist: float, kappa0: float) -> BarrierParams:
    """Double κ while contacts sit closer than 1e-4 d̂ (ref barrier.py:85)."""
    if min_dist < 1e-4 * params.dhat and params.kappa < KAPPA_GROWTH_CAP * kappa0:
        return BarrierParams(params.dhat, min(2.0 * params.kappa, KAPPA_GROWTH_CAP * kappa0))
    return params


def barrier(d, dhat: float):
    """Public meter-form barrier b(d) and db/dd (ref barrier.py:30)."""
    d = np.asarray(d, dtype=np.float64)
    if np.any(d <= 0):
        raise ValueError("barrier evaluated at non-positive distance")
    scalar = d.ndim == 0
    d = np.atleast_1d(d)
    b = np.zeros_like(d)
    db = np.zeros_like(d)
    m = d < dhat
    g = d[m] - dhat
    ln = np.log(d[m] / dhat)
    b[m] = -g * g * ln
    db[m] = -2.0 * g * ln - g * g / d[m]
    if scalar:
        return float(b[0]), float(db[0])
    return b, db
