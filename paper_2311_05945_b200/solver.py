"""Placeholder; replaced by the GPU engine binding."""
from dataclasses import dataclass


@dataclass
class SolverConfig:
    h: float = 0.01
    newton_tol: float = 1e-2
    max_newton_iters: int = 100
    max_line_search_halvings: int = 64
    ccd_conservative_factor: float = 0.9
    friction_fixed_point_iters: int = 1
    al_max_outer: int = 20
