"""Drop-in time step on the GPU (ref: pkg/src/srsim/solver.py).

``step(scene, config)`` has the reference's signature and semantics: it
advances the scene's bodies in place by one barrier-augmented implicit
Euler step (projected Newton, CCD-filtered line search, lagged friction,
augmented-Lagrangian kinematic targets, κ adaptation) and returns
``(state, StepReport)``. All of the per-step work runs in
``libipc_b200.so``; there is no CPU path.

Host ↔ device traffic per call: the scene's DoF state and velocities are
uploaded (the caller may have edited bodies between steps, e.g. a gripper
placement), then downloaded after the step together with κ and the
kinematic multipliers. ``GpuWorld`` (world.py) keeps batches resident.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from .world import GpuWorld

PHASES = ("DCD", "Energy", "Hess", "Linear", "CCD", "Others")


class IntersectionError(RuntimeError):
    """The incoming state already touches or penetrates (ref ccd.py:21)."""


@dataclass
class SolverConfig:
    """ref solver.py:56."""

    h: float = 0.01
    newton_tol: float = 1e-2
    max_newton_iters: int = 100
    max_line_search_halvings: int = 64
    ccd_conservative_factor: float = 0.9
    friction_fixed_point_iters: int = 1
    al_max_outer: int = 20

    def __post_init__(self):
        if self.h <= 0:
            raise ValueError("time step must be positive")
        if self.newton_tol <= 0:
            raise ValueError("newton_tol must be positive")
        if not 0.0 < self.ccd_conservative_factor < 1.0:
            raise ValueError("ccd_conservative_factor must lie in (0, 1)")


# device work -> reference phase (ref solver.py:52 PHASES, timed at :303-352):
# per-kernel CUDA-event times of the batched launch sequence, and the
# per-phase SM cycles of the fused per-env kernels that finish each Newton loop
KERNEL_PHASE = {"broad_dcd": "DCD", "broad_ccd": "CCD", "ccd": "CCD", "pairs_deriv": "Energy",
                "pairs_value": "Energy", "tet": "Energy", "body": "Energy", "ground": "Energy",
                "friction": "Energy", "energy_reduce": "Energy", "lags": "Energy", "world_pos": "Energy",
                "assembly": "Hess", "dense_solve": "Linear", "pcg": "Linear"}
FUSED_PHASE = {"world": "Energy", "broad_dcd": "DCD", "terms": "Energy", "energy": "Energy",
               "dense": "Linear", "ccd_prep": "CCD", "broad_ccd": "CCD", "ccd": "CCD",
               "line_search": "Energy"}


@dataclass
class StepReport:
    """ref solver.py:75. ``times`` splits the step's device time into the
    reference's phases (DCD / Energy / Hess / Linear / CCD) from the
    per-kernel CUDA events and the fused kernels' phase timers; ``Others`` is
    the remainder of the step's wall time, as ref solver.py:88 closes it.
    The dense per-env solve assembles and factors in one kernel, so its
    assembly is booked under Linear (the sparse path books BSR assembly
    under Hess)."""

    newton_iters: int = 0
    final_grad_norm: float = 0.0
    min_dist_before: float = np.inf
    min_dist_after: float = np.inf
    ccd_invocations: int = 0
    converged: bool = True
    line_search_failed: bool = False
    al_outer: int = 0
    times: dict = field(default_factory=lambda: {k: 0.0 for k in PHASES})
    total_time: float = 0.0

    def as_dict(self) -> dict:
        return {"newton_iters": self.newton_iters, "final_grad_norm": self.final_grad_norm,
                "min_dist_before": self.min_dist_before, "min_dist_after": self.min_dist_after,
                "ccd_invocations": self.ccd_invocations, "converged": self.converged,
                "line_search_failed": self.line_search_failed, "al_outer": self.al_outer,
                "times": dict(self.times), "total_time": self.total_time}

    @classmethod
    def from_c(cls, r, t, phases=None):
        rep = cls(newton_iters=r.newton_iters, final_grad_norm=r.final_grad_norm,
                  min_dist_before=r.min_dist_before, min_dist_after=r.min_dist_after,
                  ccd_invocations=r.ccd_invocations, converged=bool(r.converged),
                  line_search_failed=bool(r.line_search_failed), al_outer=r.al_outer)
        rep.total_time = t
        for k, v in (phases or {}).items():
            rep.times[k] += v
        accounted = sum(v for k, v in rep.times.items() if k != "Others")
        rep.times["Others"] = max(t - accounted, 0.0)
        return rep


class _PhaseClock:
    """Per-step phase seconds of one device world (differences of the
    cumulative kernel-event and fused-timer counters)."""

    def __init__(self, w: GpuWorld):
        self.w = w
        w.profile(True)
        w.set_fused_timers(True)
        self.hz = 1e3 * w.clock_khz()
        self.prev = self._read()

    def _read(self):
        prof, _ = self.w.profile_read()
        return {k: v[0] for k, v in prof.items()}, self.w.fused_timers()

    def split(self) -> dict:
        (ms0, ft0), (ms1, ft1) = self.prev, self._read()
        self.prev = (ms1, ft1)
        out = {k: 0.0 for k in PHASES}
        for k, ph in KERNEL_PHASE.items():
            out[ph] += 1e-3 * (ms1.get(k, 0.0) - ms0.get(k, 0.0))
        for k, ph in FUSED_PHASE.items():
            out[ph] += (ft1.get(k, 0) - ft0.get(k, 0)) / self.hz
        out.pop("Others")
        return out


_ENGINES: dict = {}  # id(scene) -> GpuWorld, dropped when the scene is collected


def engine_of(scene) -> GpuWorld:
    """The device world bound to ``scene``, created on first use.

    The cache lives here, keyed by the scene's identity and released by a
    weakref finalizer, so any object with the reference Scene's fields works
    (an unmodified ``srsim.scene.Scene`` has no engine slot, ref
    scene.py:112; the dataclass is unhashable, hence no WeakKeyDictionary)."""
    key = id(scene)
    w = _ENGINES.get(key)
    if w is None:
        w = GpuWorld([scene])
        if hasattr(w, "profile"):
            w.phase_clock = _PhaseClock(w)
        _ENGINES[key] = w
        weakref.finalize(scene, _ENGINES.pop, key, None)
    return w


def release_engine(scene) -> None:
    """Drop the device world of ``scene`` (the next step re-uploads it)."""
    _ENGINES.pop(id(scene), None)


def convergence_check(p, h: float, tol: float) -> bool:
    """‖p‖∞ / h ≤ tol (ref solver.py:234)."""
    p = np.asarray(p)
    return True if len(p) == 0 else bool(np.abs(p).max() / h <= tol)


def _sync_to_device(scene, w: GpuWorld):
    st = scene.state
    w.set_state(st.gather(), st.gather_velocity())
    w.set_kappa(np.array([scene.barrier.kappa]))


def _scatter_velocity(state, v) -> None:
    """Velocities through the bodies' own fields (q_dot / v), as ref
    bodies.py:315-326 finalize_step writes them; the reference GlobalState
    has no scatter_velocity."""
    for blk in state.blocks:
        seg = np.array(v[blk.offset:blk.offset + blk.dof], dtype=np.float64)
        if blk.is_affine:
            blk.body.q_dot = seg
        else:
            blk.body.v = seg.reshape(-1, 3)


def _sync_from_device(scene, w: GpuWorld, h):
    x, v = w.get_state()
    scene.state.scatter(x)
    _scatter_velocity(scene.state, v)
    k = float(w.get_kappa()[0])
    if k != scene.barrier.kappa:
        scene.barrier = type(scene.barrier)(scene.barrier.dhat, k)
    if scene.constraints:
        lam, kap = w.get_constraints()
        for c, l, kk in zip(scene.constraints, lam, kap):
            c.lam = l.copy()
            c.kappa = float(kk)
            if c.body.target_q is not None:  # ref solver.py:399-400
                c.target = np.asarray(c.body.target_q, dtype=np.float64).copy()


def step(scene, config: SolverConfig):
    """Advance one time step on the GPU; returns (state, StepReport)
    (ref solver.py:360). Raises IntersectionError on an intersecting start."""
    t0 = time.perf_counter()
    w = engine_of(scene)
    _sync_to_device(scene, w)
    reps = w.step(config)
    r = reps[0]
    if r.error:
        raise IntersectionError("step started from an intersecting state")
    _sync_from_device(scene, w, config.h)
    phases = w.phase_clock.split() if hasattr(w, "phase_clock") else None
    return scene.state, StepReport.from_c(r, time.perf_counter() - t0, phases)


def simulate(scene, config: SolverConfig, n_steps: int, callback=None):
    """ref solver.py:457."""
    out = []
    for i in range(n_steps):
        _, rep = step(scene, config)
        out.append(rep)
        if callback is not None:
            callback(i, scene, rep)
    return out


class _GpuBackend:
    """Grasp-driver backend on the GPU engine (robot/grasp.py)."""

    def step(self, scene, cfg):
        return step(scene, cfg)

    def finger_forces(self, scene, gripper, h):
        w = engine_of(scene)
        _sync_to_device(scene, w)
        groups = np.array([[w.mask(0, [gripper.links[ln] for ln in gripper.finger_groups[fn]])
                            for fn in gripper.finger_names]], dtype=np.uint64)
        f = w.group_forces(h, groups)[0]
        return np.linalg.norm(f, axis=1)

    def min_group_distance(self, scene, a, b):
        w = engine_of(scene)
        _sync_to_device(scene, w)
        return float(w.group_distance(np.array([w.mask(0, a)], np.uint64),
                                      np.array([w.mask(0, b)], np.uint64))[0])

    def min_ground_distance(self, scene, bodies):
        if scene.ground_y is None:
            return np.inf
        w = engine_of(scene)
        _sync_to_device(scene, w)
        return float(w.ground_distance(np.array([w.mask(0, bodies)], np.uint64))[0])


GPU_BACKEND = _GpuBackend()
