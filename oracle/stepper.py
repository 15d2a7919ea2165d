"""Oracle: one implicit time step — projected Newton with CCD-filtered
backtracking, lagged friction, augmented-Lagrangian kinematic targets and
barrier-stiffness adaptation. TEST INFRASTRUCTURE ONLY.

Restates ref pkg/src/srsim/solver.py (step :360, _newton_solve :295,
_assemble :146, _total_value :178, newton_iteration :241,
filtered_line_search :257, friction_update :275) on the scene data format
of ``paper_2311_05945_b200.scene`` (which mirrors ref scene.py).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import collide as C
from . import energies as E

ALPHA_FLOOR = 1e-12  # ref solver.py:49
AL_TOL = 1e-6        # ref solver.py:50
KAPPA_A_GROWTH_CAP = 1e6
KAPPA_GROWTH_CAP = 1e8


@dataclass
class Config:
    h: float = 0.01
    newton_tol: float = 1e-2
    max_newton_iters: int = 100
    max_line_search_halvings: int = 64
    ccd_conservative_factor: float = 0.9
    friction_fixed_point_iters: int = 1
    al_max_outer: int = 20


@dataclass
class Report:
    newton_iters: int = 0
    final_grad_norm: float = 0.0
    min_dist_before: float = np.inf
    min_dist_after: float = np.inf
    ccd_invocations: int = 0
    converged: bool = True
    line_search_failed: bool = False
    al_outer: int = 0
    total_time: float = 0.0
    alphas: list = field(default_factory=list)
    pnorms: list = field(default_factory=list)  # ‖p‖∞ of every Newton direction


class Layout:
    """Per-scene mass blocks / orthogonality coefficients / soft bodies."""

    def __init__(self, scene):
        st = scene.state
        self.mass_blocks = []
        self.ortho = []
        self.soft = []
        for blk in st.blocks:
            if blk.is_affine:
                self.mass_blocks.append((blk.offset, 12, blk.body.M_b))
                self.ortho.append((blk.offset, blk.body.stiffness * blk.body.volume))
            else:
                self.mass_blocks.append((blk.offset, blk.dof, blk.body.mass))
                self.soft.append((blk.offset, blk.dof, blk.body))
        self.n_dof = st.n_dof


def _constraint_terms(scene, x):
    out = []
    for c in scene.constraints:
        off = scene.state.offset_of(c.body)
        out.append(E.kinematic(c, x[off:off + 12], off))
    return out


def assemble(scene, lay, x, xhat, xw0, lags, cand, h):
    """All derivative terms at x (ref solver.py:146)."""
    h2 = h * h
    terms = [E.inertia(x, xhat, lay)]
    for off, dof, body in lay.soft:
        terms.append(E.elastic(body, x[off:off + dof].reshape(-1, 3), off).scaled(h2))
    terms.append(E.orthogonality(x, lay).scaled(h2))
    xw = scene.cindex.world_positions(x)
    bp = scene.barrier
    ct, mind = E.contact(xw, cand, scene.tables, scene.cindex, bp.dhat, bp.kappa, scene.ground_y)
    terms.append(ct)
    if lags is not None and lags.total:
        terms.append(E.friction(xw, xw0, lags, scene.mu, scene.eps_v, h, scene.cindex))
    terms += _constraint_terms(scene, x)
    return terms, mind


def total_value(scene, lay, x, xhat, xw0, lags, cand, h):
    """Objective value only; ∞ past intersection or inversion (ref solver.py:178)."""
    h2 = h * h
    tot = E.inertia(x, xhat, lay, derivatives=False).value
    for off, dof, body in lay.soft:
        v = E.elastic(body, x[off:off + dof].reshape(-1, 3), off, derivatives=False).value
        if not np.isfinite(v):
            return np.inf
        tot += h2 * v
    tot += h2 * E.orthogonality(x, lay, derivatives=False).value
    xw = scene.cindex.world_positions(x)
    bp = scene.barrier
    ct, _ = E.contact(xw, cand, scene.tables, scene.cindex, bp.dhat, bp.kappa, scene.ground_y,
                      derivatives=False)
    if not np.isfinite(ct.value):
        return np.inf
    tot += ct.value
    if lags is not None and lags.total:
        tot += E.friction(xw, xw0, lags, scene.mu, scene.eps_v, h, scene.cindex,
                          derivatives=False).value
    for t in _constraint_terms(scene, x):
        tot += t.value
    return tot


def combine(terms, n):
    val = 0.0
    g = np.zeros(n)
    for t in terms:
        val += t.value
        if len(t.gi):
            np.add.at(g, t.gi, t.gv)
    hr = np.concatenate([t.hr for t in terms])
    hc = np.concatenate([t.hc for t in terms])
    hv = np.concatenate([t.hv for t in terms])
    return val, g, sp.coo_matrix((hv, (hr, hc)), shape=(n, n)).tocsc()


def newton_direction(g, hmat):
    """Solve H p = −g; gradient fallback on failure or ascent (ref solver.py:241)."""
    if len(g) == 0:
        return np.zeros(0)
    try:
        p = splu(hmat).solve(-g)
    except RuntimeError:
        return -g
    if not np.all(np.isfinite(p)) or p @ g > 0.0:
        return -g
    return p


def line_search(fn, x, p, e0, alpha, halvings):
    """Backtrack from the CCD bound until E(x + αp) ≤ E0 (ref solver.py:257)."""
    for _ in range(halvings):
        if alpha < ALPHA_FLOOR:
            break
        xn = x + alpha * p
        en = fn(xn)
        if en <= e0:
            return alpha, xn, en
        alpha *= 0.5
    return 0.0, x, e0


def newton_solve(scene, lay, x0, xhat, xw0, lags, cfg, rep):
    """ref solver.py:295, including the two-small-steps stopping rule."""
    h = cfg.h
    dhat = scene.barrier.dhat
    x = x0.copy()
    gnorm = 0.0
    small_run = 0
    prev = np.inf
    for _ in range(cfg.max_newton_iters):
        xw = scene.cindex.world_positions(x)
        cand = C.broad_phase(xw, scene.tables, dhat, scene.ground_y)
        terms, mind = assemble(scene, lay, x, xhat, xw0, lags, cand, h)
        rep.min_dist_before = min(rep.min_dist_before, mind)
        e0, g, hmat = combine(terms, lay.n_dof)
        gnorm = float(np.abs(g).max()) if len(g) else 0.0
        p = newton_direction(g, hmat)
        rep.newton_iters += 1
        pn = float(np.abs(p).max()) if len(p) else 0.0
        rep.pnorms.append(pn)
        small = (pn / h <= cfg.newton_tol) if len(p) else True
        if small and small_run >= 1 and (pn <= prev or small_run >= 7):
            return x, gnorm
        small_run = small_run + 1 if small else 0
        prev = pn
        dxw = scene.cindex.world_positions(x + p) - xw
        sweep = C.broad_phase_ccd(xw, dxw, scene.tables, inflation=dhat, ground_y=scene.ground_y)
        amax = C.ccd_alpha(xw, dxw, sweep, scene.tables, scene.ground_y,
                           conservative=cfg.ccd_conservative_factor)
        rep.ccd_invocations += 1
        rep.alphas.append(amax)
        alpha, x, _ = line_search(
            lambda xt: total_value(scene, lay, xt, xhat, xw0, lags, sweep, h),
            x, p, e0, amax, cfg.max_line_search_halvings)
        if alpha == 0.0:
            rep.line_search_failed = True
            rep.converged = False
            return x, gnorm
    rep.converged = False
    return x, gnorm


def multiplier_update(c, q):
    """First-order AL step; κ doubles unless the residual halved (ref constraints.py:215)."""
    d = q - c.target
    res = float(np.linalg.norm(d))
    c.lam = c.lam - c.kappa * d / np.sqrt(c.mass_scale)
    if res > 0.5 * c.last_residual:
        c.kappa = min(2.0 * c.kappa, KAPPA_A_GROWTH_CAP * c.kappa0)
    c.last_residual = res
    return res


def adapt_kappa(scene, min_dist):
    """ref barrier.py:85."""
    bp = scene.barrier
    if min_dist < 1e-4 * bp.dhat and bp.kappa < KAPPA_GROWTH_CAP * scene.kappa0:
        bp.kappa = min(2.0 * bp.kappa, KAPPA_GROWTH_CAP * scene.kappa0)


def step(scene, cfg: Config, layout: Layout | None = None):
    """Advance one time step in place; returns a Report (ref solver.py:360)."""
    t0 = time.perf_counter()
    rep = Report()
    st = scene.state
    lay = layout or Layout(scene)
    h = cfg.h
    bp = scene.barrier
    x_prev = st.gather()
    xw0 = scene.cindex.world_positions(x_prev)
    cand0 = C.broad_phase(xw0, scene.tables, bp.dhat, scene.ground_y)
    v0, _ = E.contact(xw0, cand0, scene.tables, scene.cindex, bp.dhat, bp.kappa, scene.ground_y,
                      derivatives=False)
    if not np.isfinite(v0.value):
        raise C.IntersectionError("step started from an intersecting state")

    # predictor (ref bodies.py:292)
    xhat = x_prev + h * st.gather_velocity()
    for blk in st.blocks:
        if blk.is_affine:
            xhat[blk.offset:blk.offset + 12] += h * h * blk.body.gravity_acceleration(scene.gravity)
        else:
            xhat[blk.offset:blk.offset + blk.dof] += (h * h) * np.tile(scene.gravity,
                                                                       blk.body.n_verts)
    cons = list(scene.constraints)
    for c in cons:
        c.lam = np.zeros(12)
        c.kappa = c.kappa0
        c.last_residual = np.inf
        if c.body.target_q is not None:
            c.target = np.asarray(c.body.target_q, dtype=np.float64).copy()

    x = x_prev
    gnorm = 0.0
    for fp in range(max(cfg.friction_fixed_point_iters, 1)):
        anchor = x_prev if fp == 0 else x
        xa = scene.cindex.world_positions(anchor)
        ca = C.broad_phase(xa, scene.tables, bp.dhat, scene.ground_y)
        lags = E.friction_lags(xa, ca, scene.tables, scene.cindex, bp.dhat, bp.kappa,
                               scene.ground_y)
        if not cons:
            rep.al_outer = max(rep.al_outer, 1)
            x, gnorm = newton_solve(scene, lay, x, xhat, xw0, lags, cfg, rep)
        else:
            for outer in range(cfg.al_max_outer):
                x, gnorm = newton_solve(scene, lay, x, xhat, xw0, lags, cfg, rep)
                res = 0.0
                for c in cons:
                    off = st.offset_of(c.body)
                    res = max(res, multiplier_update(c, x[off:off + 12]))
                rep.al_outer = max(rep.al_outer, outer + 1)
                if res <= AL_TOL or rep.line_search_failed:
                    break
        if rep.line_search_failed:
            break
    rep.final_grad_norm = gnorm
    xw1 = scene.cindex.world_positions(x)
    cand1 = C.broad_phase(xw1, scene.tables, bp.dhat, scene.ground_y)
    _, md = E.contact(xw1, cand1, scene.tables, scene.cindex, bp.dhat, bp.kappa, scene.ground_y,
                      derivatives=False)
    rep.min_dist_after = md
    adapt_kappa(scene, md)
    st.scatter(x)
    st.scatter_velocity((x - x_prev) / h)
    rep.total_time = time.perf_counter() - t0
    return rep
