"""Oracle: broad phase and continuous collision detection.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference answers box queries with a median-split BVH
(ref geometry/bvh.py) but finishes every leaf with an exact per-primitive
box test (ref bvh.py:118,129-130), so its output equals the exhaustive
filtered pair list. This restatement enumerates pairs exhaustively, in
blocks, with the identical floating-point box tests; results are returned
in the reference's lexicographic order (ref broadphase.py:162-166).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import distance as D

CONSERVATIVE = 0.9  # ref ccd.py:16
STOP_RATIO = 0.01   # ref ccd.py:17
MAX_ITER = 64       # ref ccd.py:18


class IntersectionError(RuntimeError):
    pass


@dataclass
class Candidates:
    pt: np.ndarray = field(default_factory=lambda: np.empty((0, 2), np.int64))
    ee: np.ndarray = field(default_factory=lambda: np.empty((0, 2), np.int64))
    ground: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))

    @property
    def total(self):
        return len(self.pt) + len(self.ee) + len(self.ground)


def _excluded_matrix(tables):
    nb = len(tables.body_is_rigid)
    ex = np.zeros((nb, nb), dtype=bool)
    for a, b in np.asarray(tables.excluded_pairs, dtype=np.int64).reshape(-1, 2):
        ex[a, b] = ex[b, a] = True
    return ex


def _overlap(qlo, qhi, plo, phi, margin):
    """Exact reference test: query box vs primitive box inflated by margin
    (ref bvh.py:87-88, :118, :129-130)."""
    pmin = plo - margin
    pmax = phi + margin
    return np.all((qlo[:, None, :] <= pmax[None]) & (qhi[:, None, :] >= pmin[None]), axis=2)


def _pairs(x_lo, x_hi, tables, margin, block=512):
    tris, edges = tables.tris, tables.edges
    # primitive boxes from both trajectory endpoints (ref broadphase.py:206-215)
    tmin, tmax = x_lo[tris].min(axis=1), x_hi[tris].max(axis=1)
    emin, emax = x_lo[edges].min(axis=1), x_hi[edges].max(axis=1)
    ex = _excluded_matrix(tables)
    rigid = tables.body_is_rigid

    pt = []
    nv = len(x_lo)
    for s in range(0, nv, block):
        v = np.arange(s, min(nv, s + block))
        hit = _overlap(x_lo[v], x_hi[v], tmin, tmax, margin)
        vi, ti = np.nonzero(hit)
        vi = v[vi]
        adj = np.any(tris[ti] == vi[:, None], axis=1)
        bv, bt = tables.vert_body[vi], tables.tri_body[ti]
        keep = ~(adj | ((bv == bt) & rigid[bv]) | ex[bv, bt])
        pt.append(np.stack([vi[keep], ti[keep]], axis=1))

    ee = []
    ne = len(edges)
    for s in range(0, ne, block):
        ei_all = np.arange(s, min(ne, s + block))
        hit = _overlap(emin[ei_all], emax[ei_all], emin, emax, margin)
        ii, jj = np.nonzero(hit)
        ei, ej = ei_all[ii], jj
        up = ei < ej
        ei, ej = ei[up], ej[up]
        a, b = edges[ei], edges[ej]
        shared = ((a[:, 0] == b[:, 0]) | (a[:, 0] == b[:, 1])
                  | (a[:, 1] == b[:, 0]) | (a[:, 1] == b[:, 1]))
        ba, bb = tables.edge_body[ei], tables.edge_body[ej]
        keep = ~(shared | ((ba == bb) & rigid[ba]) | ex[ba, bb])
        ee.append(np.stack([ei[keep], ej[keep]], axis=1))

    pt = np.concatenate(pt) if pt else np.empty((0, 2), np.int64)
    ee = np.concatenate(ee) if ee else np.empty((0, 2), np.int64)
    return pt.astype(np.int64), ee.astype(np.int64)


def _ground(y_lo, tables, margin, ground_y):
    """ref broadphase.py:142."""
    m = (y_lo < ground_y + margin) & ~tables.body_is_kinematic[tables.vert_body]
    return np.nonzero(m)[0].astype(np.int64)


def broad_phase(x, tables, inflation, ground_y=None):
    """Discrete candidates within `inflation` at x (ref broadphase.py:169)."""
    out = Candidates()
    if tables.needs_pair_search():
        out.pt, out.ee = _pairs(x, x, tables, inflation)
    if ground_y is not None:
        out.ground = _ground(x[:, 1], tables, inflation, ground_y)
    return out


def broad_phase_ccd(x, dx, tables, inflation=1e-9, ground_y=None):
    """Swept candidates over x → x + dx (ref broadphase.py:192)."""
    out = Candidates()
    xe = x + dx
    if tables.needs_pair_search():
        out.pt, out.ee = _pairs(np.minimum(x, xe), np.maximum(x, xe), tables, inflation)
    if ground_y is not None:
        out.ground = _ground(np.minimum(x[:, 1], xe[:, 1]), tables, inflation, ground_y)
    return out


# ---------------------------------------------------------------------------
# CCD: per-pair conservative advancement (ref ccd.py:34)
# ---------------------------------------------------------------------------


def _dist(px, kind):
    if kind == "pt":
        return np.sqrt(D.pt_dist2(px[:, 0], px[:, 1], px[:, 2], px[:, 3])[0])
    return np.sqrt(D.ee_dist2(px[:, 0], px[:, 1], px[:, 2], px[:, 3])[0])


def pair_ccd(px, pdx, kind, conservative=CONSERVATIVE):
    n = len(px)
    if n == 0:
        return np.ones(0)
    mean = (((pdx[:, 0] + pdx[:, 1]) + pdx[:, 2]) + pdx[:, 3]) / 4.0
    speed = np.sqrt(np.sum((pdx - mean[:, None]) ** 2, axis=2))
    if kind == "pt":
        bound = speed[:, 0] + speed[:, 1:].max(axis=1)
    else:
        bound = speed[:, :2].max(axis=1) + speed[:, 2:].max(axis=1)
    d0 = _dist(px, kind)
    if np.any(d0 <= 0):
        raise IntersectionError("CCD started from a touching or intersecting pair")
    alpha = np.ones(n)
    live = np.nonzero(bound > 1e-300)[0]
    t = np.zeros(len(live))
    d = d0[live]
    stop = STOP_RATIO * d0[live]
    for _ in range(MAX_ITER):
        if len(live) == 0:
            break
        tn = t + d / bound[live]
        keep = tn < 1.0  # crossing the whole step without contact: safe
        live, t, tn, stop = live[keep], t[keep], tn[keep], stop[keep]
        if len(live) == 0:
            break
        d = _dist(px[live] + tn[:, None, None] * pdx[live], kind)
        t = tn
        hit = d <= stop
        alpha[live[hit]] = conservative * t[hit]
        live, t, d, stop = live[~hit], t[~hit], d[~hit], stop[~hit]
    if len(live):
        alpha[live] = np.minimum(1.0, np.maximum(conservative * t, 1e-12))
    return alpha


def ground_ccd(y, dy, ground_y, conservative=CONSERVATIVE):
    """ref ccd.py:90."""
    if len(y) == 0:
        return 1.0
    if np.any(y <= ground_y):
        raise IntersectionError("CCD started with a vertex at or below the ground")
    f = dy < 0
    if not f.any():
        return 1.0
    t = (y[f] - ground_y) / -dy[f]
    t = t[t <= 1.0]
    return 1.0 if len(t) == 0 else float(min(1.0, conservative * t.min()))


def ccd_alpha(x, dx, cand, tables, ground_y=None, conservative=CONSERVATIVE):
    """Largest safe step fraction over the swept candidates (ref ccd.py:107)."""
    a = 1.0
    if len(cand.pt):
        ids = np.concatenate([cand.pt[:, :1], tables.tris[cand.pt[:, 1]]], axis=1)
        a = min(a, pair_ccd(x[ids], dx[ids], "pt", conservative).min())
    if len(cand.ee):
        ids = np.concatenate([tables.edges[cand.ee[:, 0]], tables.edges[cand.ee[:, 1]]], axis=1)
        a = min(a, pair_ccd(x[ids], dx[ids], "ee", conservative).min())
    if ground_y is not None and len(cand.ground):
        g = cand.ground
        a = min(a, ground_ccd(x[g, 1], dx[g, 1], ground_y, conservative))
    return float(a)
