"""Oracle for the penetrated-grasp repair geometry — TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

Restates ref pkg/src/srsim/robot/proximity.py (segment/triangle hits :110,
triangle_pairs_intersect :146, count_mesh_intersections :163, winding_numbers
:183, surface_distance :214, surface_samples :232, max_penetration :254) and
the geometric half of ref robot/repair.py (overlap test :49, retraction
probe loop :98-113).

The BVH the reference uses to pair triangles (ref geometry/bvh.py:100) is
documented to return exactly the O(n^2) closed-box overlap filter with
margin 0, so the restatement uses that filter directly.
"""

from __future__ import annotations

import numpy as np

from . import distance as D

RETRACT_STEP = 1e-3  # ref repair.py:36
RETRACT_MAX = 0.5    # ref repair.py:37


def _dot(a, b):
    return np.einsum("ij,ij->i", a, b)


def segment_triangle_hits(orig, vec, t0, t1, t2):
    """Möller–Trumbore restricted to the segment parameter [0, 1]
    (ref proximity.py:110-125)."""
    eps = 1e-14
    e1, e2 = t1 - t0, t2 - t0
    p = np.cross(vec, e2)
    det = _dot(e1, p)
    ok = np.abs(det) > eps
    inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
    s = orig - t0
    u = _dot(s, p) * inv
    q = np.cross(s, e1)
    v = _dot(vec, q) * inv
    t = _dot(e2, q) * inv
    return ok & (u >= 0) & (v >= 0) & (u + v <= 1) & (t >= 0) & (t <= 1)


def triangle_pairs_intersect(va, ta, vb, tb):
    """Per row: does an edge of one triangle pass through the other
    (ref proximity.py:146-160)."""
    a, b = va[ta], vb[tb]
    hits = np.zeros(len(ta), dtype=bool)
    for i, j in ((0, 1), (1, 2), (2, 0)):
        hits |= segment_triangle_hits(a[:, i], a[:, j] - a[:, i], b[:, 0], b[:, 1], b[:, 2])
        hits |= segment_triangle_hits(b[:, i], b[:, j] - b[:, i], a[:, 0], a[:, 1], a[:, 2])
    return hits


def box_pairs(va, ta, vb, tb):
    """All (i, j) with closed-box overlap, lexicographic (== ref Bvh.query
    with margin 0, bvh.py:100-140)."""
    amin, amax = va[ta].min(axis=1), va[ta].max(axis=1)
    bmin, bmax = vb[tb].min(axis=1), vb[tb].max(axis=1)
    ok = ((amin[:, None, :] <= bmax[None]) & (amax[:, None, :] >= bmin[None])).all(axis=2)
    return np.nonzero(ok)


def count_mesh_intersections(va, ta, vb, tb) -> int:
    """Crossing triangle pairs between two surfaces (ref proximity.py:163)."""
    ta = np.asarray(ta, dtype=np.int64)
    tb = np.asarray(tb, dtype=np.int64)
    if len(ta) == 0 or len(tb) == 0:
        return 0
    qa, pb = box_pairs(va, ta, vb, tb)
    if len(qa) == 0:
        return 0
    return int(triangle_pairs_intersect(va, ta[qa], vb, tb[pb]).sum())


def winding_numbers(points, verts, tris):
    """Generalized winding number (van Oosterom–Strackee solid angles,
    ref proximity.py:183-211)."""
    points = np.atleast_2d(points)
    tris = np.asarray(tris, dtype=np.int64)
    a = verts[tris[:, 0]][None] - points[:, None]
    b = verts[tris[:, 1]][None] - points[:, None]
    c = verts[tris[:, 2]][None] - points[:, None]
    la, lb, lc = (np.linalg.norm(z, axis=2) for z in (a, b, c))
    num = np.einsum("ptk,ptk->pt", a, np.cross(b, c))
    den = (la * lb * lc + np.einsum("ptk,ptk->pt", a, b) * lc
           + np.einsum("ptk,ptk->pt", b, c) * la + np.einsum("ptk,ptk->pt", c, a) * lb)
    return np.arctan2(num, den).sum(axis=1) / (2.0 * np.pi)


def surface_distance(points, verts, tris):
    """Unsigned point-to-surface distance (ref proximity.py:214-229)."""
    points = np.atleast_2d(points)
    tris = np.asarray(tris, dtype=np.int64)
    n, m = len(points), len(tris)
    p = np.repeat(points, m, axis=0)
    t0, t1, t2 = (np.tile(verts[tris[:, k]], (n, 1)) for k in range(3))
    d2, _ = D.pt_dist2(p, t0, t1, t2)
    return np.sqrt(d2.reshape(n, m).min(axis=1))


def unique_edges(tris):
    t = np.asarray(tris, dtype=np.int64)
    raw = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]], axis=0)
    raw.sort(axis=1)
    return np.unique(raw, axis=0)


def surface_samples(verts, tris, edges=None):
    """Vertices + edge midpoints + triangle centroids (ref proximity.py:232)."""
    tris = np.asarray(tris, dtype=np.int64)
    edges = unique_edges(tris) if edges is None else np.asarray(edges, dtype=np.int64)
    mids = 0.5 * (verts[edges[:, 0]] + verts[edges[:, 1]])
    cents = verts[tris].mean(axis=1)
    return np.concatenate([verts, mids, cents])


def max_penetration(points, verts, tris) -> float:
    """Deepest contained point's surface distance, 0 if none contained
    (ref proximity.py:235-246)."""
    if len(points) == 0:
        return 0.0
    inside = winding_numbers(points, verts, tris) > 0.5
    if not inside.any():
        return 0.0
    return float(surface_distance(points[inside], verts, tris).max())


def hand_object_overlap(hand, ov, ot) -> bool:
    """ref repair.py:49-62. hand: [(world verts, tris)] per link body."""
    for hv, ht in hand:
        if count_mesh_intersections(hv, ht, ov, ot):
            return True
        if (winding_numbers(hv, ov, ot) > 0.5).any():
            return True
        if (winding_numbers(ov[:1], hv, ht) > 0.5).any():
            return True
    return False


def retraction_schedule():
    """The probe distances the reference visits: retraction accumulated by
    repeated += RETRACT_STEP while <= RETRACT_MAX (ref repair.py:103-113)."""
    out, r = [], 0.0
    while r <= RETRACT_MAX:
        out.append(r)
        r += RETRACT_STEP
    return np.array(out), r


def retract(gripper, pose, opened, ov, ot):
    """The probe loop of ref repair.py:103-113 through the gripper's FK at
    every probe. Returns (cleared, retraction_m, probe_index)."""
    normal = gripper.palm_normal(pose)
    retraction, k = 0.0, 0
    while retraction <= RETRACT_MAX:
        probe = np.array(pose, dtype=np.float64)
        probe[:3, 3] -= retraction * normal
        gripper.place(probe, opened)
        hand = [(b.world_vertices(), np.asarray(b.mesh.triangles, dtype=np.int64))
                for b in gripper.bodies()]
        if not hand_object_overlap(hand, ov, ot):
            return True, retraction, k
        retraction += RETRACT_STEP
        k += 1
    return False, retraction, k
