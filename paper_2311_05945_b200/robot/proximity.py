"""Mesh proximity queries for grasp evaluation and repair (ref
pkg/src/srsim/robot/proximity.py), computed by the CUDA library.

Same names, arguments and results as the reference: ``winding_numbers``
(:183), ``count_mesh_intersections`` (:163), ``max_penetration`` (:254),
``surface_samples`` (:232, host-side sample construction). The scene-level
``min_group_distance`` / ``min_ground_distance`` of the reference are
``GpuWorld.group_distance`` / ``ground_distance`` (batched over envs).
Batched forms (``max_penetration_batch``) take one problem per env.
No CPU fallback: every query raises when the library or device is missing.
"""

from __future__ import annotations

import numpy as np

from .. import _native as N
from ..mesh import SurfaceMesh, unique_edges


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def winding_numbers(points, verts, tris) -> np.ndarray:
    """Generalized winding number of each point w.r.t. a closed surface
    (ref proximity.py:183)."""
    lib = N.load()
    p = _f64(np.atleast_2d(points)).reshape(-1, 3)
    v, t = _f64(verts).reshape(-1, 3), _i32(tris).reshape(-1, 3)
    out = np.zeros(len(p))
    N.check(lib.ipc_winding_numbers(len(p), N.ptr(p, N._f64p), len(v), N.ptr(v, N._f64p), len(t),
                                    N.ptr(t, N._i32p), N.ptr(out, N._f64p)))
    return out


def count_mesh_intersections(verts_a, tris_a, verts_b, tris_b) -> int:
    """Number of crossing triangle pairs between two surfaces (ref proximity.py:163)."""
    lib = N.load()
    va, ta = _f64(verts_a).reshape(-1, 3), _i32(tris_a).reshape(-1, 3)
    vb, tb = _f64(verts_b).reshape(-1, 3), _i32(tris_b).reshape(-1, 3)
    c = np.zeros(1, np.int64)
    N.check(lib.ipc_count_mesh_intersections(len(va), N.ptr(va, N._f64p), len(ta),
                                             N.ptr(ta, N._i32p), len(vb), N.ptr(vb, N._f64p),
                                             len(tb), N.ptr(tb, N._i32p), N.ptr(c, N._i64p)))
    return int(c[0])


def surface_samples(verts, tris, edges=None) -> np.ndarray:
    """Vertices + edge midpoints + triangle centroids (ref proximity.py:232)."""
    tris = np.asarray(tris, dtype=np.int64)
    edges = unique_edges(tris) if edges is None else edges
    edges = np.asarray(edges, dtype=np.int64)
    mids = 0.5 * (verts[edges[:, 0]] + verts[edges[:, 1]])
    cents = verts[tris].mean(axis=1)
    return np.concatenate([verts, mids, cents])


def _prefix(sizes):
    return _i32(np.concatenate([[0], np.cumsum(sizes)]))


def max_penetration_batch(points, meshes) -> np.ndarray:
    """ref proximity.py:235 for E (points, object mesh) problems at once.

    points: list of (n_e, 3) arrays; meshes: list of (verts, tris)."""
    lib = N.load()
    E = len(points)
    if E == 0:
        return np.zeros(0)
    env_pt = _prefix([len(p) for p in points])
    env_ov = _prefix([len(m[0]) for m in meshes])
    env_ot = _prefix([len(m[1]) for m in meshes])
    pts = _f64(np.concatenate([np.reshape(p, (-1, 3)) for p in points]))
    ov = _f64(np.concatenate([m[0] for m in meshes]))
    ot = _i32(np.concatenate([np.reshape(m[1], (-1, 3)) for m in meshes]))
    out = np.zeros(E)
    N.check(lib.ipc_max_penetration(E, N.ptr(env_pt, N._i32p), N.ptr(pts, N._f64p),
                                    N.ptr(env_ov, N._i32p), N.ptr(env_ot, N._i32p),
                                    N.ptr(ov, N._f64p), N.ptr(ot, N._i32p), N.ptr(out, N._f64p)))
    return out


def max_penetration(hand_points, object_mesh: SurfaceMesh) -> float:
    """Deepest intrusion (m) of the points into a watertight mesh, 0 when no
    point is contained (ref proximity.py:235)."""
    if len(hand_points) == 0:
        return 0.0
    return float(max_penetration_batch([hand_points],
                                       [(object_mesh.vertices, object_mesh.triangles)])[0])
