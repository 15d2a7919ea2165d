"""Oracle backend for the grasp driver: force readout and proximity queries.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ref pkg/src/srsim/robot/sensing.py (slot_contact_forces :30,
finger_forces :61) and robot/proximity.py (min_group_distance :245,
min_ground_distance :286).
"""

from __future__ import annotations

import numpy as np

from . import collide as C
from . import distance as D
from . import energies as E
from . import stepper as S


class _Identity:
    """Slot index whose every slot owns three DoF (ref sensing.py:19)."""

    def __init__(self, cidx):
        n = len(cidx.is_affine)
        self.is_affine = np.zeros(n, dtype=bool)
        self.soft_dof = 3 * np.arange(n, dtype=np.int64)[:, None] + np.arange(3)
        self.body_offset = np.zeros(n, dtype=np.int64)
        self.rest = cidx.rest
        self.edge_rest_len2 = cidx.edge_rest_len2


def slot_contact_forces(scene, h, x=None):
    xw = scene.world_slots(x)
    bp = scene.barrier
    cand = C.broad_phase(xw, scene.tables, bp.dhat, scene.ground_y)
    f = np.zeros((len(xw), 3))
    if cand.total == 0:
        return f
    term, _ = E.contact(xw, cand, scene.tables, _Identity(scene.cindex), bp.dhat, bp.kappa,
                        scene.ground_y, derivatives=True)
    np.add.at(f.ravel(), term.gi, term.gv)
    return -f / (h * h)


def finger_forces(scene, gripper, h, x=None):
    sf = slot_contact_forces(scene, h, x)
    index = {id(b.body): i for i, b in enumerate(scene.state.blocks)}
    out = np.zeros(len(gripper.finger_names))
    for k, fn in enumerate(gripper.finger_names):
        tot = np.zeros(3)
        for ln in gripper.finger_groups[fn]:
            tot += sf[scene.tables.vert_body == index[id(gripper.links[ln])]].sum(axis=0)
        out[k] = np.linalg.norm(tot)
    return out


def _blocks(scene, bodies):
    want = {id(b) for b in bodies}
    return [i for i, b in enumerate(scene.state.blocks) if id(b.body) in want]


def min_group_distance(scene, a, b, x=None):
    ia, ib = _blocks(scene, a), _blocks(scene, b)
    xw = scene.world_slots(x)
    t = scene.tables
    cand = C.broad_phase(xw, t, scene.barrier.dhat, scene.ground_y)
    best = np.inf
    if len(cand.pt):
        vb, tb = t.vert_body[cand.pt[:, 0]], t.tri_body[cand.pt[:, 1]]
        keep = (np.isin(vb, ia) & np.isin(tb, ib)) | (np.isin(vb, ib) & np.isin(tb, ia))
        if keep.any():
            tri = t.tris[cand.pt[keep, 1]]
            d2, _ = D.pt_dist2(xw[cand.pt[keep, 0]], xw[tri[:, 0]], xw[tri[:, 1]], xw[tri[:, 2]])
            best = min(best, float(np.sqrt(d2.min())))
    if len(cand.ee):
        b1, b2 = t.edge_body[cand.ee[:, 0]], t.edge_body[cand.ee[:, 1]]
        keep = (np.isin(b1, ia) & np.isin(b2, ib)) | (np.isin(b1, ib) & np.isin(b2, ia))
        if keep.any():
            ea, eb = t.edges[cand.ee[keep, 0]], t.edges[cand.ee[keep, 1]]
            d2, _ = D.ee_dist2(xw[ea[:, 0]], xw[ea[:, 1]], xw[eb[:, 0]], xw[eb[:, 1]])
            best = min(best, float(np.sqrt(d2.min())))
    return best


def min_ground_distance(scene, bodies, x=None):
    if scene.ground_y is None:
        return np.inf
    idx = _blocks(scene, bodies)
    xw = scene.world_slots(x)
    m = np.isin(scene.tables.vert_body, idx)
    return float(xw[m, 1].min() - scene.ground_y) if m.any() else np.inf


class OracleBackend:
    """Backend object consumed by paper_2311_05945_b200.robot.grasp."""

    def __init__(self):
        self._layouts = {}

    def step(self, scene, cfg):
        key = id(scene)
        if key not in self._layouts:
            self._layouts[key] = S.Layout(scene)
        c = S.Config(h=cfg.h, newton_tol=cfg.newton_tol, max_newton_iters=cfg.max_newton_iters,
                     max_line_search_halvings=cfg.max_line_search_halvings,
                     ccd_conservative_factor=cfg.ccd_conservative_factor,
                     friction_fixed_point_iters=cfg.friction_fixed_point_iters,
                     al_max_outer=cfg.al_max_outer)
        return S.step(scene, c, self._layouts[key])

    finger_forces = staticmethod(finger_forces)
    min_group_distance = staticmethod(min_group_distance)
    min_ground_distance = staticmethod(min_ground_distance)
