"""Penetrated-grasp repair: open, retract, re-grasp under spring targets
(ref pkg/src/srsim/robot/repair.py).

Same names, arguments and results as the reference: ``repair_grasp`` (:82),
``RepairResult`` (:40), ``RETRACT_STEP`` / ``RETRACT_MAX`` (:36-37). The
geometric half (the retraction probe loop, ref :98-113, with the overlap test
of :49) runs on the GPU as one ``ipc_repair_retract`` call that evaluates
every crossing-pair and containment test of a window of probes at once; the
dynamic half is AutoGrasp on the GPU step engine. ``repair_batch`` repairs E
grasps together (config 4): one retraction launch for all envs, one
``BatchGrasp`` world for the cleared ones, one batched penetration query.

No CPU fallback: with the library or device missing every call raises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import _native as N
from .grasp import GraspConfig, GraspOutcome, GraspPhase, GraspTrial, autograsp, build_grasp_scene
from .proximity import max_penetration_batch, surface_samples

RETRACT_STEP = 1e-3  # m per probe (ref repair.py:36)
RETRACT_MAX = 0.5    # m; beyond this the grasp is unsalvageable (ref :37)


@dataclass
class RepairResult:
    """ref repair.py:40"""
    trial: GraspTrial
    cleared: bool  # retraction found an intersection-free placement
    retraction_m: float
    penetration_before_m: float
    penetration_after_m: float


def retraction_schedule():
    """Probe distances the reference visits — retraction accumulated by
    repeated ``+= RETRACT_STEP`` while ``<= RETRACT_MAX`` (ref :103-113) —
    and the distance it reports when no probe clears."""
    out, r = [], 0.0
    while r <= RETRACT_MAX:
        out.append(r)
        r += RETRACT_STEP
    return np.array(out), r


def _world_mesh(obj):
    """(world vertices, triangles) of the object (ref repair.py:65)."""
    from ..bodies import SoftBody

    if isinstance(obj, SoftBody):
        return obj.x.copy(), np.asarray(obj.mesh.surface.triangles)
    return obj.world_vertices(), np.asarray(obj.mesh.triangles)


def _hand_points(gripper) -> np.ndarray:
    """ref repair.py:73"""
    return np.concatenate([surface_samples(b.world_vertices(), b.mesh.triangles, b.mesh.edges)
                           for b in gripper.bodies()])


def _hand_points_batch(g0, link_q) -> np.ndarray:
    """_hand_points of E placements of one gripper model at once: link_q maps
    link name -> (E, 12) affine DoFs. Same operations as world_vertices() +
    surface_samples() per env, stacked (bit-identical). Returns (E, P, 3)."""
    out = []
    for ln in sorted(g0.links):
        b = g0.links[ln]
        q = np.asarray(link_q[ln], dtype=np.float64)
        a = q[:, 3:].reshape(-1, 3, 3)
        v = b.mesh.vertices[None] @ np.transpose(a, (0, 2, 1)) + q[:, None, :3]
        e = np.asarray(b.mesh.edges, dtype=np.int64)
        t = np.asarray(b.mesh.triangles, dtype=np.int64)
        out += [v, 0.5 * (v[:, e[:, 0]] + v[:, e[:, 1]]), v[:, t].mean(axis=2)]
    return np.concatenate(out, axis=1)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class RetractBatch:
    """Persistent retraction batch: E grasps of one gripper model on fixed
    objects. The object meshes and the hand topology (triangles, per-link
    ranges) are packed once; run(poses, opened) evaluates the batched FK,
    the hand's world vertices and the palm normals and launches the probe
    search (ipc_repair_retract, every array uploaded per call). Same arrays,
    bit for bit, as retract_batch packs for a shared-model batch."""

    def __init__(self, gripper, obj_meshes):
        self.g0 = gripper
        self.E = E = len(obj_meshes)
        self.sched, self.end = retraction_schedule()
        g0 = gripper
        self.names = names = sorted(g0.links)  # == Gripper.bodies() order
        nv = [len(g0.links[ln].mesh.vertices) for ln in names]
        nt = [len(g0.links[ln].mesh.triangles) for ln in names]
        vo = np.concatenate([[0], np.cumsum(nv)[:-1]])
        tri_one = np.concatenate([np.asarray(g0.links[ln].mesh.triangles, dtype=np.int32) + o
                                  for ln, o in zip(names, vo)]).astype(np.int32)
        per_env = int(np.sum(nv))
        L = len(names)
        self.lo = np.array([jt.lower for jt in g0.joints])
        self.hi = np.array([jt.upper for jt in g0.joints])
        self.rest = [g0.links[ln].mesh.vertices[None] for ln in names]
        self.arrs = dict(
            env_link=_i32(np.arange(E + 1) * L),
            link_vert=_i32(np.concatenate([[0], np.cumsum(np.tile(nv, E))])),
            link_tri=_i32(np.concatenate([[0], np.cumsum(np.tile(nt, E))])),
            hand_t=_i32((tri_one[None] + (per_env * np.arange(E, dtype=np.int32))[:, None, None]).reshape(-1, 3)),
            obj_v=_f64(np.concatenate([m[0] for m in obj_meshes])) if E else _f64(np.zeros((0, 3))),
            obj_t=_i32(np.concatenate([m[1] for m in obj_meshes]).reshape(-1, 3)) if E else _i32(np.zeros((0, 3))),
            env_ov=_i32(np.concatenate([[0], np.cumsum([len(m[0]) for m in obj_meshes])])),
            env_ot=_i32(np.concatenate([[0], np.cumsum([np.size(m[1]) // 3 for m in obj_meshes])])),
            retr=_f64(self.sched))

    def hand_world(self, poses, opened):
        """World vertices of every link of every env, (E * per_env, 3)."""
        from .batch import batch_fk

        fk = batch_fk(self.g0, np.asarray(poses, dtype=np.float64),
                      np.clip(np.asarray(opened, dtype=np.float64), self.lo, self.hi))
        per = []
        for ln, x0 in zip(self.names, self.rest):
            t = fk[ln]
            a = t[:, :3, :3].reshape(-1, 9).reshape(-1, 3, 3)
            per.append(x0 @ np.transpose(a, (0, 2, 1)) + t[:, None, :3, 3])
        return np.concatenate(per, axis=1).reshape(-1, 3)

    def run(self, poses, opened):
        """(cleared bool[E], retraction_m float[E], probe_index int[E])"""
        lib = N.load()
        E = self.E
        if E == 0:
            return np.zeros(0, bool), np.zeros(0), np.zeros(0, np.int32)
        a = self.arrs
        hv = _f64(self.hand_world(poses, opened))
        normal = _f64(np.asarray(poses, dtype=np.float64)[:, :3, :3] @ self.g0.palm_normal_local)
        d = N.RepairDesc(E, N.ptr(a["env_link"], N._i32p), N.ptr(a["link_vert"], N._i32p),
                         N.ptr(a["link_tri"], N._i32p), N.ptr(hv, N._f64p),
                         N.ptr(a["hand_t"], N._i32p), N.ptr(a["env_ov"], N._i32p),
                         N.ptr(a["env_ot"], N._i32p), N.ptr(a["obj_v"], N._f64p),
                         N.ptr(a["obj_t"], N._i32p), N.ptr(normal, N._f64p),
                         len(self.sched), N.ptr(a["retr"], N._f64p))
        idx = np.zeros(E, np.int32)
        N.check(lib.ipc_repair_retract(N.C.byref(d), N.ptr(idx, N._i32p)))
        cleared = idx < len(self.sched)
        retraction = np.where(cleared, self.sched[np.minimum(idx, len(self.sched) - 1)], self.end)
        return cleared, retraction, idx


def retract_batch(grippers, poses, opened, obj_meshes):
    """The probe loop of ref repair.py:98-113 for E envs in one launch.

    grippers: E Gripper instances (when they do not share one URDF model
    they are placed at each env's probe-0 pose and left there); poses
    (E,4,4); opened (E,J) already clamped to the joint limits;
    obj_meshes: E (world verts, tris). Returns (cleared bool[E],
    retraction_m float[E], probe_index int[E]); retraction_m is the
    reference's accumulated distance (the past-the-cap value when no probe
    clears)."""
    lib = N.load()
    E = len(grippers)
    sched, end = retraction_schedule()
    if E == 0:
        return np.zeros(0, bool), np.zeros(0), np.zeros(0, np.int32)
    env_link, link_vert, link_tri = [0], [0], [0]
    hv, ht = [], []
    g0 = grippers[0]
    if all(g.model is g0.model for g in grippers):
        # one model: vectorized FK over the batch (batch_fk) and per-link
        # world vertices x0 @ Aᵀ + p — bit-identical to place() +
        # world_vertices(); the grippers are left untouched
        from .batch import batch_fk

        lo = np.array([j.lower for j in g0.joints])
        hi = np.array([j.upper for j in g0.joints])
        fk = batch_fk(g0, np.asarray(poses, dtype=np.float64),
                      np.clip(np.asarray(opened, dtype=np.float64), lo, hi))
        names = sorted(g0.links)  # == Gripper.bodies() order
        per = []
        for ln in names:
            t = fk[ln]
            a = t[:, :3, :3].reshape(-1, 9).reshape(-1, 3, 3)
            per.append(g0.links[ln].mesh.vertices[None] @ np.transpose(a, (0, 2, 1))
                       + t[:, None, :3, 3])
        hv = np.concatenate(per, axis=1).reshape(-1, 3)
        nv = [len(g0.links[ln].mesh.vertices) for ln in names]
        nt = [len(g0.links[ln].mesh.triangles) for ln in names]
        vo = np.concatenate([[0], np.cumsum(nv)[:-1]])
        tri_one = np.concatenate([np.asarray(g0.links[ln].mesh.triangles, dtype=np.int32) + o
                                  for ln, o in zip(names, vo)]).astype(np.int32)
        per_env = int(np.sum(nv))
        ht = (tri_one[None] + (per_env * np.arange(E, dtype=np.int32))[:, None, None]).reshape(-1, 3)
        L = len(names)
        link_vert = np.concatenate([[0], np.cumsum(np.tile(nv, E))])
        link_tri = np.concatenate([[0], np.cumsum(np.tile(nt, E))])
        env_link = np.arange(E + 1) * L
    else:
        for g, p, q in zip(grippers, poses, opened):
            g.place(p, q)
            for b in g.bodies():
                v = b.world_vertices()
                ht.append(np.asarray(b.mesh.triangles, dtype=np.int64) + link_vert[-1])
                hv.append(v)
                link_vert.append(link_vert[-1] + len(v))
                link_tri.append(link_tri[-1] + len(b.mesh.triangles))
            env_link.append(len(link_vert) - 1)
        hv, ht = np.concatenate(hv), np.concatenate(ht)
    if len({g.palm_normal_local.tobytes() for g in grippers}) == 1:
        normals = np.asarray(poses, dtype=np.float64)[:, :3, :3] @ g0.palm_normal_local
    else:
        normals = [g.palm_normal(p) for g, p in zip(grippers, poses)]
    ov = _f64(np.concatenate([m[0] for m in obj_meshes]))
    ot = np.concatenate([m[1] for m in obj_meshes]).reshape(-1, 3)
    nov = np.fromiter((len(m[0]) for m in obj_meshes), dtype=np.int64, count=E)
    env_ov = _i32(np.concatenate([[0], np.cumsum(nov)]))
    env_ot = _i32(np.concatenate([[0], np.cumsum(np.fromiter(
        (np.size(m[1]) // 3 for m in obj_meshes), dtype=np.int64, count=E))]))
    ot = _i32(ot)
    arrs = dict(env_link=_i32(env_link), link_vert=_i32(link_vert), link_tri=_i32(link_tri),
                hand_v=_f64(hv), hand_t=_i32(ht),
                env_ov=env_ov, env_ot=env_ot, obj_v=ov, obj_t=ot,
                normal=_f64(np.array(normals)), retr=_f64(sched))
    d = N.RepairDesc(E, N.ptr(arrs["env_link"], N._i32p), N.ptr(arrs["link_vert"], N._i32p),
                     N.ptr(arrs["link_tri"], N._i32p), N.ptr(arrs["hand_v"], N._f64p),
                     N.ptr(arrs["hand_t"], N._i32p), N.ptr(arrs["env_ov"], N._i32p),
                     N.ptr(arrs["env_ot"], N._i32p), N.ptr(arrs["obj_v"], N._f64p),
                     N.ptr(arrs["obj_t"], N._i32p), N.ptr(arrs["normal"], N._f64p),
                     len(sched), N.ptr(arrs["retr"], N._f64p))
    idx = np.zeros(E, np.int32)
    N.check(lib.ipc_repair_retract(N.C.byref(d), N.ptr(idx, N._i32p)))
    cleared = idx < len(sched)
    retraction = np.where(cleared, sched[np.minimum(idx, len(sched) - 1)], end)
    return cleared, retraction, idx


def clone_grippers(model, n: int, density: float = 2000.0):
    """n independent Gripper instances of one URDF model. The first is built
    normally; the rest are deep copies that share the model, the link
    meshes and the (read-only) mass properties — ~5x cheaper than building
    each Gripper (which integrates every link's mass matrix again)."""
    import copy

    from .gripper import Gripper

    if n <= 0:
        return []
    g0 = Gripper(model, density=density)
    shared = [model, *model.actuated()]
    for b in g0.links.values():
        shared += [b.mesh, b.M_b, b.first_moment]
    out = [g0]
    for _ in range(n - 1):
        out.append(copy.deepcopy(g0, {id(o): o for o in shared}))
    return out


def _probe_pose(pose, gripper, r):
    probe = np.array(pose, dtype=np.float64)
    probe[:3, 3] -= r * gripper.palm_normal(pose)
    return probe


def repair_grasp(obj, gripper, pose, joint_values, open_offset: float = 0.01,
                 grasp_cfg: GraspConfig = None, solver_cfg=None, backend=None,
                 **scene_kwargs) -> RepairResult:
    """Clear interpenetration, then AutoGrasp with springs to the input pose
    (ref repair.py:82)."""
    from ..solver import SolverConfig

    gc = grasp_cfg or GraspConfig()
    sc = solver_cfg or SolverConfig()
    pose = np.asarray(pose, dtype=np.float64)
    joint_values = np.asarray(joint_values, dtype=np.float64)
    trial = GraspTrial(pose.copy(), joint_values.copy())
    ov, ot = _world_mesh(obj)

    gripper.place(pose, joint_values)
    pen_before = float(max_penetration_batch([_hand_points(gripper)], [(ov, ot)])[0])

    opened = gripper.clamp_joints(joint_values - open_offset)
    cleared, retraction, _ = retract_batch([gripper], [pose], [opened], [(ov, ot)])
    cleared, retraction = bool(cleared[0]), float(retraction[0])
    trial.retraction_m = retraction
    if not cleared:
        trial.outcome = GraspOutcome.ABORTED
        trial.advance(GraspPhase.DONE)
        return RepairResult(trial, False, retraction, pen_before, pen_before)

    probe = _probe_pose(pose, gripper, retraction)
    gripper.place(probe, opened)
    scene = build_grasp_scene(obj, gripper, probe, opened, h=sc.h, **scene_kwargs)
    gripper.set_targets(pose=pose)
    autograsp(scene, gripper, trial, gc, sc, backend)

    pv, pt = _world_mesh(obj)
    pen_after = float(max_penetration_batch([_hand_points(gripper)], [(pv, pt)])[0])
    trial.penetration_m = pen_after
    if trial.outcome is None:
        trial.outcome = GraspOutcome.SUCCESS
        trial.advance(GraspPhase.DONE)
    return RepairResult(trial, True, retraction, pen_before, pen_after)


def repair_batch(model, objects, poses, joint_values, open_offset: float = 0.01,
                 grasp_cfg: GraspConfig = None, solver_cfg=None, density: float = 2000.0,
                 max_ticks: int = 100_000, **scene_kwargs):
    """``repair_grasp`` for E grasps at once (config 4). Returns E RepairResults.

    Geometry: one retraction launch for every env; dynamics: the cleared envs
    share one BatchGrasp world running AutoGrasp only, with link targets at
    the input poses; penetration before/after: one batched query each."""
    from .batch import BatchGrasp, batch_fk

    E = len(objects)
    poses = np.asarray(poses, dtype=np.float64).reshape(E, 4, 4)
    joint_values = np.asarray(joint_values, dtype=np.float64).reshape(E, -1)
    grippers = clone_grippers(model, E, density)
    meshes = [_world_mesh(o) for o in objects]
    # penetration before: hand samples at the input placements (vectorized FK)
    g0 = grippers[0]
    lo = np.array([j.lower for j in g0.joints])
    hi = np.array([j.upper for j in g0.joints])
    fk = batch_fk(g0, poses, np.clip(joint_values, lo, hi))
    q0 = {ln: np.concatenate([fk[ln][:, :3, 3], fk[ln][:, :3, :3].reshape(-1, 9)], axis=1)
          for ln in g0.links}
    pen_before = max_penetration_batch(list(_hand_points_batch(g0, q0)), meshes)
    opened = np.array([g.clamp_joints(q - open_offset) for g, q in zip(grippers, joint_values)])
    cleared, retraction, _ = retract_batch(grippers, poses, opened, meshes)

    trials = [GraspTrial(p.copy(), q.copy()) for p, q in zip(poses, joint_values)]
    results = [None] * E
    for e in np.nonzero(~cleared)[0]:
        t = trials[e]
        t.retraction_m = float(retraction[e])
        t.outcome = GraspOutcome.ABORTED
        t.advance(GraspPhase.DONE)
        results[e] = RepairResult(t, False, float(retraction[e]), float(pen_before[e]),
                                  float(pen_before[e]))
    live = np.nonzero(cleared)[0]
    if len(live) == 0:
        return results
    probes = np.array([_probe_pose(poses[e], grippers[e], retraction[e]) for e in live])
    bg = BatchGrasp(model, [objects[e] for e in live], probes, opened[live],
                    grasp_cfg=grasp_cfg, solver_cfg=solver_cfg,
                    grippers=[grippers[e] for e in live], target_poses=poses[live],
                    autograsp_only=True, **scene_kwargs)
    bg.run(max_ticks)
    bg.sync_scenes()
    qa = {ln: np.array([grippers[e].links[ln].q for e in live]) for ln in g0.links}
    pen_after = max_penetration_batch(list(_hand_points_batch(g0, qa)),
                                      [_world_mesh(objects[e]) for e in live])
    for i, e in enumerate(live):
        t = trials[e]
        t.retraction_m = float(retraction[e])
        t.advance(GraspPhase.AUTOGRASP)
        t.forces = bg.forces[i]
        t.increments = bg.increments[i]
        t.steps = int(bg.steps[i])
        t.penetration_m = float(pen_after[i])
        t.outcome = bg.outcome[i] if bg.outcome[i] is not None else GraspOutcome.SUCCESS
        t.advance(GraspPhase.DONE)
        results[e] = RepairResult(t, True, float(retraction[e]), float(pen_before[e]),
                                  float(pen_after[i]))
    return results
