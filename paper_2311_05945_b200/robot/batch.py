"""Batched grasp evaluation: E independent gripper+object environments stepped
together on one GPU (parallel grasp generation, paper §V.A; the reference
runs one trial per worker process: pkg/src/srsim/batch.py:39).

Each environment runs the reference's per-trial program (robot/grasp.py:224
autograsp, :372 lift_and_shake) — same control law, phase schedule and
success test — but all environments advance in lock-step. One control
tick: score / sense / decide for every env with one device call each,
update all joint and pose targets with vectorized forward kinematics, and
advance every unfinished scene with one ``ipc_world_step``; finished envs
are masked out of the step.
"""

from __future__ import annotations

import math

import numpy as np

from ..solver import _scatter_velocity
from ..world import GpuWorld
from .grasp import GraspConfig, GraspOutcome, build_grasp_scene
from .gripper import Gripper, _rodrigues

AUTO, LIFT_CHECK, LIFT, SHAKE, SETTLE, SCORE, DONE = range(7)
PHASE_NAMES = ("AutoGrasp", "LiftCheck", "Lift", "Shake", "Settle", "Score", "Done")


def phi_vec(f, k=20.0, f_star=0.5):
    """Vectorized Eq. 12 (ref grasp.py:69)."""
    f = np.asarray(f, dtype=np.float64)
    if np.any(f < 0):
        raise ValueError("contact force magnitude cannot be negative")
    out = (np.exp(-k * f) - math.exp(-k * f_star)) / (1.0 - math.exp(-k * f_star))
    return np.where(f >= f_star, 0.0, out)


def batch_fk(gripper: Gripper, poses, joints):
    """World 4x4 per link for E commanded states (ref gripper.py:116): {link: (E,4,4)}."""
    model = gripper.model
    E = len(poses)
    jidx = {n: i for i, n in enumerate(gripper.joint_names)}
    out = {model.root: np.asarray(poses, dtype=np.float64)}
    todo = [model.root]
    while todo:
        par = todo.pop()
        for j in model.children_of(par):
            t = out[par] @ j.origin
            if j.type != "fixed":
                mo = np.broadcast_to(np.eye(4), (E, 4, 4)).copy()
                if j.type == "prismatic":
                    mo[:, :3, 3] = j.axis[None, :] * joints[:, jidx[j.name]][:, None]
                else:  # Rodrigues for all E angles at once (= _rodrigues per env)
                    a = np.asarray(j.axis, dtype=np.float64)
                    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
                    th = joints[:, jidx[j.name]]
                    # scalar sin/cos per angle, as ref gripper.py:38 evaluates them
                    # (numpy's vectorized loops may round differently)
                    sn = np.array([np.sin(t) for t in th])
                    cs = np.array([np.cos(t) for t in th])
                    mo[:, :3, :3] = (np.eye(3)[None] + sn[:, None, None] * k[None]
                                     + (1 - cs)[:, None, None] * (k @ k)[None])
                t = t @ mo
            out[j.child] = t
            todo.append(j.child)
    return out


class BatchGrasp:
    """E grasp trials in one device world.

    objects: E object bodies (AffineBody or SoftBody); poses (E,4,4) initial
    gripper poses; joints (E,J) initial joint values. One Gripper instance per
    env is built from the URDF `model`.
    """

    def __init__(self, model, objects, poses, joints, grasp_cfg=None, solver_cfg=None,
                 density=2000.0, grippers=None, target_poses=None, autograsp_only=False,
                 **scene_kwargs):
        from ..solver import SolverConfig

        self.gc = grasp_cfg or GraspConfig()
        self.sc = solver_cfg or SolverConfig()
        self.E = E = len(objects)
        self.objects = list(objects)
        self.grippers = (list(grippers) if grippers is not None
                         else [Gripper(model, density=density) for _ in range(E)])
        # autograsp_only: stop after AutoGrasp (ref repair.py:129 runs only
        # that phase); envs that reach the stop force finish with no outcome
        self.autograsp_only = autograsp_only
        g0 = self.grippers[0]
        self.joint_names, self.finger_names = g0.joint_names, g0.finger_names
        self.lo = np.array([j.lower for j in g0.joints])
        self.hi = np.array([j.upper for j in g0.joints])
        mus = scene_kwargs.pop("mu", 0.4)
        mus = list(mus) if np.ndim(mus) else [mus] * E
        self.scenes = [build_grasp_scene(o, g, p, q, h=self.sc.h, mu=m, **scene_kwargs)
                       for o, g, p, q, m in zip(self.objects, self.grippers, poses, joints, mus)]
        self.world = w = GpuWorld(self.scenes)
        self.links = sorted(g0.links)  # == order of Gripper.constraints()
        self.pose = np.array([g.pose for g in self.grippers])
        if target_poses is not None:
            # scenes start at `poses`, targets command `target_poses`
            # (ref repair.py:126 gripper.set_targets(pose=pose))
            self.pose = np.array(target_poses, dtype=np.float64)
            for g, tp in zip(self.grippers, self.pose):
                g.set_targets(pose=tp)
        self.q = np.array([g.joint_values for g in self.grippers])
        self.base = self.pose.copy()
        self.lifted = self.pose.copy()
        self.phase = np.full(E, AUTO)
        self.k = np.zeros(E, dtype=np.int64)
        self.frames = np.zeros(E, dtype=np.int64)
        self.steps = np.zeros(E, dtype=np.int64)
        self.outcome = [None] * E
        self.forces = [[] for _ in range(E)]
        self.increments = [[] for _ in range(E)]
        self.finger_masks = np.array(
            [[w.mask(e, [g.links[ln] for ln in g.finger_groups[fn]]) for fn in self.finger_names]
             for e, g in enumerate(self.grippers)], dtype=np.uint64)
        self.hand_mask = np.array([w.mask(e, g.bodies()) for e, g in enumerate(self.grippers)],
                                  dtype=np.uint64)
        self.obj_mask = np.array([w.mask(e, [o]) for e, o in enumerate(self.objects)],
                                 dtype=np.uint64)
        self.dhat = np.array([s.barrier.dhat for s in self.scenes])
        self.n_shake = int(round(self.gc.shake_cycles / self.gc.shake_hz / self.sc.h))
        self.targets = self.targets_for(self.pose, self.q)
        self.last_reports = None

    def targets_for(self, pose, q):
        fk = batch_fk(self.grippers[0], pose, q)
        per = [np.concatenate([fk[ln][:, :3, 3], fk[ln][:, :3, :3].reshape(-1, 9)], axis=1)
               for ln in self.links]
        return np.ascontiguousarray(np.stack(per, axis=1).reshape(-1))

    def finger_forces(self):
        return np.linalg.norm(self.world.group_forces(self.sc.h, self.finger_masks), axis=2)

    def _finish(self, mask, outcome):
        for e in np.nonzero(mask)[0]:
            self.outcome[e] = outcome
        self.phase[mask] = DONE

    def tick(self) -> bool:
        gc = self.gc
        ph = self.phase
        # 1. score envs whose settle schedule ended (ref grasp.py:213-219)
        sc = ph == SCORE
        if sc.any():
            held = self.world.group_distance(self.hand_mask, self.obj_mask) < self.dhat
            clear = self.world.ground_distance(self.obj_mask) > self.dhat
            ok = sc & held & clear
            self._finish(ok, GraspOutcome.SUCCESS)
            self._finish(sc & ~ok, GraspOutcome.DROPPED)
        # 2. AutoGrasp: read forces, stop, abort, or close (ref grasp.py:151-166)
        auto = ph == AUTO
        stepping = np.zeros(self.E, dtype=bool)
        if auto.any():
            f = self.finger_forces()
            for e in np.nonzero(auto)[0]:
                self.forces[e].append(f[e].copy())
            reached = auto & np.all(f >= gc.stop_force, axis=1)
            self._finish(auto & ~reached & (self.frames >= gc.budget), GraspOutcome.ABORTED)
            if self.autograsp_only:
                ph[reached] = DONE
            else:
                ph[reached] = LIFT_CHECK
            close = (ph == AUTO)
            if close.any():
                inc = gc.close_rate * phi_vec(f, gc.phi_k, gc.phi_f_star)
                fi = {n: i for i, n in enumerate(self.finger_names)}
                dq = np.stack([inc[:, fi[n]] if n in fi else np.zeros(self.E)
                               for n in self.joint_names], axis=1)
                self.q[close] = np.clip(self.q[close] + dq[close], self.lo, self.hi)
                for e in np.nonzero(close)[0]:
                    self.increments[e].append(inc[e].copy())
                self.frames[close] += 1
                stepping |= close
        # 3. held-before-lift test (ref grasp.py:184-190)
        lc = ph == LIFT_CHECK
        if lc.any():
            d = self.world.group_distance(self.hand_mask, self.obj_mask)
            never = lc & ~(d < self.dhat)
            self._finish(never, GraspOutcome.NEVER_HELD)
            go = lc & ~never
            ph[go] = LIFT
            self.k[go] = 0
            self.base[go] = self.pose[go]
        # 4. kinematic schedules (ref grasp.py:195-215)
        nxt = ph.copy()
        for e in np.nonzero(ph == LIFT)[0]:
            self.k[e] += 1
            self.pose[e] = self.base[e]
            self.pose[e, 1, 3] += gc.lift_height * self.k[e] / gc.lift_steps
            if self.k[e] == gc.lift_steps:
                self.lifted[e] = self.pose[e]
                nxt[e], self.k[e] = SHAKE, 0
        for e in np.nonzero(ph == SHAKE)[0]:
            self.k[e] += 1
            self.pose[e] = self.lifted[e]
            t = self.k[e] * self.sc.h  # ref robot/grasp.py:205-209 evaluates t first
            self.pose[e, 0, 3] += gc.shake_amplitude * math.sin(2.0 * math.pi * gc.shake_hz * t)
            if self.k[e] == self.n_shake:
                nxt[e], self.k[e] = SETTLE, 0
        for e in np.nonzero(ph == SETTLE)[0]:
            self.k[e] += 1
            self.pose[e] = self.lifted[e]
            if self.k[e] == gc.settle_steps:
                nxt[e] = SCORE
        stepping |= (ph == LIFT) | (ph == SHAKE) | (ph == SETTLE)
        if not stepping.any():
            self.phase = nxt
            return bool((self.phase != DONE).any())
        # 5. one batched implicit step of every env still running
        self.targets = self.targets_for(self.pose, self.q)
        self.last_reports = self.world.step(self.sc, targets=self.targets, enable=stepping)
        self.steps[stepping] += 1
        self.phase = nxt
        return True

    def sync_scenes(self):
        """Copy the device state back into the scenes' bodies (gripper links,
        objects) so host-side queries see the final placement."""
        x, v = self.world.get_state()
        off = 0
        for sc in self.scenes:
            n = len(sc.state.gather())
            sc.state.scatter(x[off:off + n])
            _scatter_velocity(sc.state, v[off:off + n])
            off += n

    def run(self, max_ticks=100_000):
        while max_ticks > 0 and self.tick():
            max_ticks -= 1
        return self.outcome
