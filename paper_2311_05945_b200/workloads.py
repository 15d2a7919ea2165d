"""Synthetic grasp workloads (BASELINE.json configs; no datasets offline).

``grasp_batch(n_env, seed)`` builds the parallel-grasp-generation batch of
config 3: each environment is the two-finger parallel-jaw gripper
(data/pj_gripper.urdf) plus one rigid affine object — a box or a Fibonacci
sphere with seeded random size and resolution — resting on the ground.
``schedule(...)`` is the open-loop command stream used by the benchmark:
the fingers close at 1 mm/step from 3 mm away to a 2 mm squeeze, then the
hand lifts 5 cm over 50 steps (the AutoGrasp + Lift phases of ref
robot/grasp.py with the force feedback replaced by a fixed squeeze so the
command stream can live in device memory).
"""

from __future__ import annotations

import numpy as np

from . import data_path
from .bodies import AffineBody, Material, SoftBody
from .mesh import box_surface, box_tet, fibonacci_sphere
from .robot.batch import batch_fk
from .robot.grasp import build_grasp_scene
from .robot.gripper import Gripper, top_down_pose
from .robot.urdf import parse_urdf

GAP = 1.5e-4          # object rests this far above the ground
HALF_APERTURE = 0.045  # finger inner face to midplane, fully open
CLOSE_RATE = 1e-3
SQUEEZE = 2e-3
LIFT_START, LIFT_STEPS, LIFT_HEIGHT = 8, 50, 0.05


def gripper_model():
    return parse_urdf(data_path("pj_gripper.urdf"))


def grasp_object(rng, kind=None):
    """One synthetic rigid object; returns (body, half width along the jaw axis, yaw)."""
    kind = kind or ("box" if rng.random() < 0.5 else "sphere")
    density = float(rng.uniform(300.0, 800.0))
    if kind == "box":
        size = np.array([rng.uniform(0.03, 0.07), rng.uniform(0.03, 0.06), rng.uniform(0.03, 0.06)])
        c = (0.0, 0.5 * size[1] + GAP, 0.0)
        return AffineBody(box_surface(size, center=c), density=density), 0.5 * size[0], 0.0
    r = float(rng.uniform(0.015, 0.03))
    nv = int(rng.integers(40, 121))
    m = fibonacci_sphere(nv, r)
    m = m.transformed(translation=(0.0, r + GAP, 0.0))
    yaw = float(rng.uniform(0, np.pi))
    axis = np.array([np.cos(yaw), 0.0, np.sin(yaw)])
    return AffineBody(m, density=density), float(np.abs(m.vertices @ axis).max()), yaw


def grasp_batch(n_env: int, seed: int = 0, mu: float = 0.5, select=None):
    """Scenes, grippers and per-env half widths for config 3.

    ``select``: env indices (increasing) of the n_env-env batch to build —
    a rank's shard, or one env of a CPU-sample task; the objects are drawn
    from the same random stream, so env e is the same scene whichever subset
    is built."""
    rng = np.random.default_rng(seed)
    model = gripper_model()
    keep = None if select is None else set(int(e) for e in select)
    scenes, grippers, half, poses = [], [], [], []
    for e in range(n_env):
        obj, hw, yaw = grasp_object(rng)
        if keep is not None and e not in keep:
            continue
        top = float(obj.world_vertices()[:, 1].max())
        g = Gripper(model)
        q0 = max(0.0, HALF_APERTURE - hw - 3e-3)
        pose = top_down_pose((0.0, max(0.5 * top, 0.022), 0.0), yaw=yaw)
        sc = build_grasp_scene(obj, g, pose, [q0, q0], mu=mu)
        scenes.append(sc)
        grippers.append(g)
        half.append(hw)
        poses.append(pose)
    return scenes, grippers, np.array(half), np.array(poses)


def schedule(grippers, half, poses, n_steps: int) -> np.ndarray:
    """Kinematic targets for steps 1..n_steps: (n_steps, E * n_links * 12)."""
    E = len(grippers)
    g0 = grippers[0]
    links = sorted(g0.links)
    q0 = np.maximum(0.0, HALF_APERTURE - half - 3e-3)
    qmax = HALF_APERTURE - half + SQUEEZE
    out = np.empty((n_steps, E * len(links) * 12))
    for k in range(1, n_steps + 1):
        q = np.minimum(q0 + CLOSE_RATE * k, qmax)
        q = np.stack([q, q], axis=1)
        pose = poses.copy()
        lift = np.clip((k - LIFT_START) / LIFT_STEPS, 0.0, 1.0) * LIFT_HEIGHT
        pose[:, 1, 3] += lift
        fk = batch_fk(g0, pose, q)
        per = [np.concatenate([fk[ln][:, :3, 3], fk[ln][:, :3, :3].reshape(-1, 9)], axis=1)
               for ln in links]
        out[k - 1] = np.stack(per, axis=1).reshape(-1)
    return out


def soft_drop(divisions: int = 6, E: float = 1e5):
    """Config 0: soft tet cube (6·d³ tets) dropped on the ground plane."""
    from .bodies import GlobalState
    from .scene import make_scene

    body = SoftBody(box_tet(0.05, divisions, center=(0.0, 0.03, 0.0)),
                    Material(youngs_modulus=E, poisson_ratio=0.3, density=1000.0))
    return make_scene(GlobalState(soft_bodies=[body]), ground_y=0.0, dhat=1e-3)


def soft_grasp(divisions: int = 12, mu: float = 0.5):
    """Config 2: the gripper pinching a soft tet cube (6·d³ tets)."""
    cy = 0.02515
    g = Gripper(gripper_model())
    cube = SoftBody(box_tet(0.05, divisions, center=(0.0, cy, 0.0)),
                    Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    sc = build_grasp_scene(cube, g, top_down_pose((0.0, cy, 0.0)), [0.0, 0.0], mu=mu)
    return sc, g, cube


def repair_batch(n_env: int, seed: int = 0):
    """Config 4: penetrated grasps to repair (ref robot/repair.py:82).

    Each env is the parallel-jaw gripper on one synthetic rigid object (a box
    or a Fibonacci sphere, ``grasp_object``) with the palm pushed 0-15 mm into
    the object top and each finger commanded up to 5 mm past contact, so the
    input placement interpenetrates. Returns (objects, poses (E,4,4),
    joints (E,2)). The objects are fresh bodies: a caller may build scenes
    from them.
    """
    rng = np.random.default_rng(seed)
    objs, poses, joints = [], [], []
    for _ in range(n_env):
        obj, hw, yaw = grasp_object(rng)
        top = float(obj.world_vertices()[:, 1].max())
        depth = float(rng.uniform(0.0, 0.015))
        # the palm face sits 6 cm above the grasp target of top_down_pose
        # (ref tests/test_robot.py:534: target 0.06 + 10 mm below the top)
        pose = top_down_pose((0.0, top - 0.06 - depth, 0.0), yaw=yaw)
        qc = HALF_APERTURE - hw
        q = np.clip(qc + rng.uniform(-0.004, 0.005, size=2), 0.0, 0.045)
        objs.append(obj)
        poses.append(pose)
        joints.append(q)
    return objs, np.array(poses), np.array(joints)


def hand_model():
    """Three-finger revolute hand (data/dex_hand.urdf) of config 4."""
    return parse_urdf(data_path("dex_hand.urdf"))


def repair_batch_hand(n_env: int, seed: int = 0):
    """Config 4 with the dexterous hand: penetrated grasps of the three-finger
    revolute hand (data/dex_hand.urdf) on the synthetic objects of
    ``grasp_object``. The palm face is pushed 0-15 mm into the object top
    and every joint is curled to 0.3-0.8 rad, so phalanges cut into the
    object. Returns (objects, poses (E,4,4), joints (E,6))."""
    rng = np.random.default_rng(seed)
    objs, poses, joints = [], [], []
    for _ in range(n_env):
        obj, hw, yaw = grasp_object(rng)
        top = float(obj.world_vertices()[:, 1].max())
        depth = float(rng.uniform(0.0, 0.015))
        # the palm face (local z = 0.01) sits 0.065 above the grasp target
        pose = top_down_pose((0.0, top - 0.065 - depth, 0.0), yaw=float(rng.uniform(0, 2 * np.pi)))
        q = rng.uniform(0.3, 0.8, size=6)
        objs.append(obj)
        poses.append(pose)
        joints.append(q)
    return objs, np.array(poses), np.array(joints)
