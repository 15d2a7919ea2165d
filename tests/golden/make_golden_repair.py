"""Golden vectors for the penetrated-grasp repair path, produced by the
UNMODIFIED reference package (build container only; never travels):

    PYTHONPATH=tests/golden/_jaxshim:/root/reference/pkg/src:. \
        python tests/golden/make_golden_repair.py [--dynamics]

* proximity.npz — ref robot/proximity.py on seeded inputs: winding numbers,
  crossing-triangle counts, surface distances, max penetration;
* repair_geom.npz — the geometric half of ref robot/repair.py:98-113
  (penetration before, retraction, cleared) for the reference's own test
  scenes (tests/test_robot.py:515-567) and 32 synthetic envs of config 4
  (paper_2311_05945_b200.workloads.repair_batch, seed 4);
* repair_full.npz (--dynamics) — complete ref repair_grasp runs (retraction,
  AutoGrasp with springs to the input pose, penetration after).
"""

from __future__ import annotations

import os
import sys

import numpy as np

from srsim.bodies import AffineBody as RAffine
from srsim.data import data_path
from srsim.geometry.mesh import SurfaceMesh as RSurface
from srsim.geometry.mesh import box_surface, fibonacci_sphere
from srsim.robot import Gripper as RGripper
from srsim.robot import parse_urdf, top_down_pose
from srsim.robot import proximity as RP
from srsim.robot import repair as RR

OUT = os.path.dirname(os.path.abspath(__file__))
CUBE_Y = 0.02515
rng = np.random.default_rng(20231111)


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def pj():
    return RGripper(parse_urdf(data_path("pj_gripper.urdf")))


def _rot(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def proximity():
    sph = fibonacci_sphere(200, radius=0.04)
    box = box_surface(0.05)
    pts = rng.uniform(-0.06, 0.06, size=(96, 3))
    w_sph = RP.winding_numbers(pts, sph.vertices, sph.triangles)
    w_box = RP.winding_numbers(pts, box.vertices, box.triangles)
    d_sph = RP.surface_distance(pts, sph)
    pen_sph = RP.max_penetration(pts, sph)
    # crossing counts between randomly placed meshes (some overlapping)
    pairs_a, pairs_b, counts = [], [], []
    meshes = [fibonacci_sphere(60, radius=0.03), box_surface(0.04), fibonacci_sphere(120, 0.02),
              box_surface((0.06, 0.02, 0.03))]
    for _ in range(24):
        ia, ib = rng.integers(0, len(meshes), size=2)
        va = meshes[ia].vertices @ _rot(rng).T + rng.uniform(-0.02, 0.02, 3)
        vb = meshes[ib].vertices @ _rot(rng).T + rng.uniform(-0.02, 0.02, 3)
        pairs_a.append(va)
        pairs_b.append(vb)
        counts.append(RP.count_mesh_intersections(
            va, np.asarray(meshes[ia].triangles, np.int64), vb,
            np.asarray(meshes[ib].triangles, np.int64)))
        pairs_a[-1] = (int(ia), va)
        pairs_b[-1] = (int(ib), vb)
    arrs = {}
    for k, ((ia, va), (ib, vb)) in enumerate(zip(pairs_a, pairs_b)):
        arrs[f"pair{k}_a"] = va
        arrs[f"pair{k}_b"] = vb
        arrs[f"pair{k}_ids"] = np.array([ia, ib])
    for i, m in enumerate(meshes):
        arrs[f"mesh{i}_v"] = m.vertices
        arrs[f"mesh{i}_t"] = np.asarray(m.triangles, np.int64)
    samples = RP.surface_samples(box.vertices, box.triangles, box.edges)
    save("proximity.npz", pts=pts, sph_v=sph.vertices, sph_t=np.asarray(sph.triangles, np.int64),
         box_v=box.vertices, box_t=np.asarray(box.triangles, np.int64), w_sph=w_sph, w_box=w_box,
         d_sph=d_sph, pen_sph=pen_sph, counts=np.array(counts), box_samples=samples, **arrs)


def _geom_repair(obj, gripper, pose, joints, open_offset=0.01):
    """ref repair.py:98-113 verbatim through the reference's own helpers."""
    obj_mesh = RR._world_mesh(obj)
    gripper.place(pose, joints)
    pen_before = RP.max_penetration(RR._hand_points(gripper), obj_mesh)
    opened = gripper.clamp_joints(joints - open_offset)
    normal = gripper.palm_normal(pose)
    retraction, cleared = 0.0, False
    while retraction <= RR.RETRACT_MAX:
        probe = pose.copy()
        probe[:3, 3] -= retraction * normal
        gripper.place(probe, opened)
        if not RR._hand_object_overlap(gripper, obj_mesh):
            cleared = True
            break
        retraction += RR.RETRACT_STEP
    return pen_before, retraction, cleared


def scenes():
    """(name, object verts, tris, pose, joints): ref tests + config-4 envs."""
    out = []
    cube = box_surface(0.05, center=(0.0, CUBE_Y, 0.0))
    out.append(("already_clear", cube.vertices, cube.triangles,
                top_down_pose((0.0, CUBE_Y, 0.0)), [0.0, 0.0]))
    out.append(("fingers_inside", cube.vertices, cube.triangles,
                top_down_pose((0.0, CUBE_Y, 0.0)), [0.021, 0.021]))
    out.append(("palm_inside", cube.vertices, cube.triangles,
                top_down_pose((0.0, 0.05015 - 0.06 - 0.010, 0.0)), [0.0, 0.0]))
    sph = fibonacci_sphere(200, radius=0.04)
    out.append(("hand_inside_sphere", sph.vertices + np.array([0.0, 0.06, 0.0]), sph.triangles,
                top_down_pose((0.0, 0.03, 0.0)), [0.0, 0.0]))
    big = box_surface(1.2, center=(0.0, 0.6, 0.0))
    out.append(("unsalvageable", big.vertices, big.triangles,
                top_down_pose((0.0, 0.6, 0.0)), [0.0, 0.0]))
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2311_05945_b200.workloads import repair_batch

    objs, poses, joints = repair_batch(32, seed=4)
    for i, (o, p, q) in enumerate(zip(objs, poses, joints)):
        out.append((f"batch{i}", o.world_vertices(), o.mesh.triangles, p, q))
    return out


def repair_geom():
    rows = scenes()
    arrs = {"names": np.array([r[0] for r in rows])}
    pen, ret, clr = [], [], []
    for k, (name, v, t, pose, q) in enumerate(rows):
        obj = RAffine(RSurface(v, t), density=500.0)
        pb, r, c = _geom_repair(obj, pj(), np.asarray(pose, np.float64), np.asarray(q, np.float64))
        pen.append(pb)
        ret.append(r)
        clr.append(c)
        arrs[f"s{k}_v"] = np.asarray(v, np.float64)
        arrs[f"s{k}_t"] = np.asarray(t, np.int64)
        arrs[f"s{k}_pose"] = np.asarray(pose, np.float64)
        arrs[f"s{k}_q"] = np.asarray(q, np.float64)
        print(name, pb, r, c, flush=True)
    save("repair_geom.npz", pen_before=np.array(pen), retraction=np.array(ret),
         cleared=np.array(clr), **arrs)


def repair_full():
    rows = [r for r in scenes() if r[0] in ("palm_inside", "hand_inside_sphere")]
    arrs = {}
    for k, (name, v, t, pose, q) in enumerate(rows):
        obj = RAffine(RSurface(v, t), density=500.0)
        g = pj()
        r = RR.repair_grasp(obj, g, np.asarray(pose, np.float64), np.asarray(q, np.float64))
        arrs[f"s{k}_name"] = np.array(name)
        arrs[f"s{k}_v"] = np.asarray(v, np.float64)
        arrs[f"s{k}_t"] = np.asarray(t, np.int64)
        arrs[f"s{k}_pose"] = np.asarray(pose, np.float64)
        arrs[f"s{k}_q"] = np.asarray(q, np.float64)
        arrs[f"s{k}_result"] = np.array([r.cleared, r.retraction_m, r.penetration_before_m,
                                         r.penetration_after_m, r.trial.steps], dtype=np.float64)
        arrs[f"s{k}_outcome"] = np.array(str(r.trial.outcome))
        arrs[f"s{k}_forces"] = np.array(r.trial.forces)
        arrs[f"s{k}_obj_q"] = obj.q.copy()
        arrs[f"s{k}_links_q"] = np.array([b.q for b in g.bodies()])
        print(name, r.cleared, r.retraction_m, r.penetration_before_m, r.penetration_after_m,
              r.trial.steps, r.trial.outcome, flush=True)
    save("repair_full.npz", n=len(rows), **arrs)


def repair_geom_hand(n=16, seed=4):
    """The geometric repair of config 4 with the three-finger revolute hand
    (paper_2311_05945_b200/data/dex_hand.urdf, a URDF the reference's own
    parser and Gripper load): n synthetic penetrated grasps
    (workloads.repair_batch_hand)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2311_05945_b200 import data_path as our_data
    from paper_2311_05945_b200.workloads import repair_batch_hand

    urdf = our_data("dex_hand.urdf")
    objs, poses, joints = repair_batch_hand(n, seed=seed)
    arrs = {}
    pen, ret, clr = [], [], []
    for k, (o, p, q) in enumerate(zip(objs, poses, joints)):
        v, t = o.world_vertices(), o.mesh.triangles
        obj = RAffine(RSurface(v, t), density=500.0)
        g = RGripper(parse_urdf(urdf))
        pb, r, c = _geom_repair(obj, g, np.asarray(p, np.float64), np.asarray(q, np.float64))
        pen.append(pb)
        ret.append(r)
        clr.append(c)
        arrs[f"s{k}_v"] = np.asarray(v, np.float64)
        arrs[f"s{k}_t"] = np.asarray(t, np.int64)
        arrs[f"s{k}_pose"] = np.asarray(p, np.float64)
        arrs[f"s{k}_q"] = np.asarray(q, np.float64)
        print("hand", k, pb, r, c, flush=True)
    save("repair_geom_hand.npz", pen_before=np.array(pen), retraction=np.array(ret),
         cleared=np.array(clr), n=n, **arrs)


if __name__ == "__main__":
    if "--hand" in sys.argv:
        repair_geom_hand()
        raise SystemExit(0)
    proximity()
    repair_geom()
    if "--dynamics" in sys.argv:
        repair_full()
