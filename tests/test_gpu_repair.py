"""Penetrated-grasp repair on the GPU (config 4) vs the reference's golden
vectors (tests/golden/make_golden_repair.py) and the CPU oracle
(oracle/proximity.py). Needs a GPU.

Tolerances: crossing counts, containment decisions, cleared flags, probe
indices / retraction distances and grasp outcomes must match exactly;
winding numbers within 1e-12 absolute (atan2 and the per-point summation
order are the only deviations); penetration depths within 1e-12 relative;
post-repair DoFs within 1e-5 relative (the 180-step grasp-trial tolerance of
test_gpu_parity.py).
"""

import numpy as np
import pytest

from oracle import proximity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prox(golden):
    return golden("proximity.npz")


@pytest.fixture(scope="module")
def geom(golden):
    return golden("repair_geom.npz")


def _gripper():
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.robot import Gripper, parse_urdf

    return Gripper(parse_urdf(data_path("pj_gripper.urdf")))


def test_winding_numbers(prox):
    from paper_2311_05945_b200.robot import proximity as G

    for m in ("sph", "box"):
        w = G.winding_numbers(prox["pts"], prox[f"{m}_v"], prox[f"{m}_t"])
        np.testing.assert_allclose(w, prox[f"w_{m}"], rtol=0, atol=1e-12)
        assert ((w > 0.5) == (prox[f"w_{m}"] > 0.5)).all()


def test_crossing_counts_exact(prox):
    from paper_2311_05945_b200.robot import proximity as G

    for k, want in enumerate(prox["counts"]):
        ia, ib = prox[f"pair{k}_ids"]
        got = G.count_mesh_intersections(prox[f"pair{k}_a"], prox[f"mesh{ia}_t"],
                                         prox[f"pair{k}_b"], prox[f"mesh{ib}_t"])
        assert got == int(want), k


def test_max_penetration(prox):
    from paper_2311_05945_b200.robot import proximity as G
    from paper_2311_05945_b200.mesh import SurfaceMesh

    got = G.max_penetration(prox["pts"], SurfaceMesh(prox["sph_v"], prox["sph_t"]))
    assert got == pytest.approx(float(prox["pen_sph"]), rel=1e-12)
    # batched form: per-env maxima, including an env with no contained point
    far = prox["pts"] + 1.0
    out = G.max_penetration_batch([prox["pts"], far, prox["pts"][:5]],
                                  [(prox["sph_v"], prox["sph_t"])] * 3)
    assert out[0] == pytest.approx(float(prox["pen_sph"]), rel=1e-12)
    assert out[1] == 0.0
    assert out[2] == pytest.approx(P.max_penetration(prox["pts"][:5], prox["sph_v"],
                                                     prox["sph_t"]), rel=1e-12, abs=0)


def test_empty_inputs():
    from paper_2311_05945_b200.robot import proximity as G

    v = np.zeros((3, 3))
    assert G.count_mesh_intersections(v, np.zeros((0, 3), np.int64), v, [[0, 1, 2]]) == 0
    assert G.max_penetration_batch([], []).shape == (0,)
    # an env with no sample points, next to one with points inside
    from paper_2311_05945_b200.mesh import box_surface
    from paper_2311_05945_b200.robot.repair import retract_batch

    box = box_surface(0.05)
    out = G.max_penetration_batch([np.zeros((0, 3)), np.zeros((1, 3))],
                                  [(box.vertices, box.triangles)] * 2)
    assert out[0] == 0.0 and out[1] == pytest.approx(0.025, rel=1e-12)
    cleared, r, idx = retract_batch([], [], [], [])
    assert len(cleared) == len(r) == len(idx) == 0


def test_random_crossings_match_oracle():
    """Dense random soups: every crossing decision of the GPU equals the oracle's."""
    from paper_2311_05945_b200.robot import proximity as G

    rng = np.random.default_rng(7)
    for n in (1, 17, 200):
        va, vb = rng.uniform(-1, 1, (3 * n, 3)), rng.uniform(-1, 1, (3 * n, 3))
        t = np.arange(3 * n).reshape(n, 3)
        assert G.count_mesh_intersections(va, t, vb, t) == P.count_mesh_intersections(va, t, vb, t)


def test_retraction_matches_reference_all_scenes(geom):
    """All 37 reference scenes (5 ref-test scenes + 32 config-4 envs) in ONE
    batched launch: cleared flags and retraction distances bit-identical."""
    from paper_2311_05945_b200.robot import Gripper
    from paper_2311_05945_b200.robot.repair import retract_batch

    n = len(geom["cleared"])
    poses = [geom[f"s{k}_pose"] for k in range(n)]
    meshes = [(geom[f"s{k}_v"], geom[f"s{k}_t"]) for k in range(n)]
    g0 = _gripper()
    # one shared URDF model: vectorized host packing; separate models: per-gripper FK
    for gs in ([g0] + [Gripper(g0.model) for _ in range(n - 1)], [_gripper() for _ in range(n)]):
        opened = [g.clamp_joints(geom[f"s{k}_q"] - 0.01) for k, g in enumerate(gs)]
        cleared, r, _ = retract_batch(gs, poses, opened, meshes)
        np.testing.assert_array_equal(cleared, geom["cleared"])
        np.testing.assert_array_equal(r, geom["retraction"])


def test_penetration_before_matches_reference(geom):
    from paper_2311_05945_b200.robot.proximity import max_penetration_batch
    from paper_2311_05945_b200.robot.repair import _hand_points

    n = len(geom["cleared"])
    pts = []
    for k in range(n):
        g = _gripper()
        g.place(geom[f"s{k}_pose"], geom[f"s{k}_q"])
        pts.append(_hand_points(g))
    got = max_penetration_batch(pts, [(geom[f"s{k}_v"], geom[f"s{k}_t"]) for k in range(n)])
    np.testing.assert_allclose(got, geom["pen_before"], rtol=1e-12, atol=1e-15)


def test_repair_grasp_matches_reference(golden):
    """Complete ref repair_grasp runs (retraction + AutoGrasp with springs to
    the input pose) on the ref test scenes palm_inside / hand_inside_sphere."""
    from paper_2311_05945_b200.bodies import AffineBody
    from paper_2311_05945_b200.mesh import SurfaceMesh
    from paper_2311_05945_b200.robot.repair import repair_grasp

    z = golden("repair_full.npz")
    for k in range(int(z["n"])):
        obj = AffineBody(SurfaceMesh(z[f"s{k}_v"], z[f"s{k}_t"]), density=500.0)
        g = _gripper()
        r = repair_grasp(obj, g, z[f"s{k}_pose"], z[f"s{k}_q"])
        cleared, ret, pb, pa, steps = z[f"s{k}_result"]
        assert r.cleared == bool(cleared) and r.retraction_m == ret, k
        assert r.penetration_before_m == pytest.approx(pb, rel=1e-12, abs=1e-15)
        assert r.trial.outcome == str(z[f"s{k}_outcome"]) and r.trial.steps == int(steps), k
        np.testing.assert_allclose(np.array(r.trial.forces), z[f"s{k}_forces"], rtol=1e-5,
                                   atol=1e-5)
        ref_q = np.concatenate([z[f"s{k}_obj_q"], z[f"s{k}_links_q"].ravel()])
        got_q = np.concatenate([obj.q, np.array([b.q for b in g.bodies()]).ravel()])
        assert np.abs(got_q - ref_q).max() <= 1e-5 * np.abs(ref_q).max(), k
        assert r.penetration_after_m == pytest.approx(pa, abs=1e-9)
        # north_star: the final state is intersection-free
        from paper_2311_05945_b200.robot.proximity import count_mesh_intersections

        ov = obj.world_vertices()
        for b in g.bodies():
            assert count_mesh_intersections(b.world_vertices(), b.mesh.triangles, ov,
                                            obj.mesh.triangles) == 0


def test_repair_batch_is_intersection_free(geom):
    """Config 4 in miniature: the batch repair of the 32 golden config-4 envs
    reproduces the reference geometry per env and ends intersection-free."""
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.robot import parse_urdf
    from paper_2311_05945_b200.robot.repair import repair_batch
    from paper_2311_05945_b200.workloads import repair_batch as make

    objs, poses, joints = make(32, seed=4)
    res = repair_batch(parse_urdf(data_path("pj_gripper.urdf")), objs, poses, joints)
    np.testing.assert_array_equal([r.cleared for r in res], geom["cleared"][5:])
    np.testing.assert_array_equal([r.retraction_m for r in res], geom["retraction"][5:])
    np.testing.assert_allclose([r.penetration_before_m for r in res], geom["pen_before"][5:],
                               rtol=1e-12, atol=1e-15)
    assert all(r.penetration_after_m == 0.0 for r in res)
    assert all(r.trial.outcome is not None for r in res)
    # the batch runs each env's program exactly as repair_grasp does alone
    from paper_2311_05945_b200.robot.repair import repair_grasp

    objs2, poses2, joints2 = make(32, seed=4)
    for e in (0, 7, 19):
        r1 = repair_grasp(objs2[e], _gripper(), poses2[e], joints2[e])
        assert (r1.cleared, r1.retraction_m) == (res[e].cleared, res[e].retraction_m)
        assert r1.trial.outcome == res[e].trial.outcome and r1.trial.steps == res[e].trial.steps
        np.testing.assert_allclose(np.array(r1.trial.forces), np.array(res[e].trial.forces),
                                   rtol=1e-6, atol=1e-9)


def test_repair_soft_object():
    """Repair with a soft tet object (the reference's SoftBody branch of
    _world_mesh, repair.py:65): the GPU retraction equals the oracle's probe
    loop on the same surface, and the two-way coupled AutoGrasp ends with no
    crossing triangles and no contained hand samples."""
    from paper_2311_05945_b200.bodies import Material, SoftBody
    from paper_2311_05945_b200.mesh import box_tet
    from paper_2311_05945_b200.robot.gripper import top_down_pose
    from paper_2311_05945_b200.robot.proximity import count_mesh_intersections
    from paper_2311_05945_b200.robot.repair import _world_mesh, repair_grasp

    cy = 0.02515
    cube = SoftBody(box_tet(0.05, 3, center=(0.0, cy, 0.0)),
                    Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    pose = top_down_pose((0.0, 0.05015 - 0.06 - 0.008, 0.0))
    q = np.array([0.02, 0.02])
    ov, ot = _world_mesh(cube)
    g0 = _gripper()
    oc, orr, _ = P.retract(g0, pose, g0.clamp_joints(q - 0.01), ov, np.asarray(ot))
    g = _gripper()
    r = repair_grasp(cube, g, pose, q)
    assert r.cleared == oc and r.retraction_m == orr and orr > 0
    assert r.penetration_before_m > 0 and r.penetration_after_m == 0.0
    assert r.trial.outcome is not None
    sv, st = _world_mesh(cube)
    for b in g.bodies():
        assert count_mesh_intersections(b.world_vertices(), b.mesh.triangles, sv, st) == 0


def test_dexterous_hand_repair_matches_reference(golden):
    """Config 4 with the three-finger revolute hand (data/dex_hand.urdf, 7
    links, 84 triangles — past round 1's 64-triangle staging cap): cleared
    flags and retraction distances bit-identical to the unmodified
    reference's repair loop, penetration-before within 1e-12."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.robot import Gripper
    from paper_2311_05945_b200.robot.proximity import max_penetration_batch
    from paper_2311_05945_b200.robot.repair import _hand_points, retract_batch

    z = golden("repair_geom_hand.npz")
    n = int(z["n"])
    model = WL.hand_model()
    poses = [z[f"s{k}_pose"] for k in range(n)]
    meshes = [(z[f"s{k}_v"], z[f"s{k}_t"]) for k in range(n)]
    gs = [Gripper(model) for _ in range(n)]
    assert sum(len(b.mesh.triangles) for b in gs[0].bodies()) == 84
    opened = [g.clamp_joints(z[f"s{k}_q"] - 0.01) for k, g in enumerate(gs)]
    cleared, r, _ = retract_batch(gs, poses, opened, meshes)
    np.testing.assert_array_equal(cleared, z["cleared"])
    np.testing.assert_array_equal(r, z["retraction"])
    pts = []
    for k in range(n):
        g = Gripper(model)
        g.place(z[f"s{k}_pose"], z[f"s{k}_q"])
        pts.append(_hand_points(g))
    got = max_penetration_batch(pts, meshes)
    np.testing.assert_allclose(got, z["pen_before"], rtol=1e-12, atol=1e-15)


def test_retract_batch_persistent_equals_one_shot():
    """RetractBatch (objects and hand topology packed once) gives the same
    probe indices as retract_batch on the dexterous hand."""
    import bench
    from paper_2311_05945_b200.robot.repair import RetractBatch, retract_batch

    model, objs, poses, joints, grippers, opened, meshes = bench._repair_inputs(48, 7, "dex")
    a = retract_batch(grippers, poses, opened, meshes)
    b = RetractBatch(grippers[0], meshes).run(poses, opened)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
