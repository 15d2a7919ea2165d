"""Pin the CPU oracle to golden vectors produced by the unmodified reference
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from oracle import collide as C
from oracle import distance as D
from oracle import energies as E
from oracle import stepper as S
from oracle.robot import OracleBackend
from paper_2311_05945_b200 import data_path
from paper_2311_05945_b200.bodies import AffineBody, GlobalState, Material, SoftBody
from paper_2311_05945_b200.mesh import box_surface, box_tet, fibonacci_sphere
from paper_2311_05945_b200.robot import (Gripper, GraspTrial, autograsp, build_grasp_scene,
                                         lift_and_shake, parse_urdf, top_down_pose)
from paper_2311_05945_b200.scene import make_scene
from paper_2311_05945_b200.solver import SolverConfig


def _dense(term, n):
    g = np.zeros(n)
    np.add.at(g, term.gi, term.gv)
    h = np.zeros((n, n))
    np.add.at(h, (term.hr, term.hc), term.hv)
    return g, h


def test_distance_regions_and_values(golden):
    z = golden("distance.npz")
    pt, ee = z["pt"], z["ee"]
    reg = D.pt_regions(*[pt[:, i] for i in range(4)])
    assert np.array_equal(reg, z["pt_region"])
    d2, _ = D.pt_dist2(*[pt[:, i] for i in range(4)], reg)
    assert np.array_equal(d2, z["pt_d2"])
    reg, par = D.ee_regions(*[ee[:, i] for i in range(4)])
    assert np.array_equal(reg, z["ee_region"])
    assert np.array_equal(par, z["ee_parallel"])
    d2, _ = D.ee_dist2(*[ee[:, i] for i in range(4)], reg)
    assert np.array_equal(d2, z["ee_d2"])


@pytest.mark.parametrize("kind", ["pt", "ee"])
def test_distance_derivatives_match_reference_autodiff(golden, kind):
    z = golden("distance.npz")
    s, g, h = D.dist2_derivatives(z[kind], z[f"{kind}_region"], kind)
    np.testing.assert_allclose(s, z[f"{kind}_s"], rtol=1e-12, atol=1e-14)
    scale = np.abs(z[f"{kind}_g"]).max(axis=1, keepdims=True)
    assert np.all(np.abs(g - z[f"{kind}_g"]) <= 1e-10 * scale + 1e-14)
    hs = np.abs(z[f"{kind}_h"]).max(axis=(1, 2), keepdims=True)
    assert np.all(np.abs(h - z[f"{kind}_h"]) <= 1e-9 * hs + 1e-14)


def test_barrier(golden):
    z = golden("barrier.npz")
    b, db, d2b = E.barrier_sq(z["s"], float(z["dhat"]) ** 2)
    assert np.array_equal(b, z["bs"]) and np.array_equal(db, z["dbs"])
    assert np.array_equal(d2b, z["d2bs"])


@pytest.mark.parametrize("model", ["NeoHookean", "StVK", "FixedCorotated"])
def test_elastic(golden, model):
    z = golden("elastic.npz")
    body = SoftBody(box_tet(0.05, 2), Material(model=model, youngs_modulus=1e5, poisson_ratio=0.3))
    t = E.elastic(body, z[f"{model}_x"], 0)
    g, h = _dense(t, body.dof)
    assert t.value == pytest.approx(float(z[f"{model}_value"]), rel=1e-12)
    np.testing.assert_allclose(g, z[f"{model}_grad"], rtol=1e-9, atol=1e-9 * np.abs(g).max())
    np.testing.assert_allclose(h, z[f"{model}_hess"], rtol=1e-7, atol=1e-9 * np.abs(h).max())


def test_orthogonality(golden):
    z = golden("orthogonality.npz")
    bodies = [AffineBody(box_surface(0.1 + 0.05 * i), density=800.0) for i in range(6)]
    scene = make_scene(GlobalState(affine_bodies=bodies))
    t = E.orthogonality(z["x"], S.Layout(scene))
    g, h = _dense(t, 72)
    assert t.value == pytest.approx(float(z["value"]), rel=1e-12)
    np.testing.assert_allclose(g, z["grad"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(h, z["hess"], rtol=1e-8, atol=1e-9 * np.abs(h).max())


def contact_scene():
    soft = SoftBody(box_tet(0.04, 2, center=(0.0, 0.0205, 0.0)),
                    Material(youngs_modulus=5e4, poisson_ratio=0.3, density=500.0))
    box = AffineBody(box_surface(0.04), density=700.0)
    c, s = np.cos(0.3), np.sin(0.3)
    box.set_pose(np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]]), np.array([0.0, 0.0655, 0.004]))
    ball = AffineBody(fibonacci_sphere(60, 0.02), density=900.0)
    ball.set_pose(np.eye(3), np.array([0.0415, 0.021, 0.0]))
    return make_scene(GlobalState(soft_bodies=[soft], affine_bodies=[box, ball]),
                      ground_y=0.0, dhat=2e-3, mu=0.4)


def test_contact_candidates_energy_friction_ccd(golden):
    z = golden("contact.npz")
    sc = contact_scene()
    assert sc.barrier.kappa == float(z["kappa"])
    n = sc.state.n_dof
    xw = sc.cindex.world_positions(z["x"])
    cand = C.broad_phase(xw, sc.tables, sc.barrier.dhat, sc.ground_y)
    assert np.array_equal(cand.pt, z["cand_pt"])
    assert np.array_equal(cand.ee, z["cand_ee"])
    assert np.array_equal(cand.ground, z["cand_ground"])
    t, md = E.contact(xw, cand, sc.tables, sc.cindex, sc.barrier.dhat, sc.barrier.kappa, 0.0)
    g, h = _dense(t, n)
    assert t.value == pytest.approx(float(z["value"]), rel=1e-11)
    assert md == pytest.approx(float(z["min_dist"]), rel=1e-12)
    np.testing.assert_allclose(g, z["grad"], rtol=1e-8, atol=1e-9 * np.abs(g).max())
    np.testing.assert_allclose(h, z["hess"], rtol=1e-6, atol=1e-8 * np.abs(h).max())
    lags = E.friction_lags(xw, cand, sc.tables, sc.cindex, sc.barrier.dhat, sc.barrier.kappa, 0.0)
    assert np.array_equal(lags.slots, z["lag_slots"])
    np.testing.assert_allclose(lags.lam, z["lag_lam"], rtol=1e-9)
    np.testing.assert_allclose(lags.gamma, z["lag_gamma"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(lags.tangent, z["lag_tangent"], rtol=1e-8, atol=1e-12)
    assert np.array_equal(lags.g_slots, z["lag_gslots"])
    np.testing.assert_allclose(lags.g_lam, z["lag_glam"], rtol=1e-12)
    xw2 = sc.cindex.world_positions(z["x2"])
    ft = E.friction(xw2, xw, lags, sc.mu, sc.eps_v, 0.01, sc.cindex)
    fg, fh = _dense(ft, n)
    assert ft.value == pytest.approx(float(z["fvalue"]), rel=1e-9)
    np.testing.assert_allclose(fg, z["fgrad"], rtol=1e-7, atol=1e-8 * np.abs(fg).max())
    np.testing.assert_allclose(fh, z["fhess"], rtol=1e-6, atol=1e-8 * np.abs(fh).max())
    sweep = C.broad_phase_ccd(xw, z["dx"], sc.tables, inflation=sc.barrier.dhat, ground_y=0.0)
    assert np.array_equal(sweep.pt, z["sweep_pt"])
    assert np.array_equal(sweep.ee, z["sweep_ee"])
    assert np.array_equal(sweep.ground, z["sweep_ground"])
    a = C.ccd_alpha(xw, z["dx"], sweep, sc.tables, 0.0)
    assert a == pytest.approx(float(z["alpha"]), rel=1e-12)


def test_ccd_pairs(golden):
    z = golden("ccd.npz")
    np.testing.assert_allclose(C.pair_ccd(z["px"], z["pdx"], "pt"), z["alpha_pt"], rtol=1e-12)
    np.testing.assert_allclose(C.pair_ccd(z["px"], z["pdx"], "ee"), z["alpha_ee"], rtol=1e-12)


def test_soft_drop_trajectory(golden):
    z = golden("traj_soft_drop.npz")
    body = SoftBody(box_tet(0.05, 3, center=(0.0, 0.03, 0.0)),
                    Material(youngs_modulus=1e5, poisson_ratio=0.3, density=1000.0))
    sc = make_scene(GlobalState(soft_bodies=[body]), ground_y=0.0, dhat=1e-3)
    lay = S.Layout(sc)
    for k in range(len(z["x"])):
        rep = S.step(sc, S.Config(), lay)
        assert rep.newton_iters == z["newton_iters"][k]
        x = sc.state.gather()
        assert np.abs(x - z["x"][k]).max() <= 1e-9 * np.abs(z["x"][k]).max()
    assert sc.barrier.kappa == float(z["kappa"])


CUBE_Y = 0.02515


def test_pinch_steps(golden):
    z = golden("traj_pinch_steps.npz")
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, CUBE_Y, 0.0)), [0.0, 0.0], mu=0.5)
    assert sc.barrier.dhat == float(z["dhat"]) and sc.barrier.kappa == float(z["kappa"])
    lay = S.Layout(sc)
    for k in range(len(z["x"])):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        rep = S.step(sc, S.Config(), lay)
        assert rep.newton_iters == z["newton_iters"][k]
        assert np.abs(sc.state.gather() - z["x"][k]).max() <= 1e-8 * np.abs(z["x"][k]).max()


@pytest.mark.parametrize("name,soft", [("traj_grasp_rigid.npz", False),
                                       ("traj_grasp_soft.npz", True)])
def test_grasp_trial_outcome(golden, name, soft):
    z = golden(name)
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    if soft:
        obj = SoftBody(box_tet(0.05, 2, center=(0.0, CUBE_Y, 0.0)),
                       Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    else:
        obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    sc = build_grasp_scene(obj, g, pose, [0.0, 0.0], mu=float(z["mu"]))
    be = OracleBackend()
    tr = GraspTrial(pose, np.zeros(2))
    autograsp(sc, g, tr, backend=be)
    lift_and_shake(sc, g, obj, tr, backend=be)
    assert tr.outcome == str(z["outcome"]) and tr.steps == int(z["steps"])
    np.testing.assert_allclose(np.array(tr.forces), z["forces"], rtol=1e-6, atol=1e-6)
    x = sc.state.gather()
    assert np.abs(x - z["x_final"]).max() <= 1e-7 * np.abs(z["x_final"]).max()


def test_config2_first_steps(golden):
    """Oracle vs the reference on config 2 at full size (10,368 tets): the
    first two steps (the GPU test covers all 12)."""
    z = golden("traj_soft_grasp_c2.npz")
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    d = int(z["divisions"])
    obj = SoftBody(box_tet(0.05, d, center=(0.0, CUBE_Y, 0.0)),
                   Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    q0 = float(z["q0"])
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, CUBE_Y, 0.0)), [q0, q0], mu=0.5)
    lay = S.Layout(sc)
    for k in range(2):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        r = S.step(sc, S.Config(), lay)
        x = sc.state.gather()
        assert r.newton_iters == z["newton_iters"][k]
        assert np.abs(x - z["x"][k]).max() <= 1e-10 * np.abs(z["x"][k]).max()
