"""CUDA path vs the CPU oracle and the reference's golden vectors (needs a GPU).

Tolerances: integer / index outputs (regions, candidate lists, grasp
outcomes, Newton iteration counts) must match exactly; fp64 DoF states
within 1e-6 relative per step (north_star), element derivatives within
1e-9 relative of the reference autodiff.
"""

import numpy as np
import pytest

from oracle import collide as C
from oracle import energies as E
from oracle import stepper as S
from oracle.robot import OracleBackend

pytestmark = pytest.mark.gpu

REL = 1e-6  # per-step DoF tolerance (north_star: "within 1e-6 relative")


@pytest.fixture(scope="module")
def native():
    from paper_2311_05945_b200 import _native

    return _native


def test_distance_kernels_match_reference(native, golden):
    z = golden("distance.npz")
    for kind in ("pt", "ee"):
        reg, s, g, h = native.dist2_derivs(kind, z[kind])
        assert np.array_equal(reg, z[f"{kind}_region"])
        np.testing.assert_allclose(s, z[f"{kind}_s"], rtol=1e-12, atol=1e-14)
        gs = np.abs(z[f"{kind}_g"]).max(axis=1, keepdims=True)
        assert np.all(np.abs(g - z[f"{kind}_g"]) <= 1e-9 * gs + 1e-14)
        hs = np.abs(z[f"{kind}_h"]).max(axis=(1, 2), keepdims=True)
        assert np.all(np.abs(h - z[f"{kind}_h"]) <= 1e-8 * hs + 1e-14)


def test_ccd_kernel_matches_reference(native, golden):
    z = golden("ccd.npz")
    for kind in ("pt", "ee"):
        a = native.ccd_pairs(kind, z["px"], z["pdx"])
        np.testing.assert_allclose(a, z[f"alpha_{kind}"], rtol=1e-12)


@pytest.mark.parametrize("dim", [6, 9, 12])
def test_psd_projection(native, dim):
    rng = np.random.default_rng(dim)
    m = rng.standard_normal((200, dim, dim))
    m = m + np.swapaxes(m, 1, 2)
    m[:50] = m[:50] @ np.swapaxes(m[:50], 1, 2)  # some already PSD
    got = native.psd_project(m)
    want = E.psd(m)
    np.testing.assert_allclose(got, want, atol=1e-10 * np.abs(m).max())
    assert np.linalg.eigvalsh(got).min() >= -1e-9 * np.abs(m).max()


@pytest.mark.parametrize("model", [0, 1, 2])
def test_elastic_models(native, model):
    names = ("NeoHookean", "StVK", "FixedCorotated")
    rng = np.random.default_rng(7 + model)
    F = np.eye(3) + 0.2 * rng.standard_normal((300, 3, 3))
    F = F[np.linalg.det(F) > 0.2]
    mu, lam = 3.8e4, 5.7e4
    psi, P, H = native.elastic_eval(model, F, mu, lam)
    rp, rP, rH = E.elastic_pk1_hess(F, names[model], mu, lam)
    np.testing.assert_allclose(psi, rp, rtol=1e-10)
    np.testing.assert_allclose(P, rP, rtol=1e-8, atol=1e-8 * np.abs(rP).max())
    np.testing.assert_allclose(H, rH, rtol=1e-7, atol=1e-8 * np.abs(rH).max())


# ---------------------------------------------------------------------------
# whole-step parity
# ---------------------------------------------------------------------------
from test_oracle_golden import CUBE_Y, contact_scene  # noqa: E402
from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200.bodies import AffineBody, GlobalState, Material, SoftBody  # noqa: E402
from paper_2311_05945_b200.mesh import box_surface, box_tet  # noqa: E402
from paper_2311_05945_b200.robot import (Gripper, GraspTrial, autograsp,  # noqa: E402
                                         build_grasp_scene, lift_and_shake, parse_urdf,
                                         top_down_pose)
from paper_2311_05945_b200.scene import make_scene  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig, step  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402


def test_candidates_match_oracle(golden):
    z = golden("contact.npz")
    sc = contact_scene()
    sc.state.scatter(z["x"])
    w = GpuWorld([sc])
    assert np.array_equal(w.candidates(0, 0), z["cand_pt"])
    assert np.array_equal(w.candidates(0, 1), z["cand_ee"])
    assert np.array_equal(w.candidates(0, 2), z["cand_ground"])
    md = w.min_distance()[0]
    assert md == pytest.approx(float(z["min_dist"]), rel=1e-12)


def test_soft_drop_trajectory(golden):
    z = golden("traj_soft_drop.npz")
    body = SoftBody(box_tet(0.05, 3, center=(0.0, 0.03, 0.0)),
                    Material(youngs_modulus=1e5, poisson_ratio=0.3, density=1000.0))
    sc = make_scene(GlobalState(soft_bodies=[body]), ground_y=0.0, dhat=1e-3)
    cfg = SolverConfig()
    for k in range(len(z["x"])):
        _, rep = step(sc, cfg)
        x = sc.state.gather()
        assert rep.newton_iters == z["newton_iters"][k], k
        assert np.abs(x - z["x"][k]).max() <= REL * np.abs(z["x"][k]).max(), k
        assert rep.min_dist_after > 0.0


def test_pinch_steps(golden):
    z = golden("traj_pinch_steps.npz")
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, CUBE_Y, 0.0)), [0.0, 0.0], mu=0.5)
    cfg = SolverConfig()
    for k in range(len(z["x"])):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        _, rep = step(sc, cfg)
        assert rep.newton_iters == z["newton_iters"][k], k
        x = sc.state.gather()
        assert np.abs(x - z["x"][k]).max() <= REL * np.abs(z["x"][k]).max(), k
        assert rep.min_dist_after > 0.0


def test_grasp_trial_flags_match_reference(golden):
    z = golden("traj_grasp_rigid.npz")
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    sc = build_grasp_scene(obj, g, pose, [0.0, 0.0], mu=float(z["mu"]))
    tr = GraspTrial(pose, np.zeros(2))
    autograsp(sc, g, tr)
    lift_and_shake(sc, g, obj, tr)
    assert tr.outcome == str(z["outcome"]) and tr.steps == int(z["steps"])
    np.testing.assert_allclose(np.array(tr.forces), z["forces"], rtol=1e-5, atol=1e-5)
    x = sc.state.gather()
    assert np.abs(x - z["x_final"]).max() <= 1e-5 * np.abs(z["x_final"]).max()


def test_config0_soft_drop_sparse_path_matches_oracle():
    """Config 0 (~1.3k tets, 1029 DoFs): BSR assembly + PCG path, per step
    against the oracle (splu direct solve)."""
    from paper_2311_05945_b200 import workloads as WL

    a, b = WL.soft_drop(divisions=6), WL.soft_drop(divisions=6)
    lay = S.Layout(b)
    cfg = SolverConfig()
    for k in range(25):
        _, rep = step(a, cfg)
        r = S.step(b, S.Config(), lay)
        xa, xb = a.state.gather(), b.state.gather()
        assert rep.newton_iters == r.newton_iters, k
        assert np.abs(xa - xb).max() <= REL * np.abs(xb).max(), k
        assert rep.min_dist_after > 0.0
    assert a.barrier.kappa == b.barrier.kappa


def test_soft_cube_grasp_trial_matches_reference(golden):
    z = golden("traj_grasp_soft.npz")
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = SoftBody(box_tet(0.05, 2, center=(0.0, CUBE_Y, 0.0)),
                   Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    sc = build_grasp_scene(obj, g, pose, [0.0, 0.0], mu=float(z["mu"]))
    tr = GraspTrial(pose, np.zeros(2))
    autograsp(sc, g, tr)
    lift_and_shake(sc, g, obj, tr)
    assert tr.outcome == str(z["outcome"]) and tr.steps == int(z["steps"])
    np.testing.assert_allclose(np.array(tr.forces), z["forces"], rtol=1e-4, atol=1e-4)
    x = sc.state.gather()
    assert np.abs(x - z["x_final"]).max() <= 1e-5 * np.abs(z["x_final"]).max()


@pytest.mark.parametrize("items", [None, "256"])
def test_broad_phase_variants_identical(monkeypatch, items):
    """The shared-memory broad phase (one CTA per env, staged boxes), the
    global-memory one, and the multi-CTA split (count + write passes) give
    bit-identical, identically ordered candidate lists on a grasp batch."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 8, 6
    cfg = SolverConfig()

    def run(env):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        scenes, grippers, half, poses = WL.grasp_batch(E, seed=11)
        w = GpuWorld(scenes)
        w.upload_schedule(WL.schedule(grippers, half, poses, K))
        for k in range(K):
            w.step_scheduled(cfg, k, want_reports=False)
        return [[w.candidates(e, which) for which in (0, 1, 2)] for e in range(E)], w.get_state()[0]

    base = {"IPC_BROAD_SM": "1"}
    alt = {"IPC_BROAD_SM": "0"}
    if items:
        alt["IPC_BROAD_ITEMS"] = items  # force several CTAs per env in the global version
    ca, xa = run(base)
    cb, xb = run(alt)
    for e in range(E):
        for which in range(3):
            assert np.array_equal(ca[e][which], cb[e][which]), (e, which)
    assert np.array_equal(xa, xb)


def _config2_scene(z):
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    d = int(z["divisions"])
    obj = SoftBody(box_tet(0.05, d, center=(0.0, CUBE_Y, 0.0)),
                   Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    q0 = float(z["q0"])
    return build_grasp_scene(obj, g, pose, [q0, q0], mu=0.5), g


def test_config2_soft_grasp_10k_tets_matches_reference(golden):
    """Config 2 at full size (10,368 tets, 6,627 DoFs, sparse BSR + PCG
    path) against the unmodified reference (make_golden.py
    traj_soft_grasp_config2): fingers close from 4 mm through contact onset
    into a 6 mm squeeze; identical Newton counts and AL outer counts, DoFs
    within 1e-6 relative every step, never intersecting."""
    z = golden("traj_soft_grasp_c2.npz")
    sc, g = _config2_scene(z)
    assert sc.state.n_dof == z["x"].shape[1]
    cfg = SolverConfig()
    for k in range(len(z["x"])):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        _, rep = step(sc, cfg)
        x = sc.state.gather()
        assert rep.newton_iters == z["newton_iters"][k], k
        assert rep.al_outer == z["al_outer"][k], k
        assert np.abs(x - z["x"][k]).max() <= REL * np.abs(z["x"][k]).max(), k
        assert rep.min_dist_after > 0.0
        # a distance: agrees to the DoF tolerance (absolute, scaled by max |x|)
        assert abs(rep.min_dist_after - z["min_dist"][k]) <= REL * np.abs(z["x"][k]).max(), k
    assert sc.barrier.kappa == float(z["kappa"])


@pytest.mark.parametrize("divisions", [8, 12])
def test_lbvh_broad_phase_identical_to_chunk_walk(golden, monkeypatch, divisions):
    """The LBVH culling of large bodies (lbvh.cuh: device radix sort, Karras
    build, refit, traversal) gives bit-identical, identically ordered
    candidate lists to the chunk walk, on the config-2 soft grasp (the soft
    cube's 1728 surface triangles and ~2600 edges get trees) before and
    during the squeeze."""
    from paper_2311_05945_b200.world import GpuWorld

    z = dict(golden("traj_soft_grasp_c2.npz"))
    z["divisions"] = divisions
    sc, g = _config2_scene(z)
    cfg = SolverConfig()
    states = [sc.state.gather()]
    for _ in range(6):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        step(sc, cfg)
        states.append(sc.state.gather())
    lists = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("IPC_LBVH", flag)
        w = GpuWorld([sc])
        out = []
        for x in states:
            w.set_state(x, np.zeros_like(x))
            out.append([w.candidates(0, which) for which in (0, 1, 2)])
        lists[flag] = out
    for a, b in zip(lists["1"], lists["0"]):
        for which in range(3):
            assert np.array_equal(a[which], b[which]), which
    assert sum(len(a[0]) + len(a[1]) for a in lists["1"]) > 0
