"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container only (the reference and this script never travel
to the GPU box):

    PYTHONPATH=tests/golden/_jaxshim:/root/reference/pkg/src \
        python tests/golden/make_golden.py

The reference (``srsim``) imports jax for autodiff of its distance formulas;
jax is not installed here, so ``_jaxshim`` maps the few jax calls it makes
onto torch.func (float64). Everything else is the reference's own code.
Outputs: tests/golden/*.npz (small, committed).
"""

from __future__ import annotations

import os

import numpy as np

from srsim.bodies import AffineBody, GlobalState, Material, SoftBody
from srsim.energy.barrier import BarrierParams, barrier, barrier_sq
from srsim.energy.contact import contact_energy
from srsim.energy.elastic import elastic_term
from srsim.energy.friction import friction_term, update_friction_lags
from srsim.energy.term import combine
from srsim.energy.terms import orthogonality_term
from srsim.geometry.broadphase import broad_phase, broad_phase_ccd
from srsim.geometry.ccd import ccd_earliest_alpha, pair_ccd
from srsim.geometry.distance import (edge_edge_dist2, edge_edge_regions, point_triangle_dist2,
                                     point_triangle_regions)
from srsim.geometry.distgrad import dist2_derivatives
from srsim.geometry.mesh import box_surface, box_tet, fibonacci_sphere
from srsim.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose
from srsim.robot.grasp import GraspTrial, autograsp, lift_and_shake
from srsim.data import data_path
from srsim.scene import make_scene
from srsim.solver import SolverConfig, step

OUT = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(20231110)


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


# ---------------------------------------------------------------------------
def distances():
    n = 400
    pt = rng.standard_normal((n, 4, 3))
    ee = rng.standard_normal((n, 4, 3))
    # near-parallel and near-touching edge pairs
    k = 40
    base = rng.standard_normal((k, 3))
    dirn = rng.standard_normal((k, 3))
    ee[:k, 0] = base
    ee[:k, 1] = base + dirn
    ee[:k, 2] = base + 1e-3 * rng.standard_normal((k, 3)) + 0.3 * dirn
    ee[:k, 3] = ee[:k, 2] + dirn * (1.0 + 1e-5 * rng.standard_normal((k, 1))) \
        + 1e-6 * rng.standard_normal((k, 3))
    pr = point_triangle_regions(pt[:, 0], pt[:, 1], pt[:, 2], pt[:, 3])
    pd, _ = point_triangle_dist2(pt[:, 0], pt[:, 1], pt[:, 2], pt[:, 3], regions=pr)
    ps, pg, ph = dist2_derivatives(pt, pr, "pt")
    er, epar = edge_edge_regions(ee[:, 0], ee[:, 1], ee[:, 2], ee[:, 3])
    ed, _, _ = edge_edge_dist2(ee[:, 0], ee[:, 1], ee[:, 2], ee[:, 3], regions=er)
    es, eg, eh = dist2_derivatives(ee, er, "ee")
    save("distance.npz", pt=pt, pt_region=pr, pt_d2=pd, pt_s=ps, pt_g=pg, pt_h=ph,
         ee=ee, ee_region=er, ee_parallel=epar, ee_d2=ed, ee_s=es, ee_g=eg, ee_h=eh)


def barriers():
    dhat = 1e-3
    d = np.linspace(1e-6, 1.5e-3, 200)
    b, db = barrier(d, dhat)
    s = d * d
    bs, dbs, d2bs = barrier_sq(s, dhat * dhat)
    save("barrier.npz", dhat=dhat, d=d, b=b, db=db, s=s, bs=bs, dbs=dbs, d2bs=d2bs)


def elastic():
    out = {}
    for model in ("NeoHookean", "StVK", "FixedCorotated"):
        mesh = box_tet(0.05, 2)
        body = SoftBody(mesh, Material(model=model, youngs_modulus=1e5, poisson_ratio=0.3))
        x = body.x + 4e-3 * rng.standard_normal(body.x.shape)
        t = elastic_term(body, x, 0)
        val, g, (r, c, v) = combine([t], body.dof)
        h = np.zeros((body.dof, body.dof))
        np.add.at(h, (r, c), v)
        out[f"{model}_x"] = x
        out[f"{model}_value"] = val
        out[f"{model}_grad"] = g
        out[f"{model}_hess"] = h
    save("elastic.npz", **out)


def orthogonality():
    bodies = [AffineBody(box_surface(0.1 + 0.05 * i), density=800.0) for i in range(6)]
    state = GlobalState(affine_bodies=bodies)
    x = state.gather() + 0.1 * rng.standard_normal(state.n_dof)
    t = orthogonality_term(x, state)
    val, g, (r, c, v) = combine([t], state.n_dof)
    h = np.zeros((state.n_dof, state.n_dof))
    np.add.at(h, (r, c), v)
    save("orthogonality.npz", x=x, value=val, grad=g, hess=h)


def _contact_scene():
    """Soft cube resting against a tilted affine box and a sphere, plus ground."""
    soft = SoftBody(box_tet(0.04, 2, center=(0.0, 0.0205, 0.0)),
                    Material(youngs_modulus=5e4, poisson_ratio=0.3, density=500.0))
    box = AffineBody(box_surface(0.04), density=700.0)
    c, s = np.cos(0.3), np.sin(0.3)
    box.set_pose(np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]]), np.array([0.0, 0.0655, 0.004]))
    ball = AffineBody(fibonacci_sphere(60, 0.02), density=900.0)
    ball.set_pose(np.eye(3), np.array([0.0415, 0.021, 0.0]))
    state = GlobalState(soft_bodies=[soft], affine_bodies=[box, ball])
    return make_scene(state, ground_y=0.0, dhat=2e-3, mu=0.4)


def contact_and_friction():
    scene = _contact_scene()
    st = scene.state
    x = st.gather()
    x_soft = x.copy()
    x_soft[: st.blocks[0].dof] += 2e-4 * rng.standard_normal(st.blocks[0].dof)
    xw = scene.cindex.world_positions(x_soft)
    cand = broad_phase(xw, scene.tables, scene.barrier.dhat, scene.ground_y)
    term, stats = contact_energy(xw, cand, scene.tables, scene.cindex, scene.barrier,
                                 scene.ground_y)
    val, g, (r, c, v) = combine([term], st.n_dof)
    h = np.zeros((st.n_dof, st.n_dof))
    np.add.at(h, (r, c), v)
    lags = update_friction_lags(xw, cand, scene.tables, scene.cindex, scene.barrier,
                                scene.ground_y)
    x2 = x_soft + 3e-5 * rng.standard_normal(st.n_dof)
    xw2 = scene.cindex.world_positions(x2)
    ft = friction_term(xw2, xw, lags, scene.mu, scene.eps_v, 0.01, scene.cindex)
    fval, fg, (fr, fc, fv) = combine([ft], st.n_dof)
    fh = np.zeros((st.n_dof, st.n_dof))
    np.add.at(fh, (fr, fc), fv)
    # swept candidates + CCD toward a displaced target
    dx = 3e-3 * rng.standard_normal(xw.shape)
    sweep = broad_phase_ccd(xw, dx, scene.tables, inflation=scene.barrier.dhat,
                            ground_y=scene.ground_y)
    alpha = ccd_earliest_alpha(xw, dx, sweep, scene.tables, scene.ground_y)
    save("contact.npz", x=x_soft, x2=x2, dhat=scene.barrier.dhat, kappa=scene.barrier.kappa,
         value=val, grad=g, hess=h, min_dist=stats.min_dist, active=stats.active,
         cand_pt=cand.pt, cand_ee=cand.ee, cand_ground=cand.ground,
         lag_slots=lags.slots, lag_gamma=lags.gamma, lag_tangent=lags.tangent, lag_lam=lags.lam,
         lag_gslots=lags.g_slots, lag_glam=lags.g_lam,
         fvalue=fval, fgrad=fg, fhess=fh,
         dx=dx, sweep_pt=sweep.pt, sweep_ee=sweep.ee, sweep_ground=sweep.ground, alpha=alpha)


def ccd_pairs():
    n = 300
    px = rng.standard_normal((n, 4, 3))
    pdx = 2.0 * rng.standard_normal((n, 4, 3))
    a_pt = pair_ccd(px, pdx, "pt")
    a_ee = pair_ccd(px, pdx, "ee")
    save("ccd.npz", px=px, pdx=pdx, alpha_pt=a_pt, alpha_ee=a_ee)


def traj_soft_drop():
    mat = Material(youngs_modulus=1e5, poisson_ratio=0.3, density=1000.0)
    body = SoftBody(box_tet(0.05, 3, center=(0.0, 0.03, 0.0)), mat)
    scene = make_scene(GlobalState(soft_bodies=[body]), ground_y=0.0, dhat=1e-3)
    cfg = SolverConfig(h=0.01)
    xs, iters = [], []
    for _ in range(40):
        _, rep = step(scene, cfg)
        xs.append(scene.state.gather())
        iters.append(rep.newton_iters)
    save("traj_soft_drop.npz", x=np.array(xs), newton_iters=np.array(iters),
         kappa=scene.barrier.kappa)


CUBE_Y = 0.02515


def traj_grasp(soft: bool, mu: float, name: str, n_auto: int = 25, n_lift: int = 10):
    gripper = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    if soft:
        obj = SoftBody(box_tet(0.05, 2, center=(0.0, CUBE_Y, 0.0)),
                       Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    else:
        obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    scene = build_grasp_scene(obj, gripper, pose, [0.0, 0.0], mu=mu)
    trial = GraspTrial(pose, np.zeros(2))
    autograsp(scene, gripper, trial)
    lift_and_shake(scene, gripper, obj, trial)
    save(name, outcome=trial.outcome, steps=trial.steps, forces=np.array(trial.forces),
         increments=np.array(trial.increments), x_final=scene.state.gather(),
         dhat=scene.barrier.dhat, kappa=scene.barrier.kappa, mu=mu)


def traj_grasp_steps(mu: float, name: str, n: int = 40):
    """Per-step DoF record of the first n steps of a rigid pinch (fixed
    closing command, no force feedback) for step-level parity."""
    gripper = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    scene = build_grasp_scene(obj, gripper, pose, [0.0, 0.0], mu=mu)
    cfg = SolverConfig()
    xs, iters, mind = [], [], []
    for k in range(n):
        gripper.set_targets(joint_values=np.minimum(gripper.joint_values + 1e-3, 0.0262))
        _, rep = step(scene, cfg)
        xs.append(scene.state.gather())
        iters.append(rep.newton_iters)
        mind.append(rep.min_dist_after)
    save(name, x=np.array(xs), newton_iters=np.array(iters), min_dist=np.array(mind),
         dhat=scene.barrier.dhat, kappa=scene.barrier.kappa)


def traj_soft_grasp_config2(n: int = 12, divisions: int = 12, q0: float = 0.016):
    """Config 2 at its full size: the gripper pinching a soft tet cube of
    6·12³ = 10,368 tets (2,197 vertices) with friction μ = 0.5. The fingers
    start 4 mm from the cube and close at 1 mm/step, so contact onset and
    the squeeze fall inside the n recorded steps."""
    gripper = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = SoftBody(box_tet(0.05, divisions, center=(0.0, CUBE_Y, 0.0)),
                   Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    scene = build_grasp_scene(obj, gripper, pose, [q0, q0], mu=0.5)
    cfg = SolverConfig()
    xs, iters, mind, als = [], [], [], []
    for k in range(n):
        gripper.set_targets(joint_values=np.minimum(gripper.joint_values + 1e-3, 0.0262))
        _, rep = step(scene, cfg)
        xs.append(scene.state.gather())
        iters.append(rep.newton_iters)
        mind.append(rep.min_dist_after)
        als.append(rep.al_outer)
        print("config2 step", k, rep.newton_iters, rep.min_dist_after, flush=True)
    save("traj_soft_grasp_c2.npz", x=np.array(xs), newton_iters=np.array(iters),
         min_dist=np.array(mind), al_outer=np.array(als), q0=q0, divisions=divisions,
         dhat=scene.barrier.dhat, kappa=scene.barrier.kappa)


if __name__ == "__main__":
    import sys

    if len(sys.argv) > 1:  # individual targets, e.g. traj_soft_grasp_config2
        for name in sys.argv[1:]:
            globals()[name]()
        raise SystemExit(0)
    distances()
    barriers()
    elastic()
    orthogonality()
    contact_and_friction()
    ccd_pairs()
    traj_soft_drop()
    traj_grasp_steps(0.5, "traj_pinch_steps.npz")
    traj_grasp(False, 0.5, "traj_grasp_rigid.npz")
    traj_grasp(True, 0.4, "traj_grasp_soft.npz")
