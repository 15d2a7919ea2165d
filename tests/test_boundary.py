"""The drop-in boundary takes the reference's own scene objects.

``solver.step`` / ``world.GpuWorld`` must accept an UNMODIFIED reference
``srsim`` Scene (ref scene.py:112, bodies.py:167/218): no engine slot on the
scene, no ``gravity_acceleration`` on AffineBody, no ``scatter_velocity`` on
GlobalState. These CPU tests import the reference from /root/reference
(build container only; skipped elsewhere) through the jax shim and check

* ``Packed([srsim_scene])`` hands the C-ABI exactly the arrays
  ``Packed([repo_scene])`` does, for a rigid grasp scene, a soft grasp scene
  and the soft drop (bit-identical, every field of ``ipc_world_desc``);
* ``solver.step`` on a reference scene goes through the host sync path
  (upload, report, download into q/q_dot and x/v, κ, AL multipliers,
  constraint targets) with the device world replaced by a recording fake.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
SHIM = os.path.join(os.path.dirname(__file__), "golden", "_jaxshim")
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def srsim():
    for p in (SHIM, REF):
        if p not in sys.path:
            sys.path.insert(0, p)
    import srsim  # noqa: F401
    import srsim.bodies
    import srsim.geometry.mesh
    import srsim.robot
    import srsim.scene
    import srsim.data
    return srsim


CUBE_Y = 0.02515


def _grasp_scenes(srsim, soft):
    from paper_2311_05945_b200 import bodies as B, mesh as M, scene as S  # noqa: F401
    from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose
    from paper_2311_05945_b200.data import __file__ as data_init

    R = srsim
    rg = R.robot.Gripper(R.robot.parse_urdf(R.data.data_path("pj_gripper.urdf")))
    gg = Gripper(parse_urdf(os.path.join(os.path.dirname(data_init), "pj_gripper.urdf")))
    if soft:
        ro = R.bodies.SoftBody(R.geometry.mesh.box_tet(0.05, 2, center=(0.0, CUBE_Y, 0.0)),
                               R.bodies.Material(youngs_modulus=1e5, poisson_ratio=0.3,
                                                 density=500.0))
        go = B.SoftBody(M.box_tet(0.05, 2, center=(0.0, CUBE_Y, 0.0)),
                        B.Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    else:
        ro = R.bodies.AffineBody(R.geometry.mesh.box_surface(0.05, center=(0.0, CUBE_Y, 0.0)),
                                 density=500.0)
        go = B.AffineBody(M.box_surface(0.05, center=(0.0, CUBE_Y, 0.0)), density=500.0)
    pose = top_down_pose((0.0, CUBE_Y, 0.0))
    rs = R.robot.build_grasp_scene(ro, rg, pose, [0.0, 0.0], mu=0.5)
    gs = build_grasp_scene(go, gg, pose, [0.0, 0.0], mu=0.5)
    return rs, gs, rg, gg


def _drop_scenes(srsim):
    from paper_2311_05945_b200 import bodies as B, mesh as M, scene as S

    R = srsim
    rb = R.bodies.SoftBody(R.geometry.mesh.box_tet(0.05, 3, center=(0.0, 0.03, 0.0)),
                           R.bodies.Material(youngs_modulus=1e5, poisson_ratio=0.3, density=1000.0))
    gb = B.SoftBody(M.box_tet(0.05, 3, center=(0.0, 0.03, 0.0)),
                    B.Material(youngs_modulus=1e5, poisson_ratio=0.3, density=1000.0))
    rs = R.scene.make_scene(R.bodies.GlobalState(soft_bodies=[rb]), ground_y=0.0, dhat=1e-3)
    gs = S.make_scene(B.GlobalState(soft_bodies=[gb]), ground_y=0.0, dhat=1e-3)
    return rs, gs


def _assert_same_packing(a, b):
    assert a.E == b.E
    for k in a.pre:
        np.testing.assert_array_equal(a.pre[k], b.pre[k], err_msg=k)
    assert set(a.arr) == set(b.arr)
    for k in a.arr:
        assert a.arr[k].dtype == b.arr[k].dtype, k
        np.testing.assert_array_equal(a.arr[k], b.arr[k], err_msg=k)
    for k in a.env:
        np.testing.assert_array_equal(a.env[k], b.env[k], err_msg=k)


@pytest.mark.parametrize("soft", [False, True])
def test_packed_reference_grasp_scene(srsim, soft):
    from paper_2311_05945_b200.world import Packed

    rs, gs, _, _ = _grasp_scenes(srsim, soft)
    assert not hasattr(rs, "engine")
    _assert_same_packing(Packed([rs]), Packed([gs]))


def test_packed_reference_soft_drop_and_mixed_batch(srsim):
    from paper_2311_05945_b200.world import Packed

    rs, gs = _drop_scenes(srsim)
    _assert_same_packing(Packed([rs]), Packed([gs]))
    r2, g2, _, _ = _grasp_scenes(srsim, False)
    # a batch may mix reference and repo scenes
    _assert_same_packing(Packed([rs, g2]), Packed([gs, r2]))


class _FakeWorld:
    """Stands in for the device world: records uploads, returns a shifted state."""

    instances = []

    def __init__(self, scenes):
        from paper_2311_05945_b200.world import Packed

        self.packed = Packed(scenes)
        self.n_dof = self.packed.n("dof")
        self.n_cons = self.packed.n("cons")
        self.x = None
        _FakeWorld.instances.append(self)

    def set_state(self, x, v):
        self.x, self.v = np.array(x), np.array(v)

    def set_kappa(self, k):
        self.kappa = float(k[0])

    def step(self, cfg):
        from paper_2311_05945_b200 import _native as N

        r = (N.StepReportC * 1)()
        r[0].newton_iters = 3
        r[0].converged = 1
        self.x = self.x + 1e-3
        self.v = self.v + 2e-3
        return r

    def get_state(self):
        return self.x.copy(), self.v.copy()

    def get_kappa(self):
        return np.array([self.kappa * 2.0])

    def get_constraints(self):
        lam = np.arange(12 * self.n_cons, dtype=np.float64).reshape(-1, 12)
        return lam, np.full(self.n_cons, 7.0)


def test_solver_step_on_reference_scene(srsim, monkeypatch):
    from paper_2311_05945_b200 import solver

    monkeypatch.setattr(solver, "GpuWorld", _FakeWorld)
    rs, _, rg, _ = _grasp_scenes(srsim, False)
    x0, v0 = rs.state.gather(), rs.state.gather_velocity()
    k0 = rs.barrier.kappa
    rg.set_targets(joint_values=[1e-3, 1e-3])
    st, rep = solver.step(rs, solver.SolverConfig())
    assert st is rs.state and rep.newton_iters == 3
    np.testing.assert_array_equal(rs.state.gather(), x0 + 1e-3)
    np.testing.assert_array_equal(rs.state.gather_velocity(), v0 + 2e-3)
    assert type(rs.barrier).__module__.startswith("srsim") and rs.barrier.kappa == 2.0 * k0
    for i, c in enumerate(rs.constraints):
        np.testing.assert_array_equal(c.lam, np.arange(12 * i, 12 * i + 12, dtype=np.float64))
        assert c.kappa == 7.0
        np.testing.assert_array_equal(c.target, c.body.target_q)
    # the world is cached per scene without touching the scene object
    n = len(_FakeWorld.instances)
    solver.step(rs, solver.SolverConfig())
    assert len(_FakeWorld.instances) == n
    solver.release_engine(rs)
