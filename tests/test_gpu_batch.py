"""Batched environments on one GPU vs per-environment CPU oracle runs."""

import numpy as np
import pytest

from oracle import stepper as S
from oracle.robot import OracleBackend

pytestmark = pytest.mark.gpu


def test_scheduled_batch_matches_oracle_per_env():
    """Config 3 workload: every env of a batch tracks its own oracle run
    step by step (DoFs within 1e-6 relative, same Newton iteration counts)."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 6, 14
    scenes, grippers, half, poses = WL.grasp_batch(E, seed=3)
    sched = WL.schedule(grippers, half, poses, K)
    ref_scenes, _, _, _ = WL.grasp_batch(E, seed=3)
    w = GpuWorld(scenes)
    w.upload_schedule(sched)
    lays = [S.Layout(s) for s in ref_scenes]
    nl = len(grippers[0].links)
    off = w.packed.pre["dof"]
    for k in range(K):
        reps = w.step_scheduled(SolverConfig(), k)
        x, _ = w.get_state()
        tg = sched[k].reshape(E, nl, 12)
        for e in range(E):
            for c, t in zip(ref_scenes[e].constraints, tg[e]):
                c.body.target_q = t
            r = S.step(ref_scenes[e], S.Config(), lays[e])
            xr = ref_scenes[e].state.gather()
            xe = x[off[e]:off[e + 1]]
            assert reps[e].newton_iters == r.newton_iters, (k, e)
            assert np.abs(xe - xr).max() <= 1e-6 * np.abs(xr).max(), (k, e)
            assert reps[e].min_dist_after > 0.0


def test_batch_grasp_outcomes_match_oracle():
    """Full AutoGrasp/lift/shake programs for several envs in one batch give
    the same outcome flags and step counts as the oracle run one at a time."""
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.bodies import AffineBody
    from paper_2311_05945_b200.mesh import box_surface
    from paper_2311_05945_b200.robot import (Gripper, GraspTrial, autograsp, build_grasp_scene,
                                             lift_and_shake, parse_urdf, top_down_pose)
    from paper_2311_05945_b200.robot.batch import BatchGrasp

    cy = 0.02515
    cases = [(0.05, 0.0, 0.5), (0.04, 0.3, 0.4), (0.05, 0.0, 0.0), (0.05, 0.0, 0.4)]
    model = parse_urdf(data_path("pj_gripper.urdf"))
    objs, poses = [], []
    for size, yaw, _ in cases:
        objs.append(AffineBody(box_surface(size, center=(0.0, cy, 0.0)), density=500.0))
        poses.append(top_down_pose((0.0, cy, 0.0), yaw=yaw))
    # last case: gripper far above the cube -> fingers meet -> NeverHeld
    poses[3] = top_down_pose((0.0, 0.3, 0.0))
    mus = [c[2] for c in cases]
    bg = BatchGrasp(model, objs, np.array(poses), np.zeros((len(cases), 2)), mu=mus)
    out = bg.run()
    for e, (size, yaw, mu) in enumerate(cases):
        g = Gripper(model)
        o = AffineBody(box_surface(size, center=(0.0, cy, 0.0)), density=500.0)
        sc = build_grasp_scene(o, g, poses[e], [0.0, 0.0], mu=mu)
        tr = GraspTrial(poses[e], np.zeros(2))
        be = OracleBackend()
        autograsp(sc, g, tr, backend=be)
        lift_and_shake(sc, g, o, tr, backend=be)
        assert out[e] == tr.outcome, (e, out[e], tr.outcome)
        assert bg.steps[e] == tr.steps, (e, bg.steps[e], tr.steps)
        np.testing.assert_allclose(np.array(bg.forces[e]), np.array(tr.forces), rtol=1e-3, atol=1e-4)


def test_run_scheduled_matches_per_step_fused():
    """Asynchronous range (each env runs its own steps back to back) gives the
    per-step fused schedule's states bit for bit, and the default (hybrid)
    per-step schedule's to 1e-9, including the contact-onset steps."""
    import os

    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 12, 10
    cfg = SolverConfig()

    def fresh():
        scenes, grippers, half, poses = WL.grasp_batch(E, seed=5)
        w = GpuWorld(scenes)
        w.upload_schedule(WL.schedule(grippers, half, poses, K))
        return w

    wa = fresh()
    reps_a = wa.run_scheduled(cfg, 0, K)
    xa, va = wa.get_state()
    wf = fresh()
    wf.set_fused(True)
    for k in range(K):
        reps_f = wf.step_scheduled(cfg, k)
    xf, vf = wf.get_state()
    assert np.array_equal(xa, xf) and np.array_equal(va, vf)
    assert [r.newton_iters for r in reps_a] == [r.newton_iters for r in reps_f]
    if os.environ.get("IPC_FUSED") != "1":
        wh = fresh()
        wh.set_fused(False)
        for k in range(K):
            wh.step_scheduled(cfg, k)
        xh, _ = wh.get_state()
        assert np.abs(xa - xh).max() <= 1e-9 * np.abs(xh).max()


def _pinch_job(q_close):
    """One job of batch_run: 6 steps of the rigid pinch closing to q_close;
    returns (Newton counts, final DoFs)."""
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.bodies import AffineBody
    from paper_2311_05945_b200.mesh import box_surface
    from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose
    from paper_2311_05945_b200.solver import SolverConfig, step

    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, 0.02515, 0.0)), density=500.0)
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, 0.02515, 0.0)), [0.015, 0.015], mu=0.5)
    its = []
    for _ in range(6):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, q_close))
        its.append(step(sc, SolverConfig())[1].newton_iters)
    return its, sc.state.gather()


def test_batch_run_gpu_workers_ordered_and_equal_to_serial():
    """ref batch.py:39 on GPUs: 2 spawned workers (each on a device) return
    the jobs' results in job order, identical to running them in-process."""
    from paper_2311_05945_b200.batch import batch_run

    jobs = [0.02, 0.022, 0.0262]
    par = batch_run(_pinch_job, jobs, workers=2)
    ser = batch_run(_pinch_job, jobs, workers=1)
    assert [r.job_id for r in par] == [0, 1, 2] and all(r.ok for r in par)
    for a, b in zip(par, ser):
        assert a.value[0] == b.value[0]
        assert np.array_equal(a.value[1], b.value[1])


def test_step_report_phase_times():
    """StepReport.times splits the device step into the reference's phases
    (ref solver.py:52, batch.py:66): contact steps spend time in DCD, Energy,
    Linear and CCD, and the phases cover the wall time."""
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.batch import profile_phases
    from paper_2311_05945_b200.bodies import AffineBody
    from paper_2311_05945_b200.mesh import box_surface
    from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose
    from paper_2311_05945_b200.solver import SolverConfig, step

    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    obj = AffineBody(box_surface(0.05, center=(0.0, 0.02515, 0.0)), density=500.0)
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, 0.02515, 0.0)), [0.018, 0.018], mu=0.5)
    reps = []
    for _ in range(5):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        reps.append(step(sc, SolverConfig())[1])
    prof = profile_phases(reps)
    for k in ("DCD", "Energy", "Linear", "CCD"):
        assert prof[k] > 0.0, k
    for r in reps:
        assert sum(r.times.values()) >= r.total_time * (1 - 1e-9)
        assert all(v >= 0.0 for v in r.times.values())


def test_programmatic_launch_is_bit_identical(monkeypatch):
    """Programmatic dependent launches (the default) and plain launches give
    the same bits: every kernel waits for its predecessor before reading."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 32, 10
    out = {}
    for pdl in ("1", "0"):
        monkeypatch.setenv("IPC_PDL", pdl)
        scenes, grippers, half, poses = WL.grasp_batch(E, seed=5)
        w = GpuWorld(scenes)
        w.upload_schedule(WL.schedule(grippers, half, poses, K))
        its = [[r.newton_iters for r in w.step_scheduled(SolverConfig(), k)] for k in range(K)]
        out[pdl] = (w.get_state()[0].copy(), its)
        del w
    assert out["1"][1] == out["0"][1]
    assert np.array_equal(out["1"][0], out["0"][0])


def test_env_start_order_is_scheduling_only(monkeypatch):
    """The heaviest-first start order of the per-env CTAs (k_env_order) only
    reorders scheduling: identity order gives the same bits."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 48, 10
    out = {}
    for order in ("1", "0"):
        monkeypatch.setenv("IPC_ENV_ORDER", order)
        scenes, grippers, half, poses = WL.grasp_batch(E, seed=11)
        w = GpuWorld(scenes)
        w.upload_schedule(WL.schedule(grippers, half, poses, K))
        its = [[r.newton_iters for r in w.step_scheduled(SolverConfig(), k)] for k in range(K)]
        out[order] = (w.get_state()[0].copy(), its)
        del w
    assert out["1"][1] == out["0"][1]
    assert np.array_equal(out["1"][0], out["0"][0])


@pytest.mark.parametrize("knob,value", [("IPC_SS_PAD", "0"), ("IPC_LOOP_GRAPH", "0")])
def test_bit_identical_knobs(monkeypatch, knob, value):
    """Knobs that only change how the step is scheduled or searched give the
    same bits: no candidate superset (plain broad phase, separate world-position
    launch) and the host-driven Newton loop instead of the conditional graph."""
    from paper_2311_05945_b200 import workloads as WL
    from paper_2311_05945_b200.solver import SolverConfig
    from paper_2311_05945_b200.world import GpuWorld

    E, K = 48, 10
    out = {}
    for v in (None, value):
        if v is None:
            monkeypatch.delenv(knob, raising=False)
        else:
            monkeypatch.setenv(knob, v)
        scenes, grippers, half, poses = WL.grasp_batch(E, seed=5)
        w = GpuWorld(scenes)
        w.upload_schedule(WL.schedule(grippers, half, poses, K))
        its = [[r.newton_iters for r in w.step_scheduled(SolverConfig(), k)] for k in range(K)]
        out[v] = (w.get_state()[0].copy(), its)
        del w
    assert out[None][1] == out[value][1]
    assert np.array_equal(out[None][0], out[value][0])
