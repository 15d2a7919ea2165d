"""CPU-only tests: C-ABI surface, scene packing, batched kinematics and
control law, workload generation, and the multi-rank (gloo) gather path."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ipc_b200.h")).read()
    return sorted(set(re.findall(r"^(?:const char \*|int )\s*(ipc_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_2311_05945_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, s
    # no device here: loading with require_device fails loudly, no fallback
    lib2 = _native.load(require_device=False)
    if lib2.ipc_device_count() == 0:
        with pytest.raises(_native.NativeError):
            _native.load(require_device=True)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2311_05945_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", txt, re.M), f


def _grasp_scene(yaw=0.0, soft=False):
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.bodies import AffineBody, Material, SoftBody
    from paper_2311_05945_b200.mesh import box_surface, box_tet
    from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose

    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    if soft:
        o = SoftBody(box_tet(0.05, 2, center=(0, 0.02515, 0)), Material(density=500.0))
    else:
        o = AffineBody(box_surface(0.05, center=(0, 0.02515, 0)), density=500.0)
    return build_grasp_scene(o, g, top_down_pose((0, 0.02515, 0), yaw=yaw), [0.0, 0.0]), g


def test_packing_layout_is_consistent():
    from paper_2311_05945_b200.world import Packed

    s1, _ = _grasp_scene()
    s2, _ = _grasp_scene(0.4, soft=True)
    P = Packed([s1, s2])
    a = P.arr
    pre = P.pre
    assert P.E == 2 and pre["dof"][-1] == s1.state.n_dof + s2.state.n_dof
    # slot DoF indices land inside their env's DoF range
    for e in range(2):
        sd = a["slot_dof"][pre["slot"][e]:pre["slot"][e + 1]]
        assert sd.min() >= pre["dof"][e] and sd.max() < pre["dof"][e + 1]
    # primitives grouped by body (engine precondition for body culling)
    for k in ("slot_cbody", "tri_cbody", "edge_cbody"):
        assert np.all(np.diff(a[k]) >= 0), k
    # world positions recomputed from the packed arrays match the scene's
    x = a["x0"]
    for e, sc in enumerate((s1, s2)):
        s0, s1_ = pre["slot"][e], pre["slot"][e + 1]
        rest = a["slot_rest"].reshape(-1, 3)[s0:s1_]
        aff = a["slot_aff"][s0:s1_].astype(bool)
        dof = a["slot_dof"][s0:s1_]
        xw = np.empty((s1_ - s0, 3))
        for i in range(len(xw)):
            d = dof[i]
            xw[i] = x[d:d + 3] + (x[d + 3:d + 12].reshape(3, 3) @ rest[i] if aff[i] else 0.0)
        np.testing.assert_allclose(xw, sc.world_slots(), atol=1e-15)
    # excluded pairs are symmetric bitmasks (palm-finger adjacency)
    ex = a["cbody_excl"]
    assert ex.dtype == np.uint64 and np.any(ex != 0)


def test_batch_fk_matches_gripper_fk():
    from paper_2311_05945_b200.robot.batch import batch_fk
    from paper_2311_05945_b200.robot.gripper import top_down_pose

    _, g = _grasp_scene()
    rng = np.random.default_rng(0)
    poses = np.array([top_down_pose(rng.standard_normal(3) * 0.1, yaw=rng.uniform(0, 3)) for _ in range(5)])
    q = rng.uniform(0, 0.045, (5, 2))
    fk = batch_fk(g, poses, q)
    for e in range(5):
        ref = g.fk(poses[e], q[e])
        for ln in g.links:
            np.testing.assert_allclose(fk[ln][e], ref[ln], atol=1e-15)


def test_phi_vectorized_matches_scalar():
    from paper_2311_05945_b200.robot import phi
    from paper_2311_05945_b200.robot.batch import phi_vec

    f = np.array([0.0, 0.1, 0.25, 0.49, 0.5, 2.0])
    np.testing.assert_allclose(phi_vec(f), [phi(v) for v in f], rtol=1e-15)
    assert phi(0.25) == pytest.approx((np.exp(-5) - np.exp(-10)) / (1 - np.exp(-10)), rel=1e-15)


def test_workload_is_deterministic_and_feasible():
    from oracle import collide as C
    from oracle import energies as E
    from paper_2311_05945_b200 import workloads as WL

    a = WL.grasp_batch(6, seed=5)
    b = WL.grasp_batch(6, seed=5)
    for sa, sb in zip(a[0], b[0]):
        assert np.array_equal(sa.state.gather(), sb.state.gather())
    sched = WL.schedule(a[1], a[2], a[3], 12)
    assert sched.shape == (12, 6 * 3 * 12)
    # every initial state is intersection-free (finite barrier energy)
    for sc in a[0]:
        xw = sc.world_slots()
        cand = C.broad_phase(xw, sc.tables, sc.barrier.dhat, sc.ground_y)
        t, md = E.contact(xw, cand, sc.tables, sc.cindex, sc.barrier.dhat, sc.barrier.kappa,
                          sc.ground_y, derivatives=False)
        assert np.isfinite(t.value) and md > 0


def _oracle_rows(n_total, lo, hi, steps, seed=5):
    """Per-env result rows of envs [lo, hi) of an n_total-env config-3 batch,
    stepped by the oracle: (env, Newton total, final-DoF checksum)."""
    from oracle import stepper as OS
    from paper_2311_05945_b200 import workloads as WL

    scenes, grippers, half, poses = WL.grasp_batch(n_total, seed=seed, select=range(lo, hi))
    sched = WL.schedule(grippers, half, poses, steps)
    nl = len(grippers[0].links)
    rows = []
    for i, sc in enumerate(scenes):
        lay, tot = OS.Layout(sc), 0
        for k in range(steps):
            for c, t12 in zip(sc.constraints, sched[k].reshape(len(scenes), nl, 12)[i]):
                c.body.target_q = t12
            tot += OS.step(sc, OS.Config(), lay).newton_iters
        x = sc.state.gather()
        rows.append([lo + i, tot, float(np.sum(x * np.arange(1, len(x) + 1)))])
    return np.array(rows)


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    t, n = bench.gather_timing(10.0 + rank, 100 * (rank + 1))
    lo, hi = bench.shard_range(3, world, rank)  # ragged: 1 + 2 envs
    rows = bench.gather_env_rows(_oracle_rows(3, lo, hi, steps=2))
    out[rank] = (t, n, bench.shard_seed(0, rank), rows)
    dist.destroy_process_group()


def test_multirank_shard_and_gather_gloo():
    """Strong-scaling shards of a config-3 batch stepped on 2 ranks, per-env
    results gathered in env order, equal a 1-process run of the whole batch."""
    import multiprocessing as mp
    import socket

    import bench

    assert [bench.shard_range(1024, 8, r) for r in (0, 7)] == [(0, 128), (896, 1024)]
    assert sum(hi - lo for lo, hi in (bench.shard_range(1000, 3, r) for r in range(3))) == 1000
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    assert out[0][:2] == out[1][:2] == (11.0, 300.0)
    assert out[0][2] != out[1][2]  # weak scaling: disjoint env batches
    whole = _oracle_rows(3, 0, 3, steps=2)
    for r in range(2):
        np.testing.assert_array_equal(out[r][3], whole)


def test_repair_packing_vectorized_equals_per_gripper(monkeypatch):
    """retract_batch's two host packings (one shared URDF model: vectorized
    FK; separate models: per-gripper place()) hand the C-ABI identical arrays."""
    from paper_2311_05945_b200 import _native as N
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.robot import Gripper, parse_urdf
    from paper_2311_05945_b200.robot import repair as R
    from paper_2311_05945_b200.workloads import repair_batch

    captured = []

    class Fake:
        def ipc_repair_retract(self, d, idx):
            d = d._obj
            E = d.n_env
            L = d.env_link[E]
            HV, HT = d.link_vert[L], d.link_tri[L]
            OV, OT = d.env_obj_vert[E], d.env_obj_tri[E]
            arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy()  # noqa: E731
            captured.append({"env_link": arr(d.env_link, E + 1), "link_vert": arr(d.link_vert, L + 1),
                             "link_tri": arr(d.link_tri, L + 1), "hand_v": arr(d.hand_v, 3 * HV),
                             "hand_t": arr(d.hand_t, 3 * HT), "obj_v": arr(d.obj_v, 3 * OV),
                             "obj_t": arr(d.obj_t, 3 * OT), "normal": arr(d.normal, 3 * E),
                             "retr": arr(d.retraction, d.n_probe)})
            return 0

    monkeypatch.setattr(N, "load", lambda *a, **k: Fake())
    objs, poses, joints = repair_batch(6, seed=3)
    meshes = [R._world_mesh(o) for o in objs]
    model = parse_urdf(data_path("pj_gripper.urdf"))
    shared = [Gripper(model) for _ in range(6)]
    separate = [Gripper(parse_urdf(data_path("pj_gripper.urdf"))) for _ in range(6)]
    opened = np.array([shared[0].clamp_joints(q - 0.01) for q in joints])
    R.retract_batch(shared, poses, opened, meshes)
    R.retract_batch(separate, poses, opened, meshes)
    a, b = captured
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(a["retr"], R.retraction_schedule()[0])


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` with WORLD_SIZE unset re-launches itself as 2
    ranks (torch.distributed.run); rank 0 alone prints the reference-arm line."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "3", "--envs", "4",
                          "--cpu-sample", "2"], capture_output=True, text=True, env=env,
                         timeout=600, check=True)
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert lines[0]["scaling"] == "strong" and lines[0]["config"]["envs"] == 4


def _neg_or_fail(x):
    if x == 3:
        raise ValueError("bad job")
    return -x


def test_batch_run_ordered_results_and_failed_slot():
    """ref batch.py:39 contract: ordered results, a raising job marks its slot."""
    from paper_2311_05945_b200.batch import batch_run

    res = batch_run(_neg_or_fail, [1, 2, 3, 4])
    assert [r.job_id for r in res] == [0, 1, 2, 3]
    assert [r.ok for r in res] == [True, True, False, True]
    assert res[1].value == -2 and "ValueError: bad job" in res[2].error
    assert batch_run(_neg_or_fail, []) == []


def test_profile_phases_and_format():
    """ref batch.py:66/:86: phase seconds summed over step reports."""
    from paper_2311_05945_b200.batch import format_profile, profile_phases
    from paper_2311_05945_b200.solver import PHASES, StepReport

    class R:  # the fields a device StepReportC carries
        newton_iters, final_grad_norm, min_dist_before, min_dist_after = 3, 0.0, 1.0, 1.0
        ccd_invocations, converged, line_search_failed, al_outer = 2, 1, 0, 1

    a = StepReport.from_c(R(), 1.0, {"DCD": 0.1, "Energy": 0.2, "Linear": 0.3})
    b = StepReport.from_c(R(), 0.5, {"DCD": 0.1, "CCD": 0.6})  # accounted > total: Others clamps at 0
    assert a.times["Others"] == pytest.approx(0.4) and b.times["Others"] == 0.0
    prof = profile_phases([a, b.as_dict()])
    assert prof["Total"] == 1.5 and prof["DCD"] == pytest.approx(0.2)
    table = format_profile(prof)
    assert all(k in table for k in (*PHASES, "Total"))
