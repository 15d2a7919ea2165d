"""Time the single-environment configurations of BASELINE.json on the GPU
(config 0: soft cube drop; config 1: rigid-cube grasp with mu=0.5; config 2:
soft-cube grasp). Prints one JSON line per config. GPU only."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig, engine_of, step  # noqa: E402


def run(name, scene, n_steps, drive=None):
    cfg = SolverConfig()
    iters, t = [], []
    for k in range(n_steps):
        if drive:
            drive(k)
        t0 = time.perf_counter()
        _, rep = step(scene, cfg)
        t.append(time.perf_counter() - t0)
        iters.append(rep.newton_iters)
    t = np.array(t[3:])
    print(json.dumps({"config": name, "steps": n_steps, "ms_per_step_median": 1e3 * float(np.median(t)),
                      "ms_per_step_mean": 1e3 * float(t.mean()), "newton_mean": float(np.mean(iters)),
                      "n_dof": scene.state.n_dof}), flush=True)


if __name__ == "__main__" and "prof2" not in sys.argv:
    which = sys.argv[1:] or ["0", "1", "2"]
    if "0" in which:
        run("config0 soft cube drop (1296 tets)", WL.soft_drop(6), 40)
    if "1" in which:
        from paper_2311_05945_b200 import data_path
        from paper_2311_05945_b200.bodies import AffineBody
        from paper_2311_05945_b200.mesh import box_surface
        from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose

        g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
        cube = AffineBody(box_surface(0.05, center=(0.0, 0.02515, 0.0)), density=500.0)
        sc = build_grasp_scene(cube, g, top_down_pose((0.0, 0.02515, 0.0)), [0.0, 0.0], mu=0.5)
        run("config1 rigid cube pinch mu=0.5", sc, 40,
            lambda k: g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262)))
    if "2" in which:
        div = int(os.environ.get("DIV", "12"))
        sc, g, cube = WL.soft_grasp(div)
        print("tets", len(cube.mesh.tets), flush=True)
        run(f"config2 soft cube grasp ({len(cube.mesh.tets)} tets)", sc, 30,
            lambda k: g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262)))


def profile_config2(div=12, n=8):
    """Per-kernel event timing of config 2 after a few warm-up steps."""
    sc, g, cube = WL.soft_grasp(div)
    cfg = SolverConfig()
    for k in range(4):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        step(sc, cfg)
    w = engine_of(sc)
    w.profile(True)
    st0 = w.stats()
    t0 = time.perf_counter()
    for k in range(n):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        step(sc, cfg)
    dt = time.perf_counter() - t0
    prof, launches = w.profile_read()
    st1 = w.stats()
    print(f"config2 {n} steps {1e3 * dt / n:.1f} ms/step, launches {launches}, "
          f"{ {k: st1[k] - st0[k] for k in st1} }")
    for name, (ms, c) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:12]:
        print(f"  {name:14s} {ms:9.2f} ms {c:6d} launches {1e3 * ms / max(c, 1):9.1f} us/launch")


if __name__ == "__main__" and "prof2" in sys.argv:
    profile_config2()
