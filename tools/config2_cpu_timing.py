"""Config-2 CPU baseline: the oracle port (numpy/scipy splu, one core) on the
golden config-2 run (10,368-tet soft cube in the gripper, the steps of
tests/golden/traj_soft_grasp_c2.npz through contact onset); checks each step
against the golden and prints ms per step.

    python tools/config2_cpu_timing.py [steps]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import stepper as S  # noqa: E402
from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200.bodies import Material, SoftBody  # noqa: E402
from paper_2311_05945_b200.mesh import box_tet  # noqa: E402
from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose  # noqa: E402

CUBE_Y = 0.02515
z = dict(np.load(os.path.join(ROOT, "tests", "golden", "traj_soft_grasp_c2.npz")))
n = min(int(sys.argv[1]) if len(sys.argv) > 1 else len(z["x"]), len(z["x"]))
g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
d = int(z["divisions"])
obj = SoftBody(box_tet(0.05, d, center=(0.0, CUBE_Y, 0.0)),
               Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
q0 = float(z["q0"])
sc = build_grasp_scene(obj, g, top_down_pose((0.0, CUBE_Y, 0.0)), [q0, q0], mu=0.5)
lay = S.Layout(sc)
ms, worst, same = [], 0.0, True
for k in range(n):
    g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
    t0 = time.perf_counter()
    r = S.step(sc, S.Config(), lay)
    ms.append(1e3 * (time.perf_counter() - t0))
    x = sc.state.gather()
    worst = max(worst, float(np.abs(x - z["x"][k]).max() / np.abs(z["x"][k]).max()))
    same &= int(r.newton_iters) == int(z["newton_iters"][k])
print(json.dumps({"scene": f"config 2, {d}^3*6 = {6 * d ** 3} tets, {n} golden steps, oracle port on one core",
                  "ms_per_step": ms, "mean_ms": float(np.mean(ms)), "median_ms": float(np.median(ms)),
                  "same_newton_counts_as_reference": bool(same), "max_rel_dof_vs_reference": worst}, indent=1))
