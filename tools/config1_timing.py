"""Config 1 (parallel-jaw gripper grasping, lifting and shaking a rigid 5 cm
cube, mu = 0.5, one env): the full trial of ref robot/grasp.py:224 through
run_grasp_trial on the GPU engine (`--gpu`) or on the oracle port (`--cpu`,
one core); prints wall seconds, steps, outcome.

    python tools/config1_timing.py --cpu|--gpu
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200.bodies import AffineBody  # noqa: E402
from paper_2311_05945_b200.mesh import box_surface  # noqa: E402
from paper_2311_05945_b200.robot import Gripper, parse_urdf, run_grasp_trial, top_down_pose  # noqa: E402

CY = 0.02515
backend = None
if sys.argv[1] == "--cpu":
    from oracle.robot import OracleBackend
    backend = OracleBackend()
g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
obj = AffineBody(box_surface(0.05, center=(0.0, CY, 0.0)), density=500.0)
t0 = time.perf_counter()
trial = run_grasp_trial(obj, g, top_down_pose((0.0, CY, 0.0)), np.zeros(2), backend=backend, mu=0.5)
dt = time.perf_counter() - t0
print(json.dumps({"mode": sys.argv[1], "seconds": dt, "steps": int(trial.steps),
                  "ms_per_step": 1e3 * dt / max(int(trial.steps), 1),
                  "outcome": str(trial.outcome), "forces_tail": np.asarray(trial.forces[-1:]).tolist()}))
