"""Config 0 (soft tet cube, 6·6³ = 1296 tets, dropped on the ground, dt 1e-2):
per-step wall ms of the GPU path (`--gpu`, public solver.step, cuda:0) or of
the oracle port on one core (`--cpu`), 100 steps by default.

    python tools/config0_timing.py --cpu|--gpu [steps]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_05945_b200 import workloads as WL  # noqa: E402

mode = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sc = WL.soft_drop(6)
ms, its = [], []
if mode == "--cpu":
    from oracle import stepper as S
    lay = S.Layout(sc)
    for k in range(n):
        t0 = time.perf_counter()
        r = S.step(sc, S.Config(), lay)
        ms.append(1e3 * (time.perf_counter() - t0))
        its.append(int(r.newton_iters))
else:
    from paper_2311_05945_b200.solver import SolverConfig, step
    cfg = SolverConfig()
    for k in range(n):
        t0 = time.perf_counter()
        _, r = step(sc, cfg)
        ms.append(1e3 * (time.perf_counter() - t0))
        its.append(int(r.newton_iters))
x = sc.state.gather()
print(json.dumps({"mode": mode, "steps": n, "tets": 1296, "ms_per_step": [round(v, 2) for v in ms],
                  "mean_ms_after_first": float(np.mean(ms[1:])), "newton_iters": its,
                  "x_final_sha": __import__("hashlib").sha256(x.tobytes()).hexdigest()[:16],
                  "x_final": x.tolist()}))
