"""Config 2 (soft cube of 6·d³ tets in the parallel-jaw gripper) step by step
on the GPU: wall ms, Newton / PCG iterations, and the per-kernel device time
of every step (CUDA events; the world profiles itself for StepReport.times).

    python tools/config2_steps.py [divisions] [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig, engine_of, step  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sc, g, cube = WL.soft_grasp(d)
cfg = SolverConfig()
prev = None
for k in range(n):
    g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
    w = engine_of(sc)
    st0 = w.stats()
    t0 = time.perf_counter()
    _, rep = step(sc, cfg)
    dt = time.perf_counter() - t0
    w = engine_of(sc)
    st1 = w.stats()
    prof, _ = w.profile_read()
    ms = {kk: v[0] for kk, v in prof.items()}
    dms = {kk: round(ms[kk] - (prev or {}).get(kk, 0.0), 3) for kk in ms if ms[kk] - (prev or {}).get(kk, 0.0) > 0.01}
    prev = ms
    print(json.dumps({"step": k, "ms": round(dt * 1e3, 2), "newton": rep.newton_iters,
                      "pcg_iters": st1["pcg_iters"] - st0["pcg_iters"],
                      "phases_ms": {kk: round(1e3 * v, 2) for kk, v in rep.times.items()},
                      "kernels_ms": dms}), flush=True)
