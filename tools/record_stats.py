"""Per-env contact candidate counts of the config-3 batch after k steps (the
record counts the dense assembly iterates over).
    python tools/record_stats.py [steps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
scenes, grippers, half, poses = WL.grasp_batch(1024, seed=0)
sched = WL.schedule(grippers, half, poses, K)
w = GpuWorld(scenes)
w.upload_schedule(sched)
cfg = SolverConfig()
for k in range(K):
    reps = w.step_scheduled(cfg, k)
print("n_dof per env", w.n_dof / 1024, "slots per env", w.n_slot / 1024)
cnt = np.array([[len(w.candidates(e, 0)), len(w.candidates(e, 1)), len(w.candidates(e, 2))]
                for e in range(0, 1024, 8)])
for i, nm in enumerate(("pt", "ee", "ground")):
    c = cnt[:, i]
    print(f"{nm}: mean {c.mean():.1f} median {np.median(c):.0f} p90 {np.percentile(c, 90):.0f} max {c.max()}")
